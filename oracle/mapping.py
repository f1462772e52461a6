"""Compressed task mapping — Algorithms 1, 2 and 4 of arXiv 2501.16103, in fp-free
integer Python.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Index convention (reading R1): the paper writes tasks 1..N (Alg. 1,
P:161) but Alg. 2 compares ``B >= TilePrefix[t]``, which is the correct
search only for a 0-based block index B.  This module uses 0-based task
indices h, 0-based tile indices l and 0-based block indices B, and follows the
algorithm listing (not the prose of P:167).
"""
from __future__ import annotations

INT32_MAX = 2**31 - 1


# ---------------------------------------------------------------------------
# Algorithm 1 — Build TilePrefix
# ---------------------------------------------------------------------------
def build_tile_prefix(nu: list[int]) -> list[int]:
    """Alg. 1: TilePrefix[i] <- sum_{j<=i} nu(T_j), 0-based storage."""
    out = []
    for i in range(len(nu)):
        out.append(sum(nu[j] for j in range(i + 1)))
    return out


def pad_tile_prefix(prefix: list[int], warp_size: int = 32, mode: str = "max") -> list[int]:
    """pad TilePrefix up to a multiple of the warp size, "by repeating its last
    element or padding with the maximum possible value" (mode 'repeat' | 'max')."""
    if not prefix:
        raise ValueError("empty TilePrefix")
    n_pad = (-len(prefix)) % warp_size
    fill = prefix[-1] if mode == "repeat" else INT32_MAX
    return list(prefix) + [fill] * n_pad


# ---------------------------------------------------------------------------
# Algorithm 4's extra stage — sigma over non-empty tasks
# ---------------------------------------------------------------------------
def nonempty_stage(nu: list[int], order: list[int] | None = None) -> tuple[list[int], list[int]]:
    """Returns (sigma, TilePrefix over the non-empty tasks).

    eta = {S_1..S_M} = tasks with nu > 0; sigma: [M] -> [N] with
    S_i = T_sigma(i), taken in the natural (increasing) order unless ``order``
    (a permutation of the non-empty task ids, §4.2) is given; TilePrefix is built
    "only ... for non-empty tasks", in sigma's order."""
    sigma = [j for j in range(len(nu)) if nu[j] > 0] if order is None else list(order)
    prefix = build_tile_prefix([nu[j] for j in sigma])
    return sigma, prefix


# ---------------------------------------------------------------------------
# Algorithm 2 — warp emulation
# ---------------------------------------------------------------------------
def warp_vote(predicates: list[bool]) -> int:
    """integer mask whose i-th bit is set iff thread i's predicate is true."""
    mask = 0
    for i, p in enumerate(predicates):
        if p:
            mask |= 1 << i
    return mask


def popcount(mask: int) -> int:
    """number of set bits."""
    n = 0
    while mask:
        n += mask & 1
        mask >>= 1
    return n


def mapping_single_warp(prefix_padded: list[int], B: int, warp_size: int = 32) -> tuple[int, int]:
    """Alg. 2 verbatim for one warp-wide chunk (needs len(prefix_padded) == warp_size)."""
    if len(prefix_padded) != warp_size:
        raise ValueError("single-warp mapping needs a warp-sized TilePrefix")
    p = [B >= prefix_padded[t] for t in range(warp_size)]   # line 186
    mask = warp_vote(p)                                      # line 187
    h = popcount(mask)                                       # line 188
    k = 0                                                    # line 189 (k = base offset)
    if h > 0:                                                # line 190
        k = prefix_padded[h - 1]                             # line 191
    l = B - k                                                # line 193
    return h, l


def mapping_chunked(prefix_padded: list[int], B: int, warp_size: int = 32) -> tuple[int, int]:
    """Alg. 2 looped over warp-sized chunks for N > warp size.

    Chunk c contributes popcount(vote(B >= TilePrefix[c*w + t])); the loop stops
    after the first chunk whose popcount is below the warp size (every later
    entry is >= that chunk's failing entry because TilePrefix is non-decreasing)."""
    if len(prefix_padded) % warp_size:
        raise ValueError("TilePrefix must be padded to a multiple of the warp size")
    h = 0
    for c in range(0, len(prefix_padded), warp_size):
        p = [B >= prefix_padded[c + t] for t in range(warp_size)]
        cnt = popcount(warp_vote(p))
        h += cnt
        if cnt < warp_size:
            break
    k = prefix_padded[h - 1] if h > 0 else 0
    return h, B - k


def mapping_extended(prefix_padded: list[int], sigma: list[int], B: int,
                     warp_size: int = 32) -> tuple[int, int, int]:
    """Alg. 4: (h, l) <- mapping(TilePrefix, B); h~ <- sigma(h)."""
    h, l = mapping_chunked(prefix_padded, B, warp_size)
    return h, sigma[h], l


def total_tiles(prefix: list[int]) -> int:
    return prefix[-1] if prefix else 0
