"""MoE application of the static batching framework — fp64 oracle.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Definitions followed (P:n = PAPER.md line n):
* token-index buckets: "a token index array for every expert, containing the
  indices of the tokens routed to the expert"; canonical order within a
  bucket is ascending token id (reading R3 — the paper's atomic
  scatter P:336 leaves it unspecified).
* experts as tasks, tile count nu = ceil(m/BM) * ceil(N/BN) per task
  (K is not split, R4), sigma over non-empty tasks.
* intra-task tile order: row-tile fastest, rt = l mod R, ct = l div R with
  R = ceil(rows/BM) (R5; the paper leaves it open, "tile
  swizzle").
* expert GEMM: Y[row_off[e] + r, :] = X[token_idx_e[r], :] @ W[e] — the unbatched
  per-expert loop of P:100-101 evaluated in fp64 (numpy matmul is the library
  primitive for each expert's product).
* expert parallelism: experts [g*E/G, (g+1)*E/G) live on rank g;
  tokens [g*T/G, (g+1)*T/G) are owned by rank g (R8).
"""
from __future__ import annotations

import numpy as np

from . import mapping


# ---------------------------------------------------------------------------
# c1 — buckets
# ---------------------------------------------------------------------------
def buckets(topk_ids: np.ndarray, E: int):
    """Returns (counts[E], row_off[E+1], token_idx[sum counts], slot[sum counts]).

    token_idx[row_off[e] + r] is the r-th smallest token routed to expert e;
    slot[...] is the top-k position j with topk_ids[t, j] == e.  Raises
    ValueError for ids outside [0, E) or a token listing one expert twice."""
    topk_ids = np.asarray(topk_ids)
    T, k = topk_ids.shape
    lists: list[list[tuple[int, int]]] = [[] for _ in range(E)]
    for t in range(T):
        seen = set()
        for j in range(k):
            e = int(topk_ids[t, j])
            if e < 0 or e >= E:
                raise ValueError(f"expert id {e} out of range")
            if e in seen:
                raise ValueError(f"token {t} routes to expert {e} twice")
            seen.add(e)
            lists[e].append((t, j))          # t visited in ascending order
    counts = np.array([len(b) for b in lists], dtype=np.int64)
    row_off = np.zeros(E + 1, dtype=np.int64)
    for e in range(E):
        row_off[e + 1] = row_off[e] + counts[e]
    token_idx = np.array([t for b in lists for (t, _) in b], dtype=np.int64)
    slot = np.array([j for b in lists for (_, j) in b], dtype=np.int64)
    return counts, row_off, token_idx, slot


# ---------------------------------------------------------------------------
# c2 — plan: experts as tasks, Alg. 1 + Alg. 4's non-empty stage
# ---------------------------------------------------------------------------
def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


def tiles_of(rows: int, N: int, bm: int, bn: int) -> int:
    """nu(T) = ceil(m/BM) * ceil(N/BN); 0 iff m == 0 (SPEC tile_count)."""
    if rows == 0:
        return 0
    return ceil_div(rows, bm) * ceil_div(N, bn)


KIND_GEMV = 2   # a whole task of <= m_max rows computed as a CUDA-core GEMV, outside the tile space
GEMV_MIN_TILES = 128
GEMV_MIN_SHARE = 10   # percent: the candidates' would-be tiles against the other tasks'
KIND_RIDE = 3   # the tail rows ride on the two 256-column halves of the expert's last full row tile


def tail_kind(m: int, bm: int, catalog, bn: int | None = None, N: int | None = None) -> int:
    """The tiling strategy of an expert's last row tile ("categorized into several
    pre-defined tiling strategies"; R6): r = m mod bm rows (0: no partial tile); the first
    catalog rule (kind, m_max) with r <= m_max gives the kind, else kind 0.  A GEMV rule (kind 2) applies
    only to a task that is a single partial row tile (m < bm): the whole task is then that strategy.  A
    RIDE rule (kind 3) applies only to a task with a full row tile (m > bm) in a plan of 256 x 512 tiles
    whose column tiles all lie inside N."""
    r = int(m) % bm
    if int(m) <= 0 or r == 0:
        return 0
    for kind, m_max in catalog:
        if int(kind) == KIND_GEMV and int(m) >= bm:
            continue
        if int(kind) == KIND_RIDE and not (int(m) > bm and bm == 256 and bn == 512 and N is not None
                                           and int(N) % 512 == 0):
            continue
        if r <= m_max:
            return int(kind)
    return 0


def make_tasks(counts, bm: int, bn: int, split_tail: bool = False, catalog=(), N: int | None = None) -> list[dict]:
    """One task per expert with tile bm x bn.

    The mapping is unchanged by the catalog, but an expert's LAST row tile (rows
    [floor(m/bm)*bm, m), or all rows when m < bm) may be executed by a second tiling strategy
    (Alg. 3 with K = 2): kind 1 = a swap-AB tile whose height is those rows
    rounded up to 16.  split_tail = the catalog ((1, bm),).  The tile partition, hence Y, is identical."""
    if split_tail:
        catalog = ((1, bm),)
    return [dict(expert=e, row_begin=0, rows=int(m), bm=bm, bn=bn, kind=tail_kind(m, bm, catalog, bn, N))
            for e, m in enumerate(counts)]


LIGHT_ROWS = 64   # a task of at most this many rows streams its W block (memory-bound)


def order_tasks(loads: list[int], strategy: str) -> list[int]:
    """§4.2 expert ordering over the NON-EMPTY tasks, as SPEC formalises it
    (S:341-346): sort by load descending, ties by lower id; 'alternating' interleaves the
    busiest half with the rest (b1, s1, b2, s2, ...); 'half_interval' puts the i-th busiest
    at the i-th slot of the bit-reversal (van der Corput) sequence over the slot range."""
    ids = [j for j in range(len(loads)) if loads[j] > 0]
    if strategy == "natural":
        return ids
    if strategy == "light_last":
        # DESIGN.md R7 / §6.7: the memory-bound ("light", <= LIGHT_ROWS rows) tasks after every other
        # non-empty task, each group in natural order, so a scheduler can interleave the two groups'
        # tiles in proportion (P:317-320's aim: a wave mixes busy and non-busy experts).
        return [j for j in ids if loads[j] > LIGHT_ROWS] + [j for j in ids if loads[j] <= LIGHT_ROWS]
    desc = sorted(ids, key=lambda j: (-loads[j], j))
    n = len(desc)
    if strategy == "alternating":
        h = (n + 1) // 2
        busy, rest = desc[:h], desc[h:]
        out = []
        for i in range(h):
            out.append(busy[i])
            if i < len(rest):
                out.append(rest[i])
        return out
    if strategy == "half_interval":
        w = 0
        while (1 << w) < n:
            w += 1
        slots = []
        for i in range(1 << w):
            r = int(format(i, f"0{w}b")[::-1], 2) if w else 0
            if r < n:
                slots.append(r)
        out = [None] * n
        for i, j in enumerate(desc):
            out[slots[i]] = j
        return out
    raise ValueError(strategy)


def plan(counts, N: int, bm: int, bn: int, pad_mode: str = "max", warp_size: int = 32,
         tasks: list[dict] | None = None, split_tail: bool = False, order: str = "natural", catalog=()) -> dict:
    """Host-side plan: nu per task, sigma (non-empty tasks, natural order or a §4.2
    ordering), TilePrefix (Alg. 1 over eta in sigma's order), padded per P:203."""
    if tasks is None:
        tasks = make_tasks(counts, bm, bn, split_tail, catalog, N)
        # GEMV rules apply only when the other tasks have >= GEMV_MIN_TILES tiles (their tensor work must
        # cover the GEMV streams) and the candidates are >= GEMV_MIN_SHARE % of the launch's tiles (a handful
        # does not repay the GEMV units' serial streams); otherwise they take the next rule.
        other = sum(tiles_of(t["rows"], N, t["bm"], t["bn"]) for t in tasks if t["kind"] != KIND_GEMV)
        n_gemv = sum(1 for t in tasks if t["kind"] == KIND_GEMV and t["rows"] > 0)
        if n_gemv and (other < GEMV_MIN_TILES or n_gemv * ceil_div(N, bn) * 100 < GEMV_MIN_SHARE * other):
            tasks = make_tasks(counts, bm, bn, split_tail, [r for r in catalog if int(r[0]) != KIND_GEMV], N)
    # Alg. 3's per-task strategies: a GEMV task has no tiles (nu = 0, so the non-empty stage leaves it out
    # of sigma / TilePrefix); its rows are computed by the GEMV strategy (R6, §6.8).
    nu = [0 if t.get("kind", 0) == KIND_GEMV else tiles_of(t["rows"], N, t["bm"], t["bn"]) for t in tasks]
    loads = [t["rows"] if nu[i] > 0 else 0 for i, t in enumerate(tasks)]     # the tasks with tiles (eta)
    sigma, prefix = mapping.nonempty_stage(nu, order_tasks(loads, order) if order != "natural" else None)
    padded = mapping.pad_tile_prefix(prefix, warp_size, pad_mode) if prefix else []
    gemv = [i for i, t in enumerate(tasks) if t.get("kind", 0) == KIND_GEMV and t["rows"] > 0]
    return dict(tasks=tasks, nu=nu, sigma=sigma, prefix=prefix, padded=padded, gemv=gemv,
                M=len(sigma), total=mapping.total_tiles(prefix), N=N, warp_size=warp_size)


# ---------------------------------------------------------------------------
# c3 — decode one virtual tile (block index) into its GEMM tile
# ---------------------------------------------------------------------------
def decode(pl: dict, row_off, B: int) -> dict:
    """Alg. 4 then the intra-task tile split (R5)."""
    if not (0 <= B < pl["total"]):
        raise ValueError("block index out of range")
    h, j, l = mapping.mapping_extended(pl["padded"], pl["sigma"], B, pl["warp_size"])
    task = pl["tasks"][j]
    R = ceil_div(task["rows"], task["bm"])
    rt = l % R
    ct = l // R
    e = task["expert"]
    r0 = int(row_off[e]) + task["row_begin"] + rt * task["bm"]
    r1 = int(row_off[e]) + task["row_begin"] + min((rt + 1) * task["bm"], task["rows"])
    c0 = ct * task["bn"]
    c1 = min(c0 + task["bn"], pl["N"])
    kind = 1 if (task["kind"] == 1 and rt == R - 1) else 0          # the tail tile of a split task
    if task["kind"] == KIND_RIDE and rt >= R - 2:
        # RIDE: slots R-2 / R-1 of the column block are its two 256-column halves, each computing the body
        # rows of row tile R-2 and the tail rows [(R-1) bm, m) — together the rows and columns of slots R-2
        # and R-1 of the plain partition
        half = rt - (R - 2)
        r0 = int(row_off[e]) + task["row_begin"] + (R - 2) * task["bm"]
        r1 = int(row_off[e]) + task["row_begin"] + task["rows"]
        c0, c1 = c0 + half * (task["bn"] // 2), min(c0 + (half + 1) * (task["bn"] // 2), pl["N"])
        tail = task["rows"] - (R - 1) * task["bm"]
        return dict(h=h, task=j, expert=e, l=l, rt=rt, ct=ct, rows=(r0, r1), cols=(c0, c1), kind=KIND_RIDE,
                    half=half, height=-(-tail // 16) * 16)
    return dict(h=h, task=j, expert=e, l=l, rt=rt, ct=ct, rows=(r0, r1), cols=(c0, c1), kind=kind,
                height=-(-(r1 - r0) // 16) * 16 if kind == 1 else task["bm"])


def tile_cover(pl: dict, row_off, n_rows: int) -> np.ndarray:
    """Write-count shadow buffer: how many tiles cover each Y element."""
    cover = np.zeros((n_rows, pl["N"]), dtype=np.int64)
    for B in range(pl["total"]):
        d = decode(pl, row_off, B)
        cover[d["rows"][0]:d["rows"][1], d["cols"][0]:d["cols"][1]] += 1
    return cover


# ---------------------------------------------------------------------------
# c4 — the expert GEMM, unbatched, fp64
# ---------------------------------------------------------------------------
def expert_gemm(X: np.ndarray, W: np.ndarray, token_idx, row_off) -> np.ndarray:
    """Y[row_off[e]+r, :] = X[token_idx[row_off[e]+r], :] @ W[e] for e = 0..E-1."""
    E = W.shape[0]
    Y = np.zeros((int(row_off[E]), W.shape[2]), dtype=np.float64)
    for e in range(E):
        a, b = int(row_off[e]), int(row_off[e + 1])
        if b > a:
            Y[a:b] = X[np.asarray(token_idx[a:b], dtype=np.int64)].astype(np.float64) @ W[e].astype(np.float64)
    return Y


def expert_gemm_entries(x_row, w_cols, token_idx, row_off, rows, cols) -> np.ndarray:
    """Sampled entries of the same product: out[i, c] = sum_h X[t_i, h] * W[e_i, h, cols[c]]
    for CSR rows ``rows`` (t_i = token_idx[row], e_i = the expert owning that row).

    ``x_row(t) -> [H]`` and ``w_cols(e, cols) -> [H, len(cols)]`` fetch inputs on
    demand so full-size parity never materialises W on the host."""
    E = len(row_off) - 1
    out = np.zeros((len(rows), len(cols)))
    for i, r in enumerate(rows):
        e = 0
        while not (row_off[e] <= r < row_off[e + 1]):
            e += 1
            if e >= E:
                raise ValueError("row outside the CSR")
        t = int(token_idx[r])
        out[i] = np.asarray(x_row(t), dtype=np.float64) @ np.asarray(w_cols(e, cols), dtype=np.float64)
    return out


# ---------------------------------------------------------------------------
# combine order and expert parallelism
# ---------------------------------------------------------------------------
def per_slot_outputs(topk_ids, X, W) -> np.ndarray:
    """Definition used by EP checks: out[t*k + j] = X[t] @ W[topk[t, j]]."""
    T, k = topk_ids.shape
    out = np.zeros((T * k, W.shape[2]))
    for t in range(T):
        for j in range(k):
            out[t * k + j] = X[t].astype(np.float64) @ W[int(topk_ids[t, j])].astype(np.float64)
    return out


def ep_simulate(topk_ids: np.ndarray, X: np.ndarray, W: np.ndarray, G: int) -> dict:
    """In-process expert-parallel simulation.

    Rank g owns experts [g*E/G, (g+1)*E/G) and tokens [g*T/G, (g+1)*T/G).
    Dispatch sends each owned token once to every rank hosting >= 1 of its
    experts (dedup per destination); the receiving rank buckets the received rows
    per local expert (ascending global token id), multiplies, and returns each
    (t, slot) row to the token's owner, which places it at t_local*k + slot."""
    T, k = topk_ids.shape
    E = W.shape[0]
    if E % G or T % G:
        raise ValueError("E and T must be divisible by G")
    El, Tl = E // G, T // G
    owner_of_expert = [e // El for e in range(E)]
    sent_rows = np.zeros((G, G), dtype=np.int64)       # [src, dst]
    recv: list[list[int]] = [[] for _ in range(G)]     # global token ids received by rank d
    for g in range(G):
        for d in range(G):
            for t in range(g * Tl, (g + 1) * Tl):
                if any(owner_of_expert[int(e)] == d for e in topk_ids[t]):
                    recv[d].append(t)
                    sent_rows[g, d] += 1
    out = [np.zeros((Tl * k, W.shape[2])) for _ in range(G)]
    local_counts = np.zeros((G, El), dtype=np.int64)
    for d in range(G):
        rows = recv[d]                                  # ascending global token ids
        for el in range(El):
            e = d * El + el
            members = [(i, t) for i, t in enumerate(rows) if e in set(int(x) for x in topk_ids[t])]
            local_counts[d, el] = len(members)
            for (i, t) in members:
                y = X[t].astype(np.float64) @ W[e].astype(np.float64)
                j = [int(x) for x in topk_ids[t]].index(e)
                g = t // Tl
                out[g][(t - g * Tl) * k + j] = y
    return dict(out=out, sent_rows=sent_rows, local_counts=local_counts, recv=recv)
