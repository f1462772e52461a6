"""Seeded input generators (routing, X, W) — no method arithmetic lives here.

Recipes (stated again in DESIGN.md §"Input recipe"):

* Routing (top-k expert ids per token, int32 [T, k]) is drawn on the host:
  - ``route_gumbel``: SURVEY §8(d) "Exact routing recipe" — numpy
    ``default_rng(seed)``; ``perm = rng.permutation(E)``; weights
    ``w[perm[:E-n_empty]] = arange(1, E-n_empty+1) ** -s`` (uniform: s=0,
    n_empty=0); Gumbel-top-k over ``log w`` with a stable argsort.  Experts with
    w=0 get log w = -inf and are never drawn, so ``n_empty`` experts are forced
    empty (the "many empty experts" DeepSeek case, "no token is routed to
    an expert").
  - ``route_balanced``: token t -> experts {(k*t + j) mod E} — "tokens are
    averagely routed to all experts".
  - ``route_paper_best`` / ``route_paper_worst``: the §5 best / worst cases
    (P:374-375).
  - ``route_tiny_a``: deterministic tiny case with one empty expert.
* X [T, H] and W [E, H, N] come from a counter-based generator so that the
  host (numpy, for the oracle) and the device (torch, for the CUDA path) produce
  bit-identical values without either side materialising the other's copy:
  ``h = fmix32(index ^ key(seed, stream))``; four 7-bit fields of h are summed
  (Irwin-Hall, approximately normal) and centred: ``c = sum - 254`` in
  [-254, 254].  ``c`` has at most 8 significant bits, so ``c * 2**-e`` is EXACT
  in bf16: no rounding step exists on either side.
  - "normal" mode: X = c * 2**-6 (std ~1.15); W = c * 2**-(6 + w_scale_exp(H))
    with ``w_scale_exp(H) = floor(log2(H)/2 + 1/2)`` (W ~ N(0,1)/sqrt(H)).
  - "int" mode: values (h mod 9) - 4 in {-4..4} (exact in bf16).
  - "generic" mode: a full bf16 bit pattern built with integer operations — sign = bit 31
    of h, a random 7-bit mantissa (bits 0-6), exponent offset ((h >> 8) & 15) - 8 (16 octaves) —
    value = (-1)^s (1 + m/128) 2^(e_off + 2 - shift).  Unlike "normal", its products carry 16
    significant bits over ~30 octaves, so fp32 accumulation must round (the regime the north
    star's tolerance is for; tests/test_synth.py proves it with exact int64 sums).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

_M32 = 0xFFFFFFFF
STREAM_X = 1
STREAM_W = 2


# ----------------------------------------------------------------------------
# Named configurations (BASELINE.json "configs")
# ----------------------------------------------------------------------------
@dataclass(frozen=True)
class Config:
    name: str
    E: int
    k: int
    T: int
    H: int
    N: int
    routing: str = "uniform"       # uniform | zipf | balanced | tiny_a | best | worst
    zipf_s: float = 0.0
    n_empty: int = 0
    notes: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def flops(self) -> int:
        """Useful flops 2*sum(m_e)*H*N = 2*T*k*H*N (SURVEY §8(c) c4 FLOP convention)."""
        return 2 * self.T * self.k * self.H * self.N


CONFIGS: dict[str, Config] = {
    "tiny": Config("tiny", E=4, k=2, T=16, H=64, N=128, routing="tiny_a",
                   notes="BASELINE configs[0]; expert 1 receives zero tokens"),
    "tiny_b": Config("tiny_b", E=4, k=2, T=16, H=64, N=128, routing="zipf", zipf_s=0.0, n_empty=1,
                     notes="seeded variant of tiny: Gumbel top-2 over 3 of 4 experts"),
    "mix": Config("mix", E=8, k=2, T=4096, H=4096, N=14336, routing="uniform",
                  notes="BASELINE configs[1]: Mixtral-8x7B FFN shape, uniform routing"),
    "mix_balanced": Config("mix_balanced", E=8, k=2, T=4096, H=4096, N=14336, routing="balanced"),
    "ds": Config("ds", E=64, k=6, T=8192, H=2048, N=1408, routing="zipf", zipf_s=1.2, n_empty=16,
                 notes="BASELINE configs[2]: DeepSeek-V2-Lite shape, Zipf s=1.2, 16 forced-empty experts"),
    "ep": Config("ep", E=8, k=2, T=32768, H=6144, N=16384, routing="uniform",
                 notes="BASELINE configs[4]: Mixtral-8x22B shape (expert-parallel at G>1)"),
    "paper_balanced": Config("paper_balanced", E=64, k=8, T=4096, H=3584, N=2560, routing="balanced",
                             notes="paper §5 balanced case (P:368-373)"),
    "paper_best": Config("paper_best", E=64, k=8, T=4096, H=3584, N=2560, routing="best",
                         notes="paper §5 best case (P:374)"),
    "paper_worst": Config("paper_worst", E=64, k=8, T=4096, H=3584, N=2560, routing="worst",
                          notes="paper §5 worst case (P:375)"),
}
CONFIGS["paper_light8"] = Config("paper_light8", E=64, k=1, T=8, H=3584, N=2560, routing="light",
                                 notes="probe: 8 experts of the paper §5 shape with one token each (memory-bound tiles)")
for _T in (1, 2, 4, 8, 16, 32, 64, 128, 256):
    CONFIGS[f"dec{_T}"] = Config(f"dec{_T}", E=8, k=2, T=_T, H=4096, N=14336, routing="uniform",
                                 notes="BASELINE configs[3]: decode regime, Mixtral shape")


# ----------------------------------------------------------------------------
# Routing
# ----------------------------------------------------------------------------
def route_gumbel(seed: int, T: int, E: int, k: int, s: float = 0.0, n_empty: int = 0) -> np.ndarray:
    """SURVEY §8(d) exact routing recipe (Gumbel-top-k without replacement)."""
    if not (0 <= n_empty <= E - k):
        raise ValueError("need at least k non-empty experts")
    rng = np.random.default_rng(seed)
    perm = rng.permutation(E)
    w = np.zeros(E)
    w[perm[: E - n_empty]] = np.arange(1, E - n_empty + 1, dtype=np.float64) ** (-s)
    with np.errstate(divide="ignore"):
        g = rng.gumbel(size=(T, E)) + np.log(w)
    ids = np.argsort(-g, axis=1, kind="stable")[:, :k]
    return np.ascontiguousarray(ids.astype(np.int32))


def route_balanced(T: int, E: int, k: int) -> np.ndarray:
    """Token t -> experts {(k*t + j) mod E : j < k} ("averagely routed")."""
    if k > E:
        raise ValueError("k > E")
    t = np.arange(T, dtype=np.int64)[:, None]
    j = np.arange(k, dtype=np.int64)[None, :]
    return np.ascontiguousarray(((k * t + j) % E).astype(np.int32))


def route_tiny_a(T: int = 16) -> np.ndarray:
    """tiny-A: token t -> virtual experts {t mod 3, (t+1) mod 3}, ids {0->0, 1->2, 2->3}.

    Expert 1 receives zero tokens (the empty-task case)."""
    idmap = np.array([0, 2, 3], dtype=np.int32)
    t = np.arange(T)
    return np.ascontiguousarray(np.stack([idmap[t % 3], idmap[(t + 1) % 3]], axis=1).astype(np.int32))


def route_paper_best(T: int = 4096, E: int = 64, k: int = 8) -> np.ndarray:
    """P:374 best case: all tokens routed to the same k experts (ids 0..k-1)."""
    return np.ascontiguousarray(np.tile(np.arange(k, dtype=np.int32), (T, 1)))


def route_paper_worst(T: int = 4096, E: int = 64, k: int = 8) -> np.ndarray:
    """P:375 worst case: the E-k other experts each receive exactly one token.

    Token t < E-k routes to experts {0..k-2} and to expert k+t; every other token
    routes to the k busy experts {0..k-1}."""
    ids = np.tile(np.arange(k, dtype=np.int32), (T, 1))
    n_light = E - k
    if T < n_light:
        raise ValueError("T too small for the worst case")
    ids[:n_light, k - 1] = k + np.arange(n_light, dtype=np.int32)
    return np.ascontiguousarray(ids)


def route(cfg: Config, seed: int = 0) -> np.ndarray:
    if cfg.routing == "uniform":
        return route_gumbel(seed, cfg.T, cfg.E, cfg.k)
    if cfg.routing == "zipf":
        return route_gumbel(seed, cfg.T, cfg.E, cfg.k, s=cfg.zipf_s, n_empty=cfg.n_empty)
    if cfg.routing == "balanced":
        return route_balanced(cfg.T, cfg.E, cfg.k)
    if cfg.routing == "tiny_a":
        return route_tiny_a(cfg.T)
    if cfg.routing == "best":
        return route_paper_best(cfg.T, cfg.E, cfg.k)
    if cfg.routing == "worst":
        return route_paper_worst(cfg.T, cfg.E, cfg.k)
    if cfg.routing == "light":                     # token t -> expert t (one token per expert)
        return np.ascontiguousarray(np.arange(cfg.T, dtype=np.int32)[:, None] % cfg.E)
    raise ValueError(cfg.routing)


# ----------------------------------------------------------------------------
# Counter-based value generator (numpy and torch twins, bit-identical)
# ----------------------------------------------------------------------------
def _fmix32_np(h: np.ndarray) -> np.ndarray:
    h = h.astype(np.uint32, copy=True)
    h ^= h >> np.uint32(16)
    h *= np.uint32(0x85EBCA6B)
    h ^= h >> np.uint32(13)
    h *= np.uint32(0xC2B2AE35)
    h ^= h >> np.uint32(16)
    return h


def _key(seed: int, stream: int) -> int:
    k = (seed * 0x9E3779B9 + stream * 0x7F4A7C15 + 0x632BE5AB) & _M32
    return int(_fmix32_np(np.array([k], dtype=np.uint32))[0])


def w_scale_exp(H: int) -> int:
    """Exponent e with 2**-e ~ 1/sqrt(H)."""
    return int(math.floor(math.log2(H) / 2.0 + 0.5))


def counter_values(seed: int, stream: int, index: np.ndarray, mode: str, shift: int) -> np.ndarray:
    """float64 values of elements at flat positions ``index`` (exact bf16 values)."""
    idx = np.asarray(index, dtype=np.int64)
    if idx.size and (idx.min() < 0 or idx.max() > _M32):
        raise ValueError("index out of 32-bit range")
    h = _fmix32_np((idx.astype(np.uint64) ^ np.uint64(_key(seed, stream))).astype(np.uint32))
    if mode == "int":
        return (h % np.uint32(9)).astype(np.float64) - 4.0
    if mode == "normal":
        c = ((h & np.uint32(127)) + ((h >> np.uint32(8)) & np.uint32(127))
             + ((h >> np.uint32(16)) & np.uint32(127)) + ((h >> np.uint32(24)) & np.uint32(127)))
        return (c.astype(np.float64) - 254.0) * 2.0 ** (-shift)
    if mode == "generic":
        bits = generic_bits_np(h, shift)
        return ((bits.astype(np.uint32) << np.uint32(16)).view(np.float32)).astype(np.float64)
    raise ValueError(mode)


def generic_bits_np(h: np.ndarray, shift: int) -> np.ndarray:
    """bf16 bit patterns of "generic" mode (uint16): sign | biased exponent | 7-bit mantissa."""
    h = np.asarray(h, dtype=np.uint32)
    sign = (h >> np.uint32(31)) & np.uint32(1)
    mant = h & np.uint32(127)
    bexp = ((h >> np.uint32(8)) & np.uint32(15)).astype(np.int64) - 8 + 2 - shift + 127
    if bexp.size and (bexp.min() < 1 or bexp.max() > 254):
        raise ValueError("generic exponent outside the bf16 normal range")
    return ((sign << np.uint32(15)) | (bexp.astype(np.uint32) << np.uint32(7)) | mant).astype(np.uint16)


def _shift_x() -> int:
    return 6


def _shift_w(H: int) -> int:
    return 6 + w_scale_exp(H)


def make_x(seed: int, T: int, H: int, mode: str = "normal") -> np.ndarray:
    """X [T, H] as float64 (every value exactly representable in bf16)."""
    return counter_values(seed, STREAM_X, np.arange(T * H, dtype=np.int64), mode, _shift_x()).reshape(T, H)


def make_w(seed: int, E: int, H: int, N: int, mode: str = "normal", experts=None) -> np.ndarray:
    """W [E, H, N] as float64; ``experts`` selects a subset of expert ids (same values)."""
    if mode == "identity":
        if H != N:
            raise ValueError("identity mode needs H == N")
        ids = range(E) if experts is None else experts
        return np.stack([(e + 1) * np.eye(H) for e in ids])
    ids = list(range(E)) if experts is None else list(experts)
    out = np.empty((len(ids), H, N))
    for i, e in enumerate(ids):
        base = e * H * N
        out[i] = counter_values(seed, STREAM_W, base + np.arange(H * N, dtype=np.int64), mode,
                                _shift_w(H)).reshape(H, N)
    return out


def w_columns(seed: int, E: int, H: int, N: int, e: int, cols: np.ndarray, mode: str = "normal") -> np.ndarray:
    """W[e][:, cols] as float64 [H, len(cols)] without materialising W."""
    cols = np.asarray(cols, dtype=np.int64)
    if mode == "identity":
        return (e + 1) * np.eye(H)[:, cols]
    idx = e * H * N + np.arange(H, dtype=np.int64)[:, None] * N + cols[None, :]
    return counter_values(seed, STREAM_W, idx, mode, _shift_w(H))


def x_rows(seed: int, T: int, H: int, rows: np.ndarray, mode: str = "normal") -> np.ndarray:
    rows = np.asarray(rows, dtype=np.int64)
    idx = rows[:, None] * H + np.arange(H, dtype=np.int64)[None, :]
    return counter_values(seed, STREAM_X, idx, mode, _shift_x())


# --- torch twin (device-side generation; same integer recipe) ----------------
def counter_values_torch(seed: int, stream: int, start: int, count: int, mode: str, shift: int,
                         device="cpu", dtype=None):
    import torch

    dtype = dtype or torch.bfloat16
    key = _key(seed, stream)
    idx = torch.arange(start, start + count, dtype=torch.int64, device=device)
    h = idx ^ key
    h = h & _M32
    h = h ^ (h >> 16)
    h = (h * 0x85EBCA6B) & _M32
    h = h ^ (h >> 13)
    h = (h * 0xC2B2AE35) & _M32
    h = h ^ (h >> 16)
    if mode == "int":
        return ((h % 9) - 4).to(torch.float32).to(dtype)
    if mode == "normal":
        c = (h & 127) + ((h >> 8) & 127) + ((h >> 16) & 127) + ((h >> 24) & 127)
        return ((c - 254).to(torch.float32) * (2.0 ** (-shift))).to(dtype)
    if mode == "generic":                          # same integer recipe as generic_bits_np
        bexp = ((h >> 8) & 15) - 8 + 2 - shift + 127
        bits = (((h >> 31) & 1) << 15) | (bexp << 7) | (h & 127)
        bits = torch.where(bits >= 32768, bits - 65536, bits).to(torch.int16)
        return bits.view(torch.bfloat16).to(dtype)
    raise ValueError(mode)


def make_x_torch(seed: int, T: int, H: int, mode: str = "normal", device="cpu"):
    return counter_values_torch(seed, STREAM_X, 0, T * H, mode, _shift_x(), device).reshape(T, H)


def make_w_torch(seed: int, E: int, H: int, N: int, mode: str = "normal", device="cpu", chunk=1 << 26,
                 experts: range | None = None):
    """W [E, H, N] (or the contiguous expert range `experts` of it, e.g. one EP rank's share)."""
    import torch

    ex = range(E) if experts is None else experts
    if mode == "identity":
        if H != N:
            raise ValueError("identity mode needs H == N")
        eye = torch.eye(H, device=device, dtype=torch.float32)
        return torch.stack([(e + 1) * eye for e in ex]).to(torch.bfloat16)
    start, total = ex.start * H * N, len(ex) * H * N
    out = torch.empty(total, dtype=torch.bfloat16, device=device)
    for s in range(0, total, chunk):
        n = min(chunk, total - s)
        out[s:s + n] = counter_values_torch(seed, STREAM_W, start + s, n, mode, _shift_w(H), device)
    return out.reshape(len(ex), H, N)
