"""fp64 CPU oracle for the statically batched MoE expert GEMM (arXiv 2501.16103).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import, call or
execute anything in this package.  The product path
(``paper_2501_16103_b200``) never imports it and has no CPU fallback.

Plain, slow, obviously-correct code written from the paper (``P:n`` = line n of
PAPER.md).  It shares no code with the CUDA path; the only common dependency is
the seeded input generator in ``synth/`` (which holds no method arithmetic).

Modules
-------
``mapping``  Alg. 1 (TilePrefix), Alg. 2 (warp vote / popcount mapping, with the
             padding rule P:203 and the chunk loop P:204-205), Alg. 4 (sigma,
             the non-empty-task stage P:262-296).  Pinned by tests against the
             SPEC worked examples and a brute-force enumeration.
``moe``      token-index buckets, the MoE plan (experts as tasks,
             P:298-301), tile decode (task, tile) -> rows/cols, the unbatched
             per-expert GEMM in fp64, tile-cover
             bookkeeping and an expert-parallel simulator.
``ffn``      the full MoE FFN layer around the expert GEMM:
             SwiGLU expert FFN (R14) and the weighted combine.
``fp8``      the OCP E4M3 decode written out and the expert GEMM on decoded FP8
             values with a per-expert scale (R15).

Parity-pin status of every function is listed in DESIGN.md §"Oracle pins";
no function here is "parity unpinned".
"""
from . import ffn, fp8, mapping, moe  # noqa: F401
