"""Expert-parallel path: exchange logic over gloo (CPU, world size 2, real torch.distributed),
G virtual ranks in one process, and the CUDA kernels on one GPU (virtual ranks and a
world-size-1 NCCL group).  Reference: the P:90 per-(token, slot) definition in the oracle."""
import os
import socket
import threading

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import synth
from oracle import moe as omoe
from paper_2501_16103_b200.ep import ExpertParallelMoE, ThreadComm, TorchComm

HERE = os.path.dirname(os.path.abspath(__file__))


def _problem(G, E=8, k=2, T_l=12, H=16, N=24, seed=0):
    T = G * T_l
    ids = synth.route_gumbel(seed, T, E, k)
    X = synth.make_x(seed, T, H, "int")
    W = synth.make_w(seed, E, H, N, "int")
    return ids, X, W, omoe.per_slot_outputs(ids, X, W)


def _cpu_kernels():
    import sys
    sys.path.insert(0, HERE)
    from ep_doubles import CpuKernels
    return CpuKernels()


def _gloo_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ids, X, W, ref = _problem(world)
        T_l, El = ids.shape[0] // world, W.shape[0] // world
        sl = slice(rank * T_l, (rank + 1) * T_l)
        moe = ExpertParallelMoE(W.shape[0], torch.from_numpy(W[rank * El:(rank + 1) * El]).float(), TorchComm(),
                                out_dtype=torch.float32, kernels=_cpu_kernels())
        out = moe.forward(torch.from_numpy(ids[sl]), torch.from_numpy(X[sl]).float())
        q.put((rank, bool(np.array_equal(out.double().numpy(), ref[rank * T_l * 2:(rank + 1) * T_l * 2])),
               moe.last))
    finally:
        dist.destroy_process_group()


def test_ep_exchange_gloo_world2():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    # conservation: rows sent by one rank are the rows received by the other
    last = {r: l for r, _, l in res}
    assert last[0]["send_rows"][1] == last[1]["recv_rows"][0]
    assert last[0]["ret_rows"] == [last[g]["back_rows"][0] for g in range(2)]


def _problem_fp8(G, E=8, k=2, T_l=12, H=16, N=24, seed=0):
    """FP8 E4M3 integer codes (synth/fp8.py), per-expert power-of-two scales; reference = the P:90
    per-(token, slot) definition on the decoded values (oracle/fp8.py), times the expert's scale."""
    from oracle import fp8 as ofp8
    from synth import fp8 as sfp8
    T = G * T_l
    ids = synth.route_gumbel(seed, T, E, k)
    X, W = sfp8.make_x_fp8(seed, T, H, "int"), sfp8.make_w_fp8(seed, E, H, N, "int")
    scale = (2.0 ** (np.arange(E) % 4 - 1)).astype(np.float32)
    ref = omoe.per_slot_outputs(ids, ofp8.e4m3_decode(X), ofp8.e4m3_decode(W)) * scale[ids.reshape(-1)][:, None]
    return ids, X, W, ref, scale


def _run_virtual(G, kernels_fn, device, out_dtype, E=8, k=2, T_l=12, H=16, N=24, seed=0, fp8=False):
    if fp8:
        ids, X, W, ref, scale = _problem_fp8(G, E, k, T_l, H, N, seed)
    else:
        ids, X, W, ref = _problem(G, E, k, T_l, H, N, seed)
    El = E // G
    comm = ThreadComm(G)
    outs, errs = [None] * G, []

    def body(r):
        try:
            comm.bind(r)
            Wl = torch.from_numpy(W[r * El:(r + 1) * El])
            Xl = torch.from_numpy(X[r * T_l:(r + 1) * T_l])
            sl = None
            if fp8:                                            # uint8 E4M3 codes travel as they are
                sl = torch.from_numpy(scale[r * El:(r + 1) * El]).to(device)
                Wl, Xl = Wl.to(device), Xl.to(device)
            elif device == "cuda":
                Wl, Xl = Wl.to(torch.bfloat16).cuda(), Xl.to(torch.bfloat16).cuda()
            else:
                Wl, Xl = Wl.float(), Xl.float()
            moe = ExpertParallelMoE(E, Wl, comm, out_dtype=out_dtype, kernels=kernels_fn(), w_scale=sl)
            outs[r] = moe.forward(torch.from_numpy(ids[r * T_l:(r + 1) * T_l]).to(device), Xl).cpu()
        except Exception as e:  # pragma: no cover
            errs.append(repr(e))
            comm._bar.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    got = torch.cat(outs).double().numpy()
    return got, ref


@pytest.mark.parametrize("G", [1, 2, 4])
def test_ep_exchange_virtual_ranks_cpu(G):
    got, ref = _run_virtual(G, _cpu_kernels, "cpu", torch.float32)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("G", [1, 2, 4])
def test_ep_exchange_virtual_ranks_cpu_fp8(G):
    """FP8 weights and token rows (E4M3 codes, per-expert scales) through the same exchange."""
    got, ref = _run_virtual(G, _cpu_kernels, "cpu", torch.float32, fp8=True)
    assert np.array_equal(got, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_ep_cuda_kernels_virtual_ranks_fp8(G):
    """moe_gemm_fp8_rowmap in the expert-parallel path: FP8 rows dispatched, results combined."""
    from paper_2501_16103_b200.ep import CudaKernels
    got, ref = _run_virtual(G, CudaKernels, "cuda", torch.float32, E=8, k=2, T_l=40, H=64, N=256, fp8=True)
    assert np.array_equal(got, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_ep_cuda_kernels_virtual_ranks(G):
    from paper_2501_16103_b200.ep import CudaKernels
    got, ref = _run_virtual(G, CudaKernels, "cuda", torch.float32, E=8, k=2, T_l=40, H=64, N=136)
    assert np.array_equal(got, ref)


@pytest.mark.gpu
def test_ep_cuda_skewed_and_large():
    """Zipf routing with empty experts: some ranks receive nothing for some experts."""
    from paper_2501_16103_b200.ep import CudaKernels
    got, ref = _run_virtual(4, CudaKernels, "cuda", torch.float32, E=16, k=4, T_l=300, H=128, N=256, seed=3)
    assert np.array_equal(got, ref)


@pytest.mark.gpu
def test_ep_nccl_world1():
    """The real NCCL collective path (a world of one rank on one GPU)."""
    import torch.distributed as dist
    from paper_2501_16103_b200.ep import CudaKernels
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        ids, X, W, ref = _problem(1, E=8, k=2, T_l=64, H=64, N=128)
        moe = ExpertParallelMoE(8, torch.from_numpy(W).to(torch.bfloat16).cuda(), TorchComm(),
                                out_dtype=torch.float32, kernels=CudaKernels())
        out = moe.forward(torch.from_numpy(ids).cuda(), torch.from_numpy(X).to(torch.bfloat16).cuda())
        assert np.array_equal(out.cpu().double().numpy(), ref)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("fused", ["1", "0"])
@pytest.mark.parametrize("fp8", [False, True])
@pytest.mark.parametrize("bm,bn", [(0, 0), (128, 256)])
def test_ep_native_nccl_world1(fp8, bm, bn, fused):
    """The library's own expert-parallel step (moe_ep_create / moe_ep_forward: NCCL called from C++,
    a one-rank communicator on one GPU; the combine fused into the GEMM epilogue, and with
    MOE_EP_UNFUSED the send buffer + exchange) against the P:90 definition."""
    import paper_2501_16103_b200 as M
    E, k, T, H, N = 8, 2, 300, 64, 256
    if fp8:
        ids, X, W, ref, scale = _problem_fp8(1, E, k, T, H, N, seed=4)
        Xd, Wd, sc = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda(), torch.from_numpy(scale).cuda()
    else:
        ids, X, W, ref = _problem(1, E, k, T, H, N, seed=4)
        Xd, Wd, sc = torch.from_numpy(X).to(torch.bfloat16).cuda(), torch.from_numpy(W).to(torch.bfloat16).cuda(), None
    ep = M.NativeExpertParallel(M.moe_ep_unique_id(), 0, 1, E, Wd, w_scale=sc, bm=bm, bn=bn, fused=fused == "1")
    topk = torch.from_numpy(ids).cuda()
    for _ in range(2):                                   # the plan and the communicator are reused
        out = ep.forward(topk, Xd, out_dtype=torch.float32)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().double().numpy(), ref)
    assert ep.last_rows() == {"sent": T, "received": T, "local_rows": T * k}
    assert ep.last_gemm_ms() > 0


@pytest.mark.gpu
@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("G,fp8", [(2, False), (4, False), (8, False), (4, True), (8, True)])
def test_ep_native_loopback_multirank(G, fp8, fused):
    """The library's multi-rank orchestration (moe_ep_forward) with G virtual ranks on one GPU: the
    test transport moves rows by device copies where NCCL would send them (moe_ep_create_loopback);
    one host thread and stream per rank; bit-exact vs the P:90 per-(token, slot) definition."""
    import paper_2501_16103_b200 as M
    E, k, T_l, H, N = 8, 2, 40, 64, 256
    if fp8:
        ids, X, W, ref, scale = _problem_fp8(G, E, k, T_l, H, N, seed=G)
    else:
        ids, X, W, ref = _problem(G, E, k, T_l, H, N, seed=G)
        scale = None
    El = E // G
    Ws, scs, Xs, tks = [], [], [], []
    for r in range(G):
        w = torch.from_numpy(W[r * El:(r + 1) * El])
        x = torch.from_numpy(X[r * T_l:(r + 1) * T_l])
        Ws.append(w.cuda() if fp8 else w.to(torch.bfloat16).cuda())
        Xs.append(x.cuda() if fp8 else x.to(torch.bfloat16).cuda())
        scs.append(torch.from_numpy(scale[r * El:(r + 1) * El]).cuda() if fp8 else None)
        tks.append(torch.from_numpy(np.ascontiguousarray(ids[r * T_l:(r + 1) * T_l])).cuda())
    torch.cuda.synchronize()
    eps = M.NativeExpertParallel.loopback_group(G, E, Ws, scs if fp8 else None, fused=fused)
    outs, errs = [None] * G, []

    def body(r):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(2):
                    outs[r] = eps[r].forward(tks[r], Xs[r], out_dtype=torch.float32)
            s.synchronize()
        except Exception as e:  # pragma: no cover
            errs.append(repr(e))

    th = [threading.Thread(target=body, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not errs, errs
    got = torch.cat([o.cpu() for o in outs]).double().numpy()
    assert np.array_equal(got, ref)
    rows = [ep.last_rows() for ep in eps]
    assert sum(r["sent"] for r in rows) == sum(r["received"] for r in rows)
    assert sum(r["local_rows"] for r in rows) == G * T_l * k


@pytest.mark.gpu
@pytest.mark.parametrize("repeat", [False, True])
@pytest.mark.parametrize("fused", [False, True])
def test_ep_native_loopback_masked_slots(fused, repeat):
    """Masked slots (negative ids) and skewed routing with empty experts through the library's
    multi-rank step (G = 4 virtual ranks): valid slots equal the P:90 definition, masked slots are
    not written (NaN sentinel kept).  repeat: some tokens list an expert twice (an invalid input,
    DESIGN.md R10) — only the first slot of that expert is computed, the repeat stays unwritten and
    nothing else is disturbed (repeated ids used to overrun the return metadata)."""
    import paper_2501_16103_b200 as M
    G, E, k, T_l, H, N = 4, 16, 4, 64, 64, 256
    T = G * T_l
    rng = np.random.default_rng(11)
    ids = synth.route_gumbel(11, T, E, k, s=1.2, n_empty=3)
    mask = rng.random((T, k)) < 0.15
    ids = np.where(mask, -1, ids).astype(np.int32)
    if repeat:
        rep = np.nonzero(rng.random(T) < 0.2)[0]
        ids[rep, 2] = ids[rep, 0]
        ids[rep[::2], 3] = ids[rep[::2], 1]
    X, W = synth.make_x(11, T, H, "int"), synth.make_w(11, E, H, N, "int")
    El = E // G
    Ws = [torch.from_numpy(W[r * El:(r + 1) * El]).to(torch.bfloat16).cuda() for r in range(G)]
    Xs = [torch.from_numpy(X[r * T_l:(r + 1) * T_l]).to(torch.bfloat16).cuda() for r in range(G)]
    tks = [torch.from_numpy(np.ascontiguousarray(ids[r * T_l:(r + 1) * T_l])).cuda() for r in range(G)]
    outs = [torch.full((T_l * k, N), float("nan"), dtype=torch.float32, device="cuda") for _ in range(G)]
    torch.cuda.synchronize()
    eps = M.NativeExpertParallel.loopback_group(G, E, Ws, fused=fused)
    errs = []

    def body(r):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                eps[r].forward(tks[r], Xs[r], out=outs[r])
            s.synchronize()
        except Exception as e:  # pragma: no cover
            errs.append(repr(e))

    th = [threading.Thread(target=body, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not errs, errs
    got = torch.cat([o.cpu() for o in outs]).double().numpy()
    first = np.array([[ids[t, j] not in ids[t, :j] for j in range(k)] for t in range(T)])
    valid = ((ids >= 0) & first).reshape(-1)
    ref = np.zeros((T * k, N))
    for t in range(T):
        for j in range(k):
            if ids[t, j] >= 0:
                ref[t * k + j] = X[t] @ W[ids[t, j]]
    assert np.array_equal(got[valid], ref[valid])
    assert np.isnan(got[~valid]).all()
    rows = [ep.last_rows() for ep in eps]
    assert sum(r["local_rows"] for r in rows) == int(valid.sum())


@pytest.mark.gpu
@pytest.mark.parametrize("fp8", [False, True])
def test_ep_native_full_size_sampled(fp8):
    """bench.py --ep's launch configuration: the Mixtral shape (T 4096, E 8, top-2, H 4096,
    N 14336) through the library's EP step (one NCCL rank, combine fused into the GEMM); sampled
    (token, slot) rows and columns against the fp64 oracle within the north-star tolerance."""
    import paper_2501_16103_b200 as M
    from oracle import fp8 as ofp8
    from synth import fp8 as sfp8
    from synth import workloads as wl
    c = synth.CONFIGS["mix"]
    ids = synth.route(c, 0)
    if fp8:
        Xd = sfp8.make_x_fp8_torch(0, c.T, c.H, device="cuda")
        Wd = sfp8.make_w_fp8_torch(0, c.E, c.H, c.N, device="cuda")
        scale = sfp8.w_scale(c.E, c.H)
        sc = torch.from_numpy(scale).cuda()
    else:
        Xd = synth.make_x_torch(0, c.T, c.H, device="cuda")
        Wd = synth.make_w_torch(0, c.E, c.H, c.N, device="cuda")
        sc = None
    ep = M.NativeExpertParallel(M.moe_ep_unique_id(), 0, 1, c.E, Wd, w_scale=sc)
    out = ep.forward(torch.from_numpy(ids).cuda(), Xd, out_dtype=torch.float32)
    torch.cuda.synchronize()
    rng = np.random.default_rng(3)
    toks = np.unique(np.concatenate([[0, c.T - 1], rng.integers(0, c.T, 10)]))
    cols = np.unique(np.concatenate([[0, c.N - 1, 255, 256], rng.integers(0, c.N, 20)]))
    got = out[torch.from_numpy(np.repeat(toks * c.k, c.k) + np.tile(np.arange(c.k), len(toks))).cuda()]
    got = got[:, torch.from_numpy(cols).cuda()].cpu().double().numpy()
    ref = np.zeros_like(got)
    for i, t in enumerate(toks):
        for j in range(c.k):
            e = int(ids[t, j])
            if fp8:
                ref[i * c.k + j] = ofp8.expert_gemm_fp8_entries(sfp8.x_fp8_rows(0, c.T, c.H, [t]),
                                                                sfp8.w_fp8_columns(0, c.E, c.H, c.N, e, cols), scale[e])[0]
            else:
                ref[i * c.k + j] = wl.x_rows(0, c.T, c.H, [t])[0] @ wl.w_columns(0, c.E, c.H, c.N, e, cols)
    d = np.abs(got - ref)
    assert (d <= 1e-2 * (np.abs(ref) + 1)).all(), d.max()
    assert np.linalg.norm(got - ref) <= 2e-3 * np.linalg.norm(ref)
