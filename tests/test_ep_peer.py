"""The library's expert-parallel step over symmetric peer memory (moe_ep_peer_*, include/moe_sm100_ep.h;
DESIGN.md §9): dispatch rows stored into the owners' receive buffers, the GEMM epilogue storing result rows
into the token owners' outputs, device-side epoch flags instead of host synchronisation.

Covered: G virtual ranks of one process driven by ONE host thread (a step never blocks the host), bf16 and
FP8, several steps with different routings (buffer reuse across steps), masked slots and repeated ids,
zero-copy output; and G separate PROCESSES on one GPU mapping each other's regions through CUDA IPC, with
the blobs all-gathered over gloo (the exact code path of one process per GPU).  Reference: the P:90
per-(token, slot) definition in the oracle (integer inputs: bit-exact)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import synth
from oracle import moe as omoe

HERE = os.path.dirname(os.path.abspath(__file__))


def _valid_ref(ids, X, W):
    T, k = ids.shape
    first = np.array([[ids[t, j] not in ids[t, :j] for j in range(k)] for t in range(T)], dtype=bool).reshape(T, k)
    valid = ((ids >= 0) & first).reshape(-1)
    ref = np.zeros((T * k, W.shape[2]))
    for t in range(T):
        for j in range(k):
            if ids[t, j] >= 0 and first[t, j]:
                ref[t * k + j] = X[t] @ W[ids[t, j]]
    return valid, ref


def _routing(step, T, E, k, masked):
    ids = synth.route_gumbel(100 + step, T, E, k, s=1.2 if step % 2 else 0.0, n_empty=2 if step % 2 else 0)
    if masked:
        rng = np.random.default_rng(step)
        ids = np.where(rng.random((T, k)) < 0.15, -1, ids).astype(np.int32)
        rep = np.nonzero(rng.random(T) < 0.1)[0]
        ids[rep, k - 1] = ids[rep, 0]
    return np.ascontiguousarray(ids.astype(np.int32))


@pytest.mark.gpu
@pytest.mark.parametrize("G,fp8", [(1, False), (2, False), (4, False), (8, False), (2, True), (4, True)])
def test_ep_peer_virtual_ranks(G, fp8):
    """G ranks of this process, one host thread, one stream per rank, three steps with different
    routings (uniform / skewed with empty experts / masked slots + repeated ids): every computed slot
    equals the P:90 definition bit for bit, masked and repeated slots keep the caller's sentinel."""
    import paper_2501_16103_b200 as M
    from oracle import fp8 as ofp8
    from synth import fp8 as sfp8
    E, k, T_l, H, N = 8, 3, 48, 128, 256
    T = G * T_l
    El = E // G
    if fp8:
        X = sfp8.make_x_fp8(G, T, H, "int")
        W = sfp8.make_w_fp8(G, E, H, N, "int")
        scale = np.array([2.0 ** (i % 3 - 1) for i in range(E)], dtype=np.float32)
        Xv, Wv = ofp8.e4m3_decode(X), ofp8.e4m3_decode(W) * scale[:, None, None]
        Ws = [torch.from_numpy(W[r * El:(r + 1) * El]).cuda() for r in range(G)]
        Xs = [torch.from_numpy(X[r * T_l:(r + 1) * T_l]).cuda() for r in range(G)]
        scs = [torch.from_numpy(scale[r * El:(r + 1) * El]).cuda() for r in range(G)]
    else:
        X, W = synth.make_x(G, T, H, "int"), synth.make_w(G, E, H, N, "int")
        Xv, Wv = X, W
        Ws = [torch.from_numpy(W[r * El:(r + 1) * El]).to(torch.bfloat16).cuda() for r in range(G)]
        Xs = [torch.from_numpy(X[r * T_l:(r + 1) * T_l]).to(torch.bfloat16).cuda() for r in range(G)]
        scs = None
    eps = M.PeerExpertParallel.group(G, E, Ws, max_tokens=T_l, k=k, w_scales=scs)
    for ep in eps:
        ep.set_timeout(20.0)
    streams = [torch.cuda.Stream() for _ in range(G)]
    for step in range(3):
        ids = _routing(step, T, E, k, masked=step == 2)
        tks = [torch.from_numpy(ids[r * T_l:(r + 1) * T_l]).cuda() for r in range(G)]
        outs = [torch.full((T_l * k, N), float("nan"), dtype=torch.float32, device="cuda") for _ in range(G)]
        torch.cuda.synchronize()
        for r in range(G):                           # one thread enqueues every rank's whole step
            with torch.cuda.stream(streams[r]):
                eps[r].forward(tks[r], Xs[r], out=outs[r])
        for s in streams:
            s.synchronize()
        assert [ep.status() for ep in eps] == [0] * G
        got = torch.cat([o.cpu() for o in outs]).double().numpy()
        valid, ref = _valid_ref(ids, Xv, Wv)
        assert np.array_equal(got[valid], ref[valid]), f"step {step}"
        assert np.isnan(got[~valid]).all()
        rows = [ep.last_rows() for ep in eps]
        assert sum(r["sent"] for r in rows) == sum(r["received"] for r in rows)
        assert sum(r["local_rows"] for r in rows) == int(valid.sum())


@pytest.mark.gpu
def test_ep_peer_zero_copy_and_bf16_out():
    """out = the handle's own output (moe_ep_peer_output): no copy; bf16 result rows; G = 4."""
    import paper_2501_16103_b200 as M
    G, E, k, T_l, H, N = 4, 8, 2, 64, 64, 512
    T = G * T_l
    El = E // G
    X, W = synth.make_x(7, T, H, "int"), synth.make_w(7, E, H, N, "int")
    ids = _routing(0, T, E, k, masked=False)
    Ws = [torch.from_numpy(W[r * El:(r + 1) * El]).to(torch.bfloat16).cuda() for r in range(G)]
    Xs = [torch.from_numpy(X[r * T_l:(r + 1) * T_l]).to(torch.bfloat16).cuda() for r in range(G)]
    tks = [torch.from_numpy(ids[r * T_l:(r + 1) * T_l]).cuda() for r in range(G)]
    eps = M.PeerExpertParallel.group(G, E, Ws, max_tokens=T_l, k=k, max_out_bytes=N * 2)
    outs = [ep.output(T_l, N) for ep in eps]
    streams = [torch.cuda.Stream() for _ in range(G)]     # one stream per rank: a rank's step waits for its peers'
    torch.cuda.synchronize()
    for r in range(G):
        with torch.cuda.stream(streams[r]):
            eps[r].forward(tks[r], Xs[r], out=outs[r])
    torch.cuda.synchronize()
    assert [ep.status() for ep in eps] == [0] * G
    got = torch.cat([o.float().cpu() for o in outs]).double().numpy()
    ref = omoe.per_slot_outputs(ids, X, W)
    assert np.array_equal(got, torch.from_numpy(ref).float().to(torch.bfloat16).double().numpy())


@pytest.mark.gpu
def test_ep_peer_capacity_and_connect_errors():
    import paper_2501_16103_b200 as M
    E, k, H, N = 4, 2, 64, 256
    W = torch.zeros((E // 2, H, N), dtype=torch.bfloat16, device="cuda")
    a = M.PeerExpertParallel(0, 2, E, W, max_tokens=8, k=k, connect=False)
    b = M.PeerExpertParallel(1, 2, E, W, max_tokens=8, k=k, connect=False)
    with pytest.raises(M.MoeError):                  # wrong rank order
        a.connect([b.blob, a.blob])
    c = M.PeerExpertParallel(1, 2, E, W, max_tokens=16, k=k, connect=False)
    with pytest.raises(M.MoeError):                  # capacities differ
        a.connect([a.blob, c.blob])
    with pytest.raises(M.MoeError):                  # not connected yet
        a.forward(torch.zeros((4, k), dtype=torch.int32, device="cuda"), torch.zeros((4, H), dtype=torch.bfloat16,
                                                                                      device="cuda"))
    a.connect([a.blob, b.blob])
    with pytest.raises(M.MoeError):                  # T > max_tokens
        a.forward(torch.zeros((9, k), dtype=torch.int32, device="cuda"), torch.zeros((9, H), dtype=torch.bfloat16,
                                                                                      device="cuda"))


@pytest.mark.gpu
def test_ep_peer_timeout_does_not_hang():
    """A rank whose peer never runs its step: the device-side wait gives up (status 2) instead of hanging."""
    import paper_2501_16103_b200 as M
    E, k, T_l, H, N = 4, 2, 8, 64, 256
    W = torch.zeros((E // 2, H, N), dtype=torch.bfloat16, device="cuda")
    eps = M.PeerExpertParallel.group(2, E, [W, W], max_tokens=T_l, k=k)
    eps[0].set_timeout(0.2)
    eps[0].forward(torch.zeros((T_l, k), dtype=torch.int32, device="cuda"),
                   torch.zeros((T_l, H), dtype=torch.bfloat16, device="cuda"))
    assert eps[0].status() == 2


def _proc_worker(rank, world, port, q, fp8):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    import paper_2501_16103_b200 as M
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        E, k, T_l, H, N = 8, 2, 40, 128, 256
        T, El = world * T_l, E // world
        if fp8:
            from oracle import fp8 as ofp8
            from synth import fp8 as sfp8
            X, W = sfp8.make_x_fp8(world, T, H, "int"), sfp8.make_w_fp8(world, E, H, N, "int")
            scale = np.ones(E, dtype=np.float32)
            Xv, Wv = ofp8.e4m3_decode(X), ofp8.e4m3_decode(W)
            Wl = torch.from_numpy(W[rank * El:(rank + 1) * El]).cuda()
            Xl = torch.from_numpy(X[rank * T_l:(rank + 1) * T_l]).cuda()
            sc = torch.from_numpy(scale[rank * El:(rank + 1) * El]).cuda()
        else:
            X, W = synth.make_x(world, T, H, "int"), synth.make_w(world, E, H, N, "int")
            Xv, Wv = X, W
            Wl = torch.from_numpy(W[rank * El:(rank + 1) * El]).to(torch.bfloat16).cuda()
            Xl = torch.from_numpy(X[rank * T_l:(rank + 1) * T_l]).to(torch.bfloat16).cuda()
            sc = None

        def allgather(blob):
            got = [None] * world
            dist.all_gather_object(got, blob)
            return got

        ep = M.PeerExpertParallel(rank, world, E, Wl, max_tokens=T_l, k=k, allgather=allgather, w_scale=sc)
        ep.set_timeout(30.0)
        ok = []
        for step in range(3):
            ids = _routing(step, T, E, k, masked=step == 2)
            out = torch.full((T_l * k, N), float("nan"), dtype=torch.float32, device="cuda")
            ep.forward(torch.from_numpy(ids[rank * T_l:(rank + 1) * T_l]).cuda(), Xl, out=out)
            torch.cuda.synchronize()
            valid, ref = _valid_ref(ids, Xv, Wv)
            sl = slice(rank * T_l * k, (rank + 1) * T_l * k)
            got = out.cpu().double().numpy()
            ok.append(bool(np.array_equal(got[valid[sl]], ref[sl][valid[sl]]) and np.isnan(got[~valid[sl]]).all()
                           and ep.status() == 0))
        dist.barrier()                                # every rank done before any region is released
        del ep
        q.put((rank, ok))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,fp8", [(2, False), (4, False), (2, True), (8, False)])
def test_ep_peer_multiprocess_one_gpu(world, fp8):
    """`world` processes (one rank each, as under torchrun) on one GPU: CUDA IPC mappings of each
    other's regions, blobs all-gathered over gloo, three steps each, bit-exact per rank."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_proc_worker, args=(r, world, port, q, fp8)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(world):
            r, v = q.get(timeout=300)
            res[r] = v
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():  # pragma: no cover
                p.kill()
    assert res == {r: [True, True, True] for r in range(world)}, res


@pytest.mark.gpu
@pytest.mark.parametrize("T,E,G,k", [(5000, 16, 4, 3), (1025, 8, 2, 2), (4096, 8, 1, 2), (3000, 64, 8, 6)])
def test_dispatch_plan_chunked_matches_definition(T, E, G, k):
    """moe_ep_dispatch_plan over chunks x G blocks (T > 1024): per destination d the tokens with a slot
    owned by d in ascending order, their d-local ids (-1: another rank's slot or a repeated id), the row /
    slot totals and offsets — written out here from the definition (R8)."""
    import paper_2501_16103_b200 as M
    rng = np.random.default_rng(T)
    ids = synth.route_gumbel(T, T, E, k, s=1.0, n_empty=1)
    ids = np.where(rng.random((T, k)) < 0.1, -1, ids).astype(np.int32)
    rep = np.nonzero(rng.random(T) < 0.05)[0]
    ids[rep, k - 1] = ids[rep, 0]
    counts2, send_off, send_tok, send_meta = M.moe_ep_dispatch_plan(torch.from_numpy(ids).cuda(), E, G)
    torch.cuda.synchronize()
    El = E // G
    off = 0
    for d in range(G):
        toks, metas, slots = [], [], 0
        for t in range(T):
            row = ids[t].tolist()
            meta = [row[j] - d * El if row[j] >= 0 and row[j] // El == d and row[j] not in row[:j] else -1
                    for j in range(k)]
            if any(r >= 0 and r // El == d for r in row):
                toks.append(t)
                metas.append(meta)
            slots += sum(m >= 0 for m in meta)
        assert counts2[d].tolist() == [len(toks), slots]
        assert int(send_off[d]) == off
        assert send_tok[off:off + len(toks)].tolist() == toks
        assert send_meta[off:off + len(toks)].tolist() == metas
        off += len(toks)
    assert int(send_off[G]) == off
