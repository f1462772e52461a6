"""GPU parity of the MoE FFN layer: moe_gemm_swiglu, moe_combine and the
MoeFFN layer against oracle/ffn.py (R14), through the C-ABI."""
import numpy as np
import pytest
import torch

import paper_2501_16103_b200 as M
import synth
from oracle import ffn as offn
from oracle import moe as omoe

pytestmark = pytest.mark.gpu


def tol_check(got, ref, what):
    """north_star tolerance: max |d| <= 1e-2 (|ref| + 1) and relative Frobenius <= 2e-3."""
    g = np.asarray(got, dtype=np.float64)
    r = np.asarray(ref, dtype=np.float64)
    d = np.abs(g - r)
    assert (d <= 1e-2 * (np.abs(r) + 1)).all(), f"{what}: max |d| {d.max()}"
    fro = np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-30)
    assert fro <= 2e-3, f"{what}: rel fro {fro}"


def _weights(seed, E, H, I, Ho):
    Wg = synth.make_w(seed, E, H, I)
    Wu = synth.make_w(seed + 1, E, H, I)
    Wd = synth.make_w(seed + 2, E, I, Ho)
    dev = [torch.from_numpy(w).to(torch.bfloat16).cuda() for w in (Wg, Wu, Wd)]
    return (Wg, Wu, Wd), dev


@pytest.mark.parametrize("T,E,k,H,I", [(300, 5, 2, 256, 512), (64, 16, 4, 128, 384), (1500, 4, 1, 128, 200),
                                       (1, 8, 2, 512, 1024), (2048, 4, 2, 64, 256)])
def test_gemm_swiglu_matches_oracle(T, E, k, H, I):
    ids = synth.route_gumbel(T + I, T, E, k)
    X = synth.make_x(T, T, H)
    (Wg, Wu, _), (Wgd, Wud, _) = _weights(T, E, H, I, 64)
    Xd = torch.from_numpy(X).to(torch.bfloat16).cuda()
    counts, row_off, tok, slot, _ = M.moe_route(torch.from_numpy(ids).cuda(), E)
    plan = M.Plan(counts.cpu().numpy(), H, I, 256, 256)
    Y = torch.full((tok.numel(), I), float("nan"), dtype=torch.bfloat16, device="cuda")
    M.moe_gemm_swiglu(plan, Xd, tok, Wgd, Wud, Y=Y)
    torch.cuda.synchronize()
    rc, rr, rt, rs = omoe.buckets(ids, E)
    ref = offn.swiglu_rows(X, Wg, Wu, rt, rr)            # bf16-rounded h (R14)
    got = Y.cpu().double().numpy()
    assert not np.isnan(got).any()
    tol_check(got, ref, f"swiglu {T},{E},{k},{H},{I}")
    # the same values in fp32 output: the unrounded activation
    Y32 = M.moe_gemm_swiglu(plan, Xd, tok, Wgd, Wud, out_dtype=torch.float32)
    torch.cuda.synchronize()
    tol_check(Y32.cpu().double().numpy(), offn.swiglu_rows(X, Wg, Wu, rt, rr, h_bf16=False), "swiglu fp32")


def test_gemm_swiglu_rejects_other_tiles():
    Xd = torch.zeros((4, 64), dtype=torch.bfloat16, device="cuda")
    W = torch.zeros((2, 64, 512), dtype=torch.bfloat16, device="cuda")
    tok = torch.zeros(2, dtype=torch.int32, device="cuda")
    with pytest.raises(M.MoeError):
        M.moe_gemm_swiglu(M.Plan([1, 1], 64, 512, 256, 512), Xd, tok, W, W)
    with pytest.raises(M.MoeError):
        M.moe_gemm_swiglu(M.Plan([1, 1], 64, 512, 128, 256), Xd, tok, W, W)


@pytest.mark.parametrize("ydt,odt", [(torch.bfloat16, torch.float32), (torch.float32, torch.float32),
                                     (torch.bfloat16, torch.bfloat16)])
def test_combine_matches_definition(ydt, odt):
    T, E, k, N = 700, 9, 3, 136
    rng = np.random.default_rng(7)
    ids = synth.route_gumbel(7, T, E, k)
    ids[rng.random((T, k)) < 0.15] = -1                   # masked slots contribute nothing
    ids[3, :] = -1                                        # a token with no slot at all -> zeros
    counts, row_off, tok, slot, _ = M.moe_route(torch.from_numpy(ids).cuda(), E)
    R = int(row_off[-1].item())
    Y = torch.from_numpy(rng.standard_normal((T * k, N))).to(ydt).cuda()
    w = rng.random((T, k)).astype(np.float32)
    out = M.moe_combine(Y, tok, slot, row_off, torch.from_numpy(w).cuda(), out_dtype=odt)
    torch.cuda.synchronize()
    Yh = Y.double().cpu().numpy()
    t_h, s_h = tok.cpu().numpy()[:R], slot.cpu().numpy()[:R]
    ref = np.zeros((T, N))
    for r in range(R):
        ref[t_h[r]] += float(w[t_h[r], s_h[r]]) * Yh[r]
    got = out.double().cpu().numpy()
    if odt == torch.float32:
        assert np.allclose(got, ref, rtol=1e-5, atol=1e-5)
    else:
        tol_check(got, ref, "combine bf16")
    assert (got[3] == 0).all()


@pytest.mark.parametrize("T,E,k,H,I,Ho,masked", [(300, 5, 2, 256, 512, 128, False), (257, 8, 2, 128, 384, 256, True),
                                                 (64, 16, 4, 192, 256, 64, False), (1, 4, 2, 256, 512, 256, False)])
def test_moe_ffn_layer_matches_oracle(T, E, k, H, I, Ho, masked):
    ids = synth.route_gumbel(T * 3 + E, T, E, k)
    rng = np.random.default_rng(T)
    if masked:
        ids[rng.random((T, k)) < 0.2] = -1
    w = rng.random((T, k)).astype(np.float32)
    X = synth.make_x(T + 1, T, H)
    (Wg, Wu, Wd), (Wgd, Wud, Wdd) = _weights(T + 5, E, H, I, Ho)
    layer = M.MoeFFN(Wgd, Wud, Wdd)
    out = layer.forward(torch.from_numpy(X).to(torch.bfloat16).cuda(), torch.from_numpy(ids).cuda(),
                        torch.from_numpy(w).cuda(), out_dtype=torch.float32)
    torch.cuda.synchronize()
    ref = offn.moe_ffn(X, Wg, Wu, Wd, ids, w)
    tol_check(out.cpu().double().numpy(), ref, f"ffn {T},{E},{k},{H},{I},{Ho}")
    # a second step on the same layer object (plans re-built on the device)
    ids2 = synth.route_gumbel(99, T, E, k)
    out2 = layer.forward(torch.from_numpy(X).to(torch.bfloat16).cuda(), torch.from_numpy(ids2).cuda(),
                         torch.from_numpy(w).cuda(), out_dtype=torch.float32)
    torch.cuda.synchronize()
    tol_check(out2.cpu().double().numpy(), offn.moe_ffn(X, Wg, Wu, Wd, ids2, w), "ffn step 2")


def test_graft_entry_smoke():
    """The driver's round-end smoke() must pass on the GPU box."""
    import __graft_entry__

    __graft_entry__.smoke()
