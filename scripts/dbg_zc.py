import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2501_16103_b200 as M, synth
from oracle import moe as omoe
sys.path.insert(0, "tests"); from test_ep_peer import _routing
G, E, k, T_l, H, N = 4, 8, 2, 64, 64, 512
T = G * T_l; El = E // G
X, W = synth.make_x(7, T, H, "int"), synth.make_w(7, E, H, N, "int")
ids = _routing(0, T, E, k, masked=False)
Ws = [torch.from_numpy(W[r * El:(r + 1) * El]).to(torch.bfloat16).cuda() for r in range(G)]
Xs = [torch.from_numpy(X[r * T_l:(r + 1) * T_l]).to(torch.bfloat16).cuda() for r in range(G)]
tks = [torch.from_numpy(ids[r * T_l:(r + 1) * T_l]).cuda() for r in range(G)]
eps = M.PeerExpertParallel.group(G, E, Ws, max_tokens=T_l, k=k, max_out_bytes=N * 2)
outs = [ep.output(T_l, N) for ep in eps]
print(outs[0].dtype, outs[0].shape, outs[0].stride(), hex(outs[0].data_ptr()))
for r in range(G):
    eps[r].forward(tks[r], Xs[r], out=outs[r])
torch.cuda.synchronize()
got = torch.cat([o.float().cpu() for o in outs]).double().numpy()
ref = omoe.per_slot_outputs(ids, X, W)
refb = torch.from_numpy(ref).float().to(torch.bfloat16).double().numpy()
bad = np.nonzero(got != refb)
print("mismatch", len(bad[0]), "of", got.size, "rows", np.unique(bad[0])[:20], "cols", np.unique(bad[1])[:20])
if len(bad[0]): 
    i, j = bad[0][0], bad[1][0]; print(got[i, j], refb[i, j], ref[i,j])
# fp32 out through the copy path for comparison
o2 = [torch.empty((T_l*k, N), dtype=torch.bfloat16, device='cuda') for _ in range(G)]
for r in range(G):
    eps[r].forward(tks[r], Xs[r], out=o2[r])
torch.cuda.synchronize()
g2 = torch.cat([o.float().cpu() for o in o2]).double().numpy()
print("copy path mismatch", int((g2 != refb).sum()))
