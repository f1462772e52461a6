"""Test double of the EP kernels (CPU, torch ops) following the contracts in
include/moe_sm100_ep.h and include/moe_sm100.h — used ONLY to drive the expert-parallel
exchange logic (splits, offsets, metadata, all-to-alls) over gloo on CPU.  The GPU tests run
the same orchestration with the real CUDA kernels."""
import torch


class CpuKernels:
    def dispatch_plan(self, topk, E, G):
        T, k = topk.shape
        El = E // G
        counts2 = torch.zeros((G, 2), dtype=torch.int32)
        toks, metas, off = [], [], [0]
        # a repeated id in a token's row counts once, at its first slot (as the CUDA kernels do)
        first = torch.ones_like(topk, dtype=torch.bool)
        for j in range(1, k):
            first[:, j] = ~(topk[:, :j] == topk[:, j:j + 1]).any(1)
        for d in range(G):
            own = (topk >= 0) & (topk // El == d) & first
            rows = torch.nonzero(own.any(1)).flatten()
            counts2[d, 0] = rows.numel()
            counts2[d, 1] = int(own.sum())
            toks.append(rows.to(torch.int32))
            metas.append(torch.where(own[rows], topk[rows] - d * El, torch.full_like(topk[rows], -1)))
            off.append(off[-1] + rows.numel())
        send_tok = torch.cat(toks) if toks else torch.zeros(0, dtype=torch.int32)
        send_meta = torch.cat(metas).to(torch.int32) if metas else torch.zeros((0, k), dtype=torch.int32)
        return counts2, torch.tensor(off, dtype=torch.int32), send_tok, send_meta

    def gather_rows(self, src, idx):
        return src[idx.long()].clone()

    def route(self, ids, E):
        R, k = ids.shape
        tok, slot, counts = [], [], torch.zeros(E, dtype=torch.int32)
        for e in range(E):
            for r in range(R):
                for j in range(k):
                    if int(ids[r, j]) == e:
                        tok.append(r)
                        slot.append(j)
                        counts[e] += 1
        return counts, torch.tensor(tok, dtype=torch.int32), torch.tensor(slot, dtype=torch.int32)

    def combine_map(self, tok, slot, recv_off, ret_off, G, k):
        n = tok.numel()
        row_map = torch.zeros(n, dtype=torch.int32)
        ret_meta = torch.zeros(n, dtype=torch.int32)
        cursor = [0] * G
        for i in range(n):
            r = int(tok[i])
            s = max(g for g in range(G) if int(recv_off[g]) <= r)
            pos = int(ret_off[s]) + cursor[s]
            cursor[s] += 1
            row_map[i] = pos
            ret_meta[pos] = (r - int(recv_off[s])) * k + int(slot[i])
        return row_map, ret_meta

    def gemm(self, key, counts, Xr, tok, W, Y, row_map, bm, bn, scale=None):
        fp8 = W.dtype == torch.uint8                      # E4M3 codes (include/moe_sm100_fp8.h)
        dec = (lambda a: a.view(torch.float8_e4m3fn).double()) if fp8 else (lambda a: a.double())
        row0 = 0
        for e in range(W.shape[0]):
            m = int(counts[e])
            s = float(scale[e]) if scale is not None else 1.0
            for i in range(row0, row0 + m):
                Y[int(row_map[i])] = (s * (dec(Xr[int(tok[i])]) @ dec(W[e]))).to(Y.dtype)
            row0 += m
        return Y

    def unpack(self, rows, ret_meta, ret_off, send_off, send_tok, G, k, out):
        for i in range(rows.shape[0]):
            d = max(g for g in range(G) if int(ret_off[g]) <= i)
            m = int(ret_meta[i])
            t = int(send_tok[int(send_off[d]) + m // k])
            out[t * k + m % k] = rows[i]
        return out
