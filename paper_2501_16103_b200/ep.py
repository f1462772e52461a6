"""Expert parallelism (EP) over G ranks: NCCL all-to-all dispatch / combine around the
single-launch expert GEMM.

The paper treats EP as background (a subset of experts per GPU; each GPU's share
of the MoE layer is still an irregular batch, handled by the same statically batched
kernel).  Sharding (R8): rank g owns experts [g*E/G, (g+1)*E/G) and its own
tokens.  One forward (`ExpertParallelMoE.forward`):

  1. moe_ep_dispatch_plan: per destination, the owned tokens with >= 1 expert there
     (deduplicated, ascending) and their destination-local expert ids (-1 elsewhere);
  2. one all-to-all of 2 ints per peer (send rows, result rows to come back) and ONE
     device->host read of those sizes (NCCL needs split sizes on the host);
  3. moe_gather_rows packs the token rows, all-to-all of rows + local-id metadata;
  4. moe_route (masked slots skipped) -> moe_plan_device -> moe_ep_combine_map ->
     moe_gemm_rowmap, whose epilogue writes every result row straight into the combine
     send buffer (no Y gather copy);
  5. all-to-all of result rows + their (row, slot) metadata back; moe_ep_unpack places
     them at (token, slot): out[t * k + j] = X[t] @ W[topk[t, j]].

torch.distributed is plumbing only (process group, collectives, memory).  `kernels` and
`comm` are injectable so tests can drive the exchange logic with gloo on CPU (with a
test double of the kernels) or with G virtual ranks in one process on one GPU; the
default is the CUDA library — there is no CPU fallback.
"""
from __future__ import annotations

import threading

import torch


class CudaKernels:
    """The library's CUDA kernels (include/moe_sm100.h, include/moe_sm100_ep.h)."""

    def __init__(self):
        from . import (Plan, moe_ep_combine_map, moe_ep_dispatch_plan, moe_ep_unpack, moe_gather_rows, moe_gemm,
                       moe_gemm_fp8, moe_route)
        self._Plan, self._gemm, self._gemm_fp8, self._route = Plan, moe_gemm, moe_gemm_fp8, moe_route
        self.dispatch_plan = moe_ep_dispatch_plan
        self.gather_rows = moe_gather_rows
        self.combine_map = moe_ep_combine_map
        self.unpack = moe_ep_unpack
        self._plans = {}

    def route(self, ids, E):
        counts, row_off, tok, slot, _ = self._route(ids, E)
        return counts, tok, slot

    def gemm(self, key, counts, Xr, tok, W, Y, row_map, bm, bn, scale=None):
        plan = self._plans.get(key)
        if plan is None:
            plan = self._Plan(None, W.shape[1], W.shape[2], bm, bn, E=W.shape[0])
            self._plans[key] = plan
        plan.update_device(counts)
        if tok.numel():
            if W.dtype in (torch.uint8, torch.float8_e4m3fn):     # FP8 E4M3 (include/moe_sm100_fp8.h)
                self._gemm_fp8(plan, Xr, tok, W, scale, Y=Y, row_map=row_map)
            else:
                self._gemm(plan, Xr, tok, W, Y=Y, row_map=row_map)
        return Y


class TorchComm:
    """All-to-all over a torch.distributed process group (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def all_to_all(self, out, inp, out_splits, in_splits):
        self.dist.all_to_all_single(out, inp, output_split_sizes=out_splits, input_split_sizes=in_splits,
                                    group=self.group)


class ThreadComm:
    """G virtual ranks in one process (one thread each): an exact in-process all-to-all.
    Used by tests to exercise the G > 1 data path on a single device."""

    def __init__(self, size: int):
        self.size = size
        self._bar = threading.Barrier(size)
        self._box = [None] * size
        self._local = threading.local()

    def bind(self, rank: int):
        self._local.rank = rank
        return self

    @property
    def rank(self):
        return self._local.rank

    def all_to_all(self, out, inp, out_splits, in_splits):
        r = self.rank
        self._bar.wait()
        self._box[r] = list(torch.split(inp, list(in_splits)))
        self._bar.wait()
        parts = [self._box[s][r] for s in range(self.size)]
        if out.numel():
            torch.cat(parts, out=out) if len(parts) > 1 else out.copy_(parts[0])
        self._bar.wait()


def _excl(x):
    o = torch.zeros(x.numel() + 1, dtype=torch.int32, device=x.device)
    o[1:] = torch.cumsum(x, 0)
    return o


class ExpertParallelMoE:
    """One rank of an expert-parallel MoE expert GEMM."""

    def __init__(self, E: int, W_local, comm, bm: int = 0, bn: int = 0, out_dtype=torch.bfloat16, kernels=None,
                 w_scale=None):
        """W_local [E/G, H, N]: bf16, or FP8 E4M3 codes (uint8 / float8_e4m3fn) with the optional
        per-local-expert fp32 w_scale [E/G]; X rows then travel as FP8 (half the dispatch bytes)."""
        self.comm = comm
        self.G = comm.size
        if E % self.G:
            raise ValueError("E must be divisible by the number of ranks")
        self.E, self.El = E, E // self.G
        if W_local.shape[0] != self.El:
            raise ValueError("W_local must hold E / G experts")
        self.W = W_local
        self.w_scale = w_scale
        self.bm, self.bn, self.out_dtype = bm, bn, out_dtype
        self.kernels = kernels if kernels is not None else CudaKernels()
        self.last = {}
        self.time_gemm = False        # bench: record CUDA events around the GEMM launch
        self.gemm_events = None

    def forward(self, topk_local, X_local):
        """topk_local [T_l, k] int32 global expert ids, X_local [T_l, H] bf16 (FP8 codes with FP8
        weights) -> out [T_l * k, N]."""
        K, G, comm = self.kernels, self.G, self.comm
        dev = X_local.device
        T_l, k = topk_local.shape
        H, N = X_local.shape[1], self.W.shape[2]
        counts2, send_off, send_tok, send_meta = K.dispatch_plan(topk_local, self.E, G)
        recv2 = torch.empty_like(counts2)
        comm.all_to_all(recv2.view(-1), counts2.view(-1), [2] * G, [2] * G)
        sizes = torch.stack([counts2, recv2]).cpu()          # the step's one host read (split sizes)
        send_rows, back_rows = sizes[0, :, 0].tolist(), sizes[0, :, 1].tolist()
        recv_rows, ret_rows = sizes[1, :, 0].tolist(), sizes[1, :, 1].tolist()
        S, R, Rr, B = sum(send_rows), sum(recv_rows), sum(ret_rows), sum(back_rows)
        # dispatch
        Xs = K.gather_rows(X_local, send_tok[:S])
        Xr = torch.empty((R, H), dtype=X_local.dtype, device=dev)
        Mr = torch.empty((R, k), dtype=torch.int32, device=dev)
        comm.all_to_all(Xr, Xs, recv_rows, send_rows)
        comm.all_to_all(Mr, send_meta[:S].contiguous(), recv_rows, send_rows)
        # local experts: route (masked slots skipped), device plan, GEMM into the combine buffer
        counts_l, tok_l, slot_l = K.route(Mr, self.El)
        tok_l, slot_l = tok_l[:Rr], slot_l[:Rr]              # valid (unmasked) local slots = sum(ret_rows)
        recv_off = _excl(recv2[:, 0])
        ret_off = _excl(recv2[:, 1])
        row_map, ret_meta = K.combine_map(tok_l, slot_l, recv_off, ret_off, G, k)
        Ysend = torch.empty((Rr, N), dtype=self.out_dtype, device=dev)
        if self.time_gemm:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
        K.gemm(("ep", self.bm, self.bn), counts_l, Xr, tok_l, self.W, Ysend, row_map, self.bm, self.bn, self.w_scale)
        if self.time_gemm:
            ev[1].record()
            self.gemm_events = ev
        # combine
        Yb = torch.empty((B, N), dtype=self.out_dtype, device=dev)
        Mb = torch.empty(B, dtype=torch.int32, device=dev)
        comm.all_to_all(Yb, Ysend, back_rows, ret_rows)
        comm.all_to_all(Mb, ret_meta.contiguous(), back_rows, ret_rows)
        out = torch.empty((T_l * k, N), dtype=self.out_dtype, device=dev)
        back_off = _excl(counts2[:, 1])
        K.unpack(Yb, Mb, back_off, send_off, send_tok, G, k, out)
        self.last = dict(send_rows=send_rows, recv_rows=recv_rows, ret_rows=ret_rows, back_rows=back_rows,
                         local_rows=int(tok_l.numel()))
        return out
