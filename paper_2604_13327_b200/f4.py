"""f4: the reference's tensor-parallel prefill workloads (ref workloads.cpp:30-79,
PAPER.md:642-702) with real data on the persistent megakernel.

GEMM + reduce-scatter at prefill scale (8192 tokens).  The reference's template
`gemm_reduce_scatter(mm_tiles, fan_in)` is a fan-in reduction gated per output
tile: `mm` tiles notify E[t0 // fan_in], each `rs` tile waits E[t0].  Here the
same structure, with the fan-in being the TP ranks' k-splits of a row-parallel
projection Y = X W^T (X [T][K] bf16, W [N][K] bf16, K split over R ranks):

    mm [J, G * R]     token block j (128 tokens), row-block group g, rank r:
                      Y_r[j, g] = X[j, K_r] W[g, K_r]^T on tcgen05 (M = 128 weight rows,
                      N = 128 tokens, K = 16), fp32 in TMEM -> rank r's partial buffer
                      (GEMV_TC tiled mode, flags bit 6)      notifies E[j, g]
    rs [J, G]         waits E[j, g] (R notifies): out[j, g] = sum_r Y_r[j, g]
                      (ET_OP_REDUCE), bf16

so every output tile is reduced the moment its R partials exist, overlapping
the reduction with the GEMM tiles still running -- the Event Tensor overlap the
paper builds the TP MLP from.  On one GPU the R ranks are the k-splits of one
program and their partial buffers live in this GPU's memory; on a TP node the
partials are the peers' buffers (the in-megakernel allreduce's P2P mapping,
tp.py).  The algorithmic work per step is 2 T N K flops.
"""

import json
import math
import time

import torch

from . import etsim
from .batch import tc_pack
from .ops import EPI_F32, OP_GEMV_TC, OP_REDUCE, make_op, pack, ptr

TB = 128  # tokens per block (the MMA N dimension)
KP = 64   # piece length: 128 tokens x 64 k = one 16 KB activation piece


def x_operand(x):
    """[T][K] bf16 -> per 128-token block, the tensor-core operand layout of
    ops.cuh xb_offset (pieces of KP, k steps of 16, 8-row groups, k halves, 8 x 8)."""
    T, K = x.shape
    assert T % TB == 0 and K % KP == 0
    v = x.reshape(T // TB, TB // 8, 8, K // KP, KP // 16, 2, 8)  # j, ngroup, n, piece, kstep, khalf, k
    return v.permute(0, 3, 4, 1, 5, 2, 6).contiguous().reshape(-1)


def gemm_rs_spec(J, G, R):
    """The reference-format graph: the fan-in structure of gemm_reduce_scatter
    (ref workloads.cpp:30-54) with 2-D grids (token block, tile)."""
    return {
        "symbols": [], "size_symbol": "",
        "duration_models": {"unit": {"kind": "constant", "value": 1}},
        "device_functions": [
            {"name": "mm", "grid": [str(J), str(G * R)], "resource": "sm", "duration": "unit"},
            {"name": "rs", "grid": [str(J), str(G)], "resource": "sm", "duration": "unit"}],
        "event_tensors": [{"name": "E", "shape": [str(J), str(G)]}],
        "calls": [
            {"fn": "mm", "out": [{"event": "E", "map": ["t0", f"t1 // {R}"]}]},
            {"fn": "rs", "in": [{"event": "E", "map": ["t0", "t1"]}]}],
    }


class GemmReduceScatter:
    """Y = X W^T with K split over `ranks`, reduce-scattered per output tile."""

    def __init__(self, tokens=8192, n=4096, k=14336, ranks=2, groups=None, device="cuda:0", seed=0,
                 num_workers=None, record_trace=False, x=None, w=None, stage_barriers=False):
        if not etsim.gpu_available():
            raise RuntimeError("GemmReduceScatter needs a CUDA device")
        assert tokens % TB == 0 and n % 128 == 0 and k % (KP * ranks) == 0
        dev = torch.device(device)
        self.T, self.N, self.K, self.R = tokens, n, k, ranks
        self.J = tokens // TB
        nblk = n // 128
        # row-block groups: two 128-row blocks per tile (2 x 128 TMEM columns per issuer)
        self.G = groups or max(1, nblk // 2)
        assert nblk % self.G == 0
        self.rows_per_group = n // self.G
        workers = num_workers or torch.cuda.get_device_properties(dev).multi_processor_count
        t0 = time.perf_counter()
        self.spec = gemm_rs_spec(self.J, self.G, ranks)
        if stage_barriers:  # the reference's barrier baseline: rs only after the whole mm call
            from .graphs import add_stage_barriers
            self.spec = add_stage_barriers(self.spec)
        self.graph = etsim.Graph.from_json(json.dumps(self.spec))
        self.kernel = etsim.lower_static(self.graph, [{}], num_sms=workers)
        self.lower_ms = (time.perf_counter() - t0) * 1e3
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        self.x = x if x is not None else torch.randn(tokens, k, device=dev, generator=g).to(torch.bfloat16)
        self.w = w if w is not None else (torch.randn(n, k, device=dev, generator=g) * (1 / math.sqrt(k))).to(
            torch.bfloat16)
        self.x_op = x_operand(self.x)
        self.w_tc = tc_pack(self.w, KP)
        self.partials = torch.zeros(ranks, tokens, n, dtype=torch.float32, device=dev)
        self.out = torch.zeros(tokens, n, dtype=torch.bfloat16, device=dev)
        self.executor = etsim.Executor(self.kernel, device=dev.index or 0, num_workers=workers,
                                       record_trace=record_trace, max_batch=TB)
        self.executor.bind_ops(pack(self._ops()))

    def _ops(self):
        T, N, K, R, G = self.T, self.N, self.K, self.R, self.G
        # i: N, K, segments, k splits (= ranks), epilogue, batch slot, kp, -, row stride,
        #    -, tokens per block, partial stride, tasks per block, -
        mm = make_op(OP_GEMV_TC, i=[N, K, 1, R, EPI_F32, -1, KP, 0, N, 0, TB, T * N, G * R, 0], flags=64,
                     p=[ptr(self.w_tc), 0, ptr(self.x_op), 0, ptr(self.partials)])
        rs = make_op(OP_REDUCE, i=[N, TB, R, T * N, self.rows_per_group, 1],
                     p=[ptr(self.partials), ptr(self.out)])
        return [mm, rs]

    def flops(self):
        return 2 * self.T * self.N * self.K

    def step(self):
        self.last_stats = self.executor.run({})
        return self.out

    def launch(self, stream=0):
        self.executor.launch({}, stream)

    def reference(self):
        """fp32 product of the same bf16 operands (torch on the device)."""
        return self.x.float() @ self.w.float().t()


class AllGatherGemm:
    """All-gather + GEMM (ref workloads.cpp:56-79, the reference's own template
    `all_gather_gemm(chunks, tiles_per_chunk)`): chunk r of the token rows belongs
    to rank r; the DMA-class `copy` tasks run in a chain (chain[r] -> copy r ->
    chain[r+1]) and release `arrival[r]`, which gates that chunk's GEMM tiles, so the
    GEMM on chunk r overlaps the gathering of the later chunks.

    B200 form (pull-based): a copy task does not move the chunk -- the GEMM tiles'
    TMA loads read it in place (the peer's buffer over NVLink on a TP node, its own
    memory here); the copy task pulls it into L2 ahead of them (cp.async.bulk.prefetch.L2)
    and releases the arrival element.  `push=True` copies it into a gather buffer
    with the DMA warp instead (one warp: slow, for checking)."""

    def __init__(self, tokens=8192, n=4096, k=4096, chunks=8, groups=None, device="cuda:0", seed=0,
                 num_workers=None, record_trace=False, push=False, x=None, w=None):
        if not etsim.gpu_available():
            raise RuntimeError("AllGatherGemm needs a CUDA device")
        assert tokens % (TB * chunks) == 0 and n % 128 == 0 and k % KP == 0
        dev = torch.device(device)
        self.T, self.N, self.K, self.C = tokens, n, k, chunks
        self.bpc = tokens // TB // chunks  # token blocks per chunk
        nblk = n // 128
        self.G = groups or max(1, nblk // 2)
        assert nblk % self.G == 0
        workers = num_workers or torch.cuda.get_device_properties(dev).multi_processor_count
        t0 = time.perf_counter()
        self.graph = etsim.all_gather_gemm(chunks, self.bpc * self.G)
        self.kernel = etsim.lower_static(self.graph, [{}], num_sms=workers)
        self.lower_ms = (time.perf_counter() - t0) * 1e3
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        self.x = x if x is not None else torch.randn(tokens, k, device=dev, generator=g).to(torch.bfloat16)
        self.w = w if w is not None else (torch.randn(n, k, device=dev, generator=g) * (1 / math.sqrt(k))).to(
            torch.bfloat16)
        self.x_src = x_operand(self.x)  # the ranks' chunks, contiguous per chunk
        self.push = push
        self.x_gather = torch.empty_like(self.x_src) if push else self.x_src
        self.w_tc = tc_pack(self.w, KP)
        self.out = torch.zeros(tokens, n, dtype=torch.float32, device=dev)
        self.executor = etsim.Executor(self.kernel, device=dev.index or 0, num_workers=workers,
                                       record_trace=record_trace, max_batch=TB)
        self.executor.bind_ops(pack(self._ops()))

    def _ops(self):
        from .ops import OP_COPY
        N, K, G = self.N, self.K, self.G
        chunk_bytes = self.bpc * TB * K * 2
        copy = make_op(OP_COPY, i=[chunk_bytes], flags=0 if self.push else 2,
                       p=[ptr(self.x_src), ptr(self.x_gather)])
        gemm = make_op(OP_GEMV_TC, i=[N, K, 1, 1, EPI_F32, -1, KP, 0, N, 0, TB, 0, G, self.bpc], flags=64 | 128,
                       p=[ptr(self.w_tc), 0, ptr(self.x_gather), 0, ptr(self.out)])
        return [copy, gemm]

    def flops(self):
        return 2 * self.T * self.N * self.K

    def step(self):
        self.last_stats = self.executor.run({})
        return self.out

    def reference(self):
        return self.x.float() @ self.w.float().t()
