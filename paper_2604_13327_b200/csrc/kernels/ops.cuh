// Tile bodies executed inside the persistent megakernel, and the streaming
// plans shared by the producer (TMA issuer) and the consumer warps.
//
// et_op parameter layout per kind
// -------------------------------
// ET_OP_SPLITK_PARTIAL  task (row, part): partial[row*parts+part] = sum of data[row][part*L:(part+1)*L]
//   i0 = L, i1 = parts; p0 = data (int32 [n][parts*L]), p1 = partials (int32 [n][parts])
// ET_OP_SPLITK_FINAL    task (row): out[row] = sum_j partials[row*parts+j]
//   i1 = parts; p1 = partials, p2 = out (int32 [n])
// ET_OP_GEMV            task t of T computes its span (gemv_span) of every segment (T = call grid
//   extent); epilogues: F32/BF16 store, RESID out = p5 + y, SILU_MUL out = silu(y0) * y1,
//   QKV_ROPE (RoPE on q/k pairs, k/v appended to the cache), ADD out += y (red.global.add).
//   flags bit 3 (QKV_ROPE): the weight rows are grouped per kv head (G q heads, k head, v head);
//   flags bit 4: grouped GEMV -- task (g, t) of grid [groups, i13]: matrix g (bf16 [N][K] frag16, the
//   matrices stacked at p0) times activation slice g (p2 + g*K), rows split over i13 tasks;
//   x mode 0: activation rows i9 elements apart (0 = K)
//   i0 = N rows per segment, i1 = K, i2 = segments (1|2), i3 = x mode (0 bf16 [b][K] at p2,
//   1 fp32 residual stream at p2 normalised with RMSNorm gamma p3), i4 = epilogue (GemvEpi),
//   i5 = batch symbol slot (-1: b = 1), i6 = position symbol slot, i7 = row alignment,
//   i8 = head_dim, i9 = x batch stride (elements), i10 = q rows, i11 = kv rows (k and v each),
//   i12 = KV capacity (positions), i13 = split-K (1: even byte spans, EPI_ADD only);
//   p0/p1 = weights (bf16 [N][K], frag16 tile order) of segment 0/1, p4 = out,
//   p5 = residual in (fp32), p6/p7 = K/V cache of the layer (bf16 [kv_heads][cap][head_dim]);
//   p8 = RoPE inverse frequencies (fp32 [head_dim/2], pair j rotates dims 2j, 2j+1); f0 = RMSNorm eps
// ET_OP_ATTN_SPLIT      task (kv_head g, split c) of grid [kv, min(ceil(s/CH), i5)]: flash-decoding
//   partial over its run of CH-position blocks (attn_blocks), online softmax across blocks;
//   i0 = head_dim, i1 = q heads per kv head, i2 = CH (block positions), i3 = KV capacity,
//   i4 = position symbol slot, i5 = split cap (partials' split dimension), i6 = kv heads,
//   i7 = q / projection row stride of a batch sequence, i8 = per-sequence cache stride (elements);
//   batch: grid dim 0 is sequence * kv_heads + kv head (partials / arrival counters per such group);
//   flags bit 8: K/V cache rows store their 16-byte chunks XOR-swizzled by position % 8
//   (chunk j of row p at j ^ (p % 8)): tensor-core reads of 8 rows hit 8 bank groups;
//   flags bit 7: one flat grid dimension [b * kv * splits] instead, with i11 = per-step split
//   budget (splits <= max(1, i11 / b)) and i10 = batch symbol slot (attn_tasks, attn_coord);
//   p0 = q (fp32 [q_heads*head_dim], RoPE applied), p1/p2 = K/V cache, p3 = partials
//   (fp32 [q_heads][max_splits][4 + head_dim]: m, l, pad, pad, o); f0 = softmax scale
// ET_OP_ATTN_MERGE      task (g): merges the splits and the new token at position s
//   (K/V row s of the cache) for the group's q heads; same i/p as ATTN_SPLIT plus
//   p4 = out (bf16 [q_heads*head_dim])
// ATTN_SPLIT flags bit 1 (fused merge): p4 = out, p5 = arrival counters (int32 [kv_heads], zero
//   between steps; the merger resets them); grid [kv, max(ceil(s/CH), 1)]; the split of
//   group g that arrives last runs the ATTN_MERGE body for g (no merge stage, one hop less).
// ATTN flags bit 0 (Qwen3 q/k-norm): q at p0 is the raw projection; SPLIT and MERGE apply
//   the per-head RMSNorm (p5 = q-norm weight, p6 = k-norm weight, fp32 [head_dim], f1 = eps)
//   and RoPE (p7 = inverse frequencies) themselves; MERGE also normalises + rotates the raw
//   new k at p8 + g*head_dim (v at p8 + (kv_heads + g)*head_dim) and appends k/v (bf16) to
//   the cache at position s before using them.  With both bits (fused q/k-norm split) p5 holds the
//   arrival counters and the q-norm weight moves to p9.
// ET_OP_MOE_ROUTE       task t of E/16: router logits rows [16t, 16t+16) (GEMV, RMSNorm prologue,
//   GEMV fields i0..i9 as ET_OP_GEMV with i3 = 1, i4 = EPI_F32); task 0 also stores the
//   normalised activations; the last task to arrive computes the routing for every token:
//   softmax over E, top-k (descending probability, lower expert index wins ties),
//   renormalised weights -- or, with flags bit 0, the host-injected topk -- then expert
//   counts, exp_indptr (tiles of TS tokens, ref workloads.cpp:140-144), task_indptr
//   (x RS), eoff (exclusive prefix of counts) and elist (slots by expert, stable).
//   i6 = top_k, i10 = index of the layer's first routing runtime tensor (in order topk,
//   counts, exp_indptr, task_indptr, elist, eoff), i12 = RS, i13 = TS; p0 = router weight (frag16
//   [E][H]), p2 = h (fp32 [b][H]), p3 = gamma, p4 = logits (fp32 [b][E]), p5 = xn out
//   (bf16 [b][H]), p6 = slot weights out (fp32 [b*top_k]), p7 = arrival counter (int32);
//   The tile table (p8, int4 per tile) holds (expert, first elist index, tokens, routing weight
//   bits of a one-token tile).
//   flags bit 1 (large batch): no GEMV -- one task reads the logits a tensor-core GEMV
//   accumulated at p1 (fp32 [b][E]), copies them to p4 and zeroes p1
// ET_OP_MOE_EXPERT      task flat = tile * RS + r (range-triggered on task_indptr, extent_from):
//   for the tile's tokens x = xn[token]: act = silu(Wg_e x) * (Wu_e x) on rows [r*IR, r*IR+IR)
//   (IR = I / RS), then h[token] += w_slot * Wd_e[:, rows] act (red.global.add).
//   i0 = I, i1 = H, i2 = RS, i3 = TS (<= 8), i4..i7 = rt exp_indptr, counts, elist, eoff,
//   i8 = top_k, i9 = batch symbol slot (-1: one sequence -- every tile is token 0 with one slot and
//   the route left its weight in the tile record's .w), i10 = E; p0/p1 = Wgate/Wup (frag16 [E][I][H]), p2 = Wdown blocks (frag16
//   [E][RS][H][IR]), p3 = xn (bf16 [b][H]), p4 = slot weights, p5 = h (fp32 [b][H]),
//   p6 = tile table (from ET_OP_MOE_ROUTE)
// ET_OP_ALLREDUCE       task t of T (static scheduler): h[r0:r1] += sum over TP ranks of their
//   stage partials (rows split evenly over the T tasks); cross-GPU Event Tensor elements
//   flags[slot][src] (epoch = step id; st.release.sys / ld.acquire.sys).
//   i0 = H, i1 = TP, i2 = this rank, i3 = slot (stage index); p0 = h (fp32 [H]),
//   p1 = local flags (uint32 [slots][TP]), p2 = local once-counters (uint32 [slots]),
//   p3 = peer table (uint64 [TP][2]: rank p's part buffer base (fp32 [slots][H]), its flags)
// ET_OP_EMBED           task (0): h[b][:] = float(table[tokens[b]][:]) for every batch row
//   i0 = hidden, i1 = batch symbol slot (-1: 1); p0 = table (bf16 [vocab][hidden]),
//   p1 = token ids (int32 [b]), p2 = out (fp32 [b][hidden]); flags bit 0: zero the step's
//   greedy argmax words at p3 (u64 [b])
// GEMV flags bit 5 (EPI_F32, b = 1): greedy decoding -- the task's rows fold into the argmax
//   word at p6 (u64: ordered float bits << 32 | ~row, atomicMax)
// ET_OP_ARGMAX          task (0): token[b] = row of the argmax word p0[b] -> p1 (int32 [b]) and,
//   if set, p2 (the next step's token input); words re-zeroed; i0 = batch symbol slot (-1: 1)
// ET_OP_GEMV_TC         large-batch GEMV on the tcgen05 tensor cores: task t of T = G * i3 takes
//   row blocks [g*nblk/G, (g+1)*nblk/G) (128 rows each, nblk = N/128) and k pieces
//   [r*np/i3, (r+1)*np/i3) (np = K/kp) with g = t / i3, r = t % i3; per piece the activation
//   piece (Npad x kp bf16, Npad = batch rounded up to 16) streams into one of two shared
//   buffers, the weight chunks (16 KB = 128 rows x 64 k) through the ring, and one thread
//   issues tcgen05.mma (M=128, N=Npad, K=16) into TMEM accumulators (column block (seg, blk)
//   at (seg*nblk_task + blk)*Npad); the epilogue reads TMEM with tcgen05.ld.
//   i0 = N rows per segment (% 128 == 0), i1 = K, i2 = segments (1|2), i3 = k splits (EPI_ADD
//   only when > 1), i4 = epilogue (F32 / BF16 / RESID / ADD: [b][N] row-major; SILU_MUL:
//   bf16 in the tensor-core operand layout with piece length i7), i5 = batch symbol slot,
//   i6 = kp (piece length, % 64 == 0, Npad * kp * 2 <= 16 KB), i8 = output rows / row stride
//   of the row-major epilogues (0 = N; rows of a zero-padded last block beyond it are dropped);
//   p0/p1 = weights in the tensor-core layout of segment 0/1 (tc_weight_offset), p2 = x in the
//   operand layout (xb_offset), p4 = out, p5 = residual in (fp32, EPI_RESID)
//   flags bit 6 (tiled GEMM, f4 workloads): grid [token blocks, i12]; task (j, t) is GEMV task t of
//   i12 on token block j (i10 tokens, the MMA N; activations at p2 + j * K * Npad, operand
//   layout); EPI_F32 writes Y[j*i10 + n][row] into the k-split's own partial buffer
//   p4 + r * i11 (r = t % i3, i11 elements apart): the reduce-scatter tasks sum them
// ET_OP_REDUCE          task (j, g): out[tokens of block j][rows of group g] = sum over i2 partial
//   buffers (i3 elements apart) at p0; i0 = N (row stride), i1 = tokens per block, i4 = rows per
//   group, i5 = out dtype (0 fp32, 1 bf16); p1 = out
// ET_OP_COPY            DMA-class task t (one warp): i0 bytes from p0 + t * i0 (flags bit 0: from the
//   address p2[t]) to p1 + t * i0; flags bit 1: pull-based all-gather -- no copy, the chunk is
//   prefetched into L2 and its consumers read it in place
// ET_OP_NORM            task n (< b): out[n] = bf16(h[n] * rsqrt(mean(h[n]^2) + eps) * gamma) in
//   the tensor-core operand layout; i0 = K, i5 = batch symbol slot, i6 = kp; p0 = h (fp32
//   [b][K]), p1 = gamma (fp32 [K]), p2 = out, p3 = optional row-major copy (bf16 [b][K]); f0 = eps
#pragma once

#include "megakernel.cuh"
#include "ptx.cuh"

namespace etk {

enum GemvEpi { EPI_F32 = 0, EPI_BF16 = 1, EPI_RESID = 2, EPI_SILU_MUL = 3, EPI_QKV_ROPE = 4, EPI_ADD = 5 };

struct Chunk {
    const uint8_t* src;
    uint32_t bytes;
};

// ---- tensor-core GEMV (ET_OP_GEMV_TC) -------------------------------------------------
constexpr int kTcChunk = 16384;      // weight chunk: 128 rows x 64 k (4 k steps of 4 KB)
constexpr int kTcXBuf = kXBytes / 2;  // largest activation piece (two slots at least)
constexpr int kTcXSlots = 4;          // activation piece slots (as many as fit, up to 4)
constexpr int kTcIssuers = 4;         // MMA issuer threads (lane 0 of consumer warps 0..3)

__host__ __device__ __forceinline__ int tc_xslots(uint32_t xbytes) {
    const int n = static_cast<int>(kXBytes / xbytes);
    return n < kTcXSlots ? n : kTcXSlots;
}
constexpr int kTmemCols = 512;

// Batch padded to the MMA N dimension (multiple of 16, at least 16).
__host__ __device__ __forceinline__ int tc_npad(int nb) { return nb <= 16 ? 16 : (nb + 15) & ~15; }

// Element offset of activation (n, k) in the operand layout: pieces of kp, then
// k steps of 16, then 8-row groups of the batch, then the two 8-wide k halves,
// then 8 rows x 8 k (16-byte core-matrix rows).
__host__ __device__ __forceinline__ long long xb_offset(int n, int k, int npad, int kp) {
    const int piece = k / kp, kk = k - piece * kp;
    return static_cast<long long>(piece) * npad * kp + (kk >> 4) * (npad * 16) + (n >> 3) * 128 + ((kk >> 3) & 1) * 64 +
           (n & 7) * 8 + (k & 7);
}

// Tiled GEMM mode (GEMV_TC flags bit 6, the f4 workloads): grid [token blocks, i12 tasks per
// block]; coordinate 1 is the GEMV task (row-block group, k split), coordinate 0 the block
// of i10 tokens.  Batch (MMA N) = i10; otherwise the batch symbol's value.
__host__ __device__ __forceinline__ bool tc_tiled(const et_op& op) { return (op.flags & 64) != 0; }
__host__ __device__ __forceinline__ int tc_batch(const et_op& op, const long long* binding) {
    if (tc_tiled(op)) return op.i[10];
    return op.i[5] >= 0 ? static_cast<int>(binding[op.i[5]]) : 1;
}

// (token block, GEMV task) of a tiled-GEMM task.  flags bit 7 (the reference's
// all_gather_gemm grid [chunks, tiles per chunk]): coordinate 1 also walks the i13
// token blocks of chunk coord 0 -- block = coord0 * i13 + coord1 / i12, task = coord1 % i12.
__host__ __device__ __forceinline__ void tc_tile(const et_op& op, const int* coord, int* j, int* t) {
    if (op.flags & 128) {
        *j = coord[0] * op.i[13] + coord[1] / op.i[12];
        *t = coord[1] % op.i[12];
    } else {
        *j = coord[0];
        *t = coord[1];
    }
}

struct TcSpan {
    int b0, nblk;  // first row block, row blocks of the task
    int p0, np;    // first k piece, pieces of the task
};

__host__ __device__ __forceinline__ TcSpan tc_span(const et_op& op, int t, int T) {
    const int splits = op.i[3] > 0 ? op.i[3] : 1;
    const int G = T / splits > 0 ? T / splits : 1;
    const int g = t / splits, r = t - g * splits;
    const int nblk = op.i[0] / 128, npc = op.i[1] / op.i[6];
    TcSpan sp;
    sp.b0 = static_cast<int>(static_cast<long long>(g) * nblk / G);
    sp.nblk = static_cast<int>(static_cast<long long>(g + 1) * nblk / G) - sp.b0;
    sp.p0 = static_cast<int>(static_cast<long long>(r) * npc / splits);
    sp.np = static_cast<int>(static_cast<long long>(r + 1) * npc / splits) - sp.p0;
    if (g >= G) sp.nblk = 0;
    return sp;
}

// Streaming plan of one task: up to two contiguous byte ranges cut into
// chunks of `cbytes` (<= one ring stage).  GEMV streams segment 0 then
// segment 1; attention interleaves them (K block 0, V block 0, K block 1, ...).
struct StreamPlan {
    static constexpr int kMaxSeg = 3;
    const uint8_t* base[kMaxSeg];
    long long bytes[kMaxSeg];
    int nseg;
    int cbytes;
    bool interleave;
    int n[kMaxSeg];  // chunks per segment (set by finish(); keeps divisions off the per-chunk path)
    // tensor-core GEMV (streamed by tc_produce, not chunk()): tc_w = weight chunks per piece,
    // tc_np = pieces (0: not a tensor-core plan), tc_pre = weight chunks streamed before X(0)
    int tc_w = 0, tc_np = 0, tc_pre = 0;
    const uint8_t* tc_x;       // activation piece p at tc_x + p * tc_xbytes
    uint32_t tc_xbytes;
    long long tc_pstride;      // weight bytes between pieces (whole matrix width)

    __device__ void finish() {
        for (int s = 0; s < kMaxSeg; ++s) n[s] = s < nseg ? static_cast<int>((bytes[s] + cbytes - 1) / cbytes) : 0;
    }
    __device__ int total_chunks() const { return n[0] + n[1] + n[2]; }
    __device__ Chunk chunk(int idx) const {
        int s = 0;
        if (interleave) {
            s = idx & 1;
            idx >>= 1;
        } else {
            while (s < kMaxSeg - 1 && idx >= n[s]) idx -= n[s++];
        }
        const long long off = static_cast<long long>(idx) * cbytes;
        const long long rem = bytes[s] - off;
        return Chunk{base[s] + off, static_cast<uint32_t>(rem < cbytes ? rem : cbytes)};
    }
};

// ---- MoE ------------------------------------------------------------------
// Expert task (tile, r) of the routed expert call: flat = tile * RS + r.  The
// tile's expert e is the group of `tile` in exp_indptr (tiles of TS tokens,
// ref workloads.cpp:140-144); its tokens are the slots elist[eoff[e] + i*TS +
// j] (slot = token * top_k + k, stable in slot order).  Valid only once the
// routing writer has finished (after the task's waits).
struct ExpertTask {
    int e, tile, r, ntok;
    int slot[8];
};

// Expert id and row split of a task (the streaming plan needs nothing else).
__device__ __forceinline__ void expert_of(const et_op& op, int flat, int* e, int* r) {
    const int RS = op.i[2];
    const int tile = flat / RS;
    *r = flat - tile * RS;
    *e = __ldcg(reinterpret_cast<const int*>(op.p[6]) + 4 * tile);
}

__device__ __forceinline__ ExpertTask expert_task(const et_op& op, int flat, int* const* rt) {
    const int RS = op.i[2];
    const int* elist = rt[op.i[6]];
    ExpertTask t;
    t.tile = flat / RS;
    t.r = flat - t.tile * RS;
    // (expert, first slot, tokens) of the tile, written by the route task
    const int4 info = __ldcg(reinterpret_cast<const int4*>(op.p[6]) + t.tile);
    t.e = info.x;
    t.ntok = info.z;
#pragma unroll
    for (int j = 0; j < 8; ++j) t.slot[j] = j < t.ntok ? __ldcg(elist + info.y + j) : 0;
    return t;
}

// Work span of GEMV task t of T, in k-step units of the frag16 tile order
// (unit u = row tile u / kst, k-step u % kst; kst = K / 16).  Without split-K
// tasks own whole row ranges ([r0, r1) split evenly in units of i7 rows, a
// multiple of 16); with split-K (i13 = 1) the N*K/256 units are split evenly,
// in pairs of k-steps, so every task streams the same number of bytes and the
// row tiles at the ends of its span are partial (their sums are combined with
// red.global.add by the epilogue).  A span is one contiguous byte range.
struct GemvSpan {
    long long u0, u1;  // [u0, u1) units
    int row0;          // first row of the first tile touched
    int rows;          // rows of all tiles touched (multiple of 16)
};

__device__ __forceinline__ GemvSpan gemv_span(const et_op& op, int t, int T) {
    const long long kst = op.i[1] / 16;
    GemvSpan sp;
    if (op.i[13] && !(op.flags & 16)) {
        const long long pairs = static_cast<long long>(op.i[0] / 16) * kst / 2;
        sp.u0 = (static_cast<long long>(t) * pairs / T) * 2;
        sp.u1 = (static_cast<long long>(t + 1) * pairs / T) * 2;
    } else {
        const int align = op.i[7] > 16 ? op.i[7] : 16;
        const long long units = op.i[0] / align;
        sp.u0 = (static_cast<long long>(t) * units / T) * (align / 16) * kst;
        sp.u1 = (static_cast<long long>(t + 1) * units / T) * (align / 16) * kst;
    }
    if (sp.u1 > sp.u0) {
        sp.row0 = static_cast<int>(sp.u0 / kst) * 16;
        sp.rows = static_cast<int>((sp.u1 - 1) / kst + 1) * 16 - sp.row0;
    } else {
        sp.row0 = 0;
        sp.rows = 0;
    }
    return sp;
}

// Attention splits: the s cached positions form ceil(s/CH) blocks of CH; the
// call runs min(blocks, cap) split tasks per kv head (cap = i5, the partials'
// split dimension; at least one with the fused merge) and split c streams blocks
// [c*bps, min(blocks, (c+1)*bps)), bps = ceil(blocks / splits).
struct AttnBlocks {
    long long p0;  // first position
    int nblk;      // blocks (the last one may be partial)
};

// Splits without a batch budget (the mma.sync instantiations' attention).
__device__ __forceinline__ int attn_splits_base(const et_op& op, const long long* binding) {
    const int s = static_cast<int>(binding[op.i[4]]), CH = op.i[2], cap = op.i[5];
    const int nb = (s + CH - 1) / CH;
    return nb < cap ? nb : cap;
}

// Splits of one (sequence, kv head) group: one per CH-position block, at most i5 (the
// partials' split dimension) and, with a per-step budget i11 > 0, at most
// max(1, i11 / b) (b from symbol slot i10): large batches get fewer, longer splits.
__device__ __forceinline__ int attn_tasks(const et_op& op, const long long* binding) {
    const int s = static_cast<int>(binding[op.i[4]]), CH = op.i[2], cap = op.i[5];
    const int nb = (s + CH - 1) / CH;
    int ns = nb < cap ? nb : cap;
    if (op.i[11] > 0) {
        const int b = static_cast<int>(binding[op.i[10]]);
        const int lim = op.i[11] / b > 1 ? op.i[11] / b : 1;
        ns = ns < lim ? ns : lim;
    }
    return ns;
}

// (group, split) of a task: flags bit 7 = flat grid [b * kv * max(splits, 1)] (split count
// depending on the batch), else the 2-D grid [b * kv, splits].
__device__ __forceinline__ void attn_coord(const et_op& op, const int* coord, const long long* binding, int* gi,
                                           int* c) {
    if (op.flags & 128) {
        const int ns0 = attn_tasks(op, binding), ns = ns0 > 1 ? ns0 : 1;
        *gi = coord[0] / ns;
        *c = coord[0] - *gi * ns;
    } else {  // i13 > 1: dim 0 = group * i13 + q-head part (body_attn_split)
        *gi = op.i[13] > 1 ? coord[0] / op.i[13] : coord[0];
        *c = coord[1];
    }
}
// flags bit 9 (tensor-core split body): a group with a single split leaves its 8 warp
// partials unfolded for the merge (which folds up to 8 in registers anyway); with more
// splits each split folds its warps in shared memory.  The partials' split stride is
// then max(i5, 8).
__device__ __forceinline__ bool attn_warp_partials(const et_op& op, const long long* binding) {
    return (op.flags & 512) && attn_tasks(op, binding) <= 1;
}
// Tensor-core split body, fused merge (flags bit 1), q/k fused mode (bit 0: this task
// appends the new k/v) and one split per group: the task finishes the group itself
// (attn_solo_finish) -- no partials, no arrival.  Its new k/v stay in shared memory at
// scratch float kAttnSoloKv (past the eight warps' P transposes, [8][16][9]).
constexpr int kAttnSoloKv = 8 * 16 * 9;
// ... and the Q^T fragments of the split ([8 k steps][32 lanes] x 16 bytes) past the solo
// split's k/v (2 x 128) and weights (2 x 8) -- 16-byte aligned
constexpr int kAttnQFrag = kAttnSoloKv + 2 * 128 + 16;
__device__ __forceinline__ bool attn_solo(const et_op& op, const long long* binding) {
    return (op.flags & 3) == 3 && attn_tasks(op, binding) <= 1;
}
__device__ __forceinline__ int attn_splits_with_data(const et_op& op, const long long* binding) {
    return attn_warp_partials(op, binding) ? 8 : attn_tasks(op, binding);  // empty splits: (m = -inf, l = 0)
}
__device__ __forceinline__ int attn_part_stride(const et_op& op) {
    return (op.flags & 512) && op.i[5] < 8 ? 8 : op.i[5];
}
__device__ __forceinline__ AttnBlocks attn_blocks(const et_op& op, int c, const long long* binding) {
    const int s = static_cast<int>(binding[op.i[4]]), CH = op.i[2];
    const int nb = (s + CH - 1) / CH;
    const int ns = attn_tasks(op, binding);
    AttnBlocks a;
    a.p0 = 0;
    a.nblk = 0;
    if (ns <= 0) return a;
    const int bps = (nb + ns - 1) / ns;
    const int b0 = c * bps, b1 = (c + 1) * bps < nb ? (c + 1) * bps : nb;
    a.p0 = static_cast<long long>(b0) * CH;
    a.nblk = b1 > b0 ? b1 - b0 : 0;
    return a;
}

// Plan for a task of `call` at row-major `flat` with sample coords `coord`.
__device__ __forceinline__ StreamPlan make_plan(const et_op& op, const int* coord, int T, const long long* binding,
                                                int* const* rt) {
    StreamPlan pl;
    pl.nseg = 0;
    pl.cbytes = kStageBytes;
    pl.interleave = false;
    if (op.kind == ET_OP_GEMV_TC) {
        const bool tiled = tc_tiled(op);
        int tj = 0, tt = 0;
        if (tiled) tc_tile(op, coord, &tj, &tt);
        const TcSpan sp = tiled ? tc_span(op, tt, op.i[12]) : tc_span(op, coord[0], T);
        if (sp.nblk <= 0 || sp.np <= 0) {  // idle task: nothing streams
            pl.finish();
            return pl;
        }
        const int nb = tc_batch(op, binding);
        const long long kp = op.i[6], blk_bytes = kp * 256;  // one 128-row block of one piece
        pl.tc_pstride = static_cast<long long>(op.i[0] / 128) * blk_bytes;
        pl.nseg = op.i[2];
        for (int s = 0; s < pl.nseg; ++s)
            pl.base[s] = reinterpret_cast<const uint8_t*>(op.p[s]) + sp.p0 * pl.tc_pstride + sp.b0 * blk_bytes;
        pl.bytes[0] = sp.nblk * blk_bytes;
        pl.tc_w = static_cast<int>(pl.nseg * pl.bytes[0] / kTcChunk);
        pl.tc_np = sp.np;
        pl.tc_pre = pl.tc_w < kStages ? pl.tc_w : kStages;
        pl.tc_xbytes = static_cast<uint32_t>(tc_npad(nb) * kp * 2);
        pl.tc_x = reinterpret_cast<const uint8_t*>(op.p[2]) + static_cast<long long>(sp.p0) * pl.tc_xbytes;
        if (tiled)  // this token block's operand-layout activations (all K pieces of the block)
            pl.tc_x += static_cast<long long>(tj) * (op.i[1] / op.i[6]) * pl.tc_xbytes;
        return pl;
    }
    if (op.kind == ET_OP_GEMV) {
        const bool grouped = (op.flags & 16) != 0;  // coord 0 = group (its own matrix), coord 1 = row span
        const GemvSpan sp = gemv_span(op, grouped ? coord[1] : coord[0], grouped ? op.i[13] : T);
        const long long gofs = grouped ? static_cast<long long>(coord[0]) * op.i[0] * op.i[1] * 2 : 0;
        pl.nseg = op.i[2];
        for (int s = 0; s < pl.nseg; ++s) {
            pl.base[s] = reinterpret_cast<const uint8_t*>(op.p[s]) + gofs + sp.u0 * 512;
            pl.bytes[s] = (sp.u1 - sp.u0) * 512;
        }
    } else if (op.kind == ET_OP_MOE_ROUTE) {
        if (op.flags & 2) {  // logits precomputed by a tensor-core GEMV: nothing streams
            pl.finish();
            return pl;
        }
        const GemvSpan sp = gemv_span(op, coord[0], T);
        pl.nseg = 1;
        pl.base[0] = reinterpret_cast<const uint8_t*>(op.p[0]) + sp.u0 * 512;
        pl.bytes[0] = (sp.u1 - sp.u0) * 512;
    } else if (op.kind == ET_OP_MOE_EXPERT) {
        // gate rows, up rows (rows [r*IR, r*IR+IR) of expert e), then down block (e, r)
        int e, r;
        expert_of(op, coord[0], &e, &r);
        const long long I = op.i[0], H = op.i[1], RS = op.i[2], IR = I / RS;
        const long long rows = IR * H * 2;
        pl.nseg = 3;
        pl.base[0] = reinterpret_cast<const uint8_t*>(op.p[0]) + (e * I + r * IR) * H * 2;
        pl.base[1] = reinterpret_cast<const uint8_t*>(op.p[1]) + (e * I + r * IR) * H * 2;
        pl.base[2] = reinterpret_cast<const uint8_t*>(op.p[2]) + (e * RS + r) * rows;
        pl.bytes[0] = pl.bytes[1] = pl.bytes[2] = rows;
    } else if (op.kind == ET_OP_ATTN_SPLIT) {
        // the split's K/V blocks, interleaved K0 V0 K1 V1 ... (one block per chunk)
        int gi, c;
        attn_coord(op, coord, binding, &gi, &c);
        const AttnBlocks a = attn_blocks(op, c, binding);
        const int dh = op.i[0], CH = op.i[2], cap = op.i[3];
        const long long s = binding[op.i[4]];
        long long p1 = a.p0 + static_cast<long long>(a.nblk) * CH;
        if (p1 > s) p1 = s;
        if (p1 > a.p0) {
            const int kvh = op.i[6], g = gi % kvh, bq = gi / kvh;  // gi = sequence * kv + head
            const long long off = static_cast<long long>(bq) * op.i[8] * 2 + (static_cast<long long>(g) * cap + a.p0) * dh * 2;
            pl.nseg = 2;
            pl.interleave = true;
            pl.cbytes = CH * dh * 2;
            pl.base[0] = reinterpret_cast<const uint8_t*>(op.p[1]) + off;
            pl.base[1] = reinterpret_cast<const uint8_t*>(op.p[2]) + off;
            pl.bytes[0] = pl.bytes[1] = (p1 - a.p0) * dh * 2;
        }
    }
    pl.finish();
    return pl;
}

}  // namespace etk
