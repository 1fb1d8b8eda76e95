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
//   QKV_ROPE (RoPE on q/k pairs, k/v appended to the cache), ADD out += y (red.global.add)
//   i0 = N rows per segment, i1 = K, i2 = segments (1|2), i3 = x mode (0 bf16 [b][K] at p2,
//   1 fp32 residual stream at p2 normalised with RMSNorm gamma p3), i4 = epilogue (GemvEpi),
//   i5 = batch symbol slot (-1: b = 1), i6 = position symbol slot, i7 = row alignment,
//   i8 = head_dim, i9 = x batch stride (elements), i10 = q rows, i11 = kv rows (k and v each),
//   i12 = KV capacity (positions), i13 = split-K (1: even byte spans, EPI_ADD only);
//   p0/p1 = weights (bf16 [N][K], frag16 tile order) of segment 0/1, p4 = out,
//   p5 = residual in (fp32), p6/p7 = K/V cache of the layer (bf16 [kv_heads][cap][head_dim]);
//   p8 = RoPE inverse frequencies (fp32 [head_dim/2], pair j rotates dims 2j, 2j+1); f0 = RMSNorm eps
// ET_OP_ATTN_SPLIT      task (kv_head g, split c): flash-decoding partial over cached
//   positions [c*CH, min(s, c*CH+CH)); i0 = head_dim, i1 = q heads per kv head, i2 = CH,
//   i3 = KV capacity, i4 = position symbol slot, i5 = max splits, i6 = kv heads;
//   p0 = q (fp32 [q_heads*head_dim], RoPE applied), p1/p2 = K/V cache, p3 = partials
//   (fp32 [q_heads][max_splits][head_dim+2]); f0 = softmax scale
// ET_OP_ATTN_MERGE      task (g): merges the splits and the new token at position s
//   (K/V row s of the cache) for the group's q heads; same i/p as ATTN_SPLIT plus
//   p4 = out (bf16 [q_heads*head_dim])
// ET_OP_EMBED           task (0): h[b][:] = float(table[tokens[b]][:]) for every batch row
//   i0 = hidden, i1 = batch symbol slot (-1: 1); p0 = table (bf16 [vocab][hidden]),
//   p1 = token ids (int32 [b]), p2 = out (fp32 [b][hidden])
#pragma once

#include "megakernel.cuh"
#include "ptx.cuh"

namespace etk {

enum GemvEpi { EPI_F32 = 0, EPI_BF16 = 1, EPI_RESID = 2, EPI_SILU_MUL = 3, EPI_QKV_ROPE = 4, EPI_ADD = 5 };

struct Chunk {
    const uint8_t* src;
    uint32_t bytes;
};

// Streaming plan of one task: up to two contiguous byte ranges cut into
// chunks of `cbytes` (<= one ring stage).  GEMV streams segment 0 then
// segment 1; attention interleaves them (K block 0, V block 0, K block 1, ...).
struct StreamPlan {
    const uint8_t* base[2];
    long long bytes[2];
    int nseg;
    int cbytes;
    bool interleave;
    int n[2];  // chunks per segment (set by finish(); keeps divisions off the per-chunk path)

    __device__ void finish() {
        for (int s = 0; s < 2; ++s) n[s] = s < nseg ? static_cast<int>((bytes[s] + cbytes - 1) / cbytes) : 0;
    }
    __device__ int total_chunks() const { return n[0] + n[1]; }
    __device__ Chunk chunk(int idx) const {
        int s = 0;
        if (interleave) {
            s = idx & 1;
            idx >>= 1;
        } else if (idx >= n[0]) {
            s = 1;
            idx -= n[0];
        }
        const long long off = static_cast<long long>(idx) * cbytes;
        const long long rem = bytes[s] - off;
        return Chunk{base[s] + off, static_cast<uint32_t>(rem < cbytes ? rem : cbytes)};
    }
};

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
    if (op.i[13]) {
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

// Plan for a task of `call` at row-major `flat` with sample coords `coord`.
__device__ __forceinline__ StreamPlan make_plan(const et_op& op, const int* coord, int T, const long long* binding) {
    StreamPlan pl;
    pl.nseg = 0;
    pl.cbytes = kStageBytes;
    pl.interleave = false;
    if (op.kind == ET_OP_GEMV) {
        const GemvSpan sp = gemv_span(op, coord[0], T);
        pl.nseg = op.i[2];
        for (int s = 0; s < pl.nseg; ++s) {
            pl.base[s] = reinterpret_cast<const uint8_t*>(op.p[s]) + sp.u0 * 512;
            pl.bytes[s] = (sp.u1 - sp.u0) * 512;
        }
    } else if (op.kind == ET_OP_ATTN_SPLIT) {
        // K rows then V rows of positions [c*CH, min(s, c*CH+CH)), one chunk each
        const int dh = op.i[0], CH = op.i[2], cap = op.i[3];
        const long long s = binding[op.i[4]];
        const long long p0 = static_cast<long long>(coord[1]) * CH;
        const long long p1 = p0 + CH < s ? p0 + CH : s;
        if (p1 > p0) {
            const long long off = (static_cast<long long>(coord[0]) * cap + p0) * dh * 2;
            pl.nseg = 2;
            pl.base[0] = reinterpret_cast<const uint8_t*>(op.p[1]) + off;
            pl.base[1] = reinterpret_cast<const uint8_t*>(op.p[2]) + off;
            pl.bytes[0] = pl.bytes[1] = (p1 - p0) * dh * 2;
        }
    }
    pl.finish();
    return pl;
}

}  // namespace etk
