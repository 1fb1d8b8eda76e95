// Tile bodies executed inside the persistent megakernel, and the streaming
// plans shared by the producer (TMA issuer) and the consumer warps.
//
// et_op parameter layout per kind
// -------------------------------
// ET_OP_SPLITK_PARTIAL  task (row, part): partial[row*parts+part] = sum of data[row][part*L:(part+1)*L]
//   i0 = L, i1 = parts; p0 = data (int32 [n][parts*L]), p1 = partials (int32 [n][parts])
// ET_OP_SPLITK_FINAL    task (row): out[row] = sum_j partials[row*parts+j]
//   i1 = parts; p1 = partials, p2 = out (int32 [n])
// ET_OP_GEMV            task t of T computes rows [r0,r1) of every segment (T = call grid extent)
//   i0 = N rows per segment, i1 = K, i2 = segments (1|2), i3 = x mode (0 bf16 [b][K] at p2,
//   1 fp32 residual stream at p2 normalised with RMSNorm gamma p3), i4 = epilogue (GemvEpi),
//   i5 = batch symbol slot (-1: b = 1), i6 = position symbol slot, i7 = row alignment,
//   i8 = head_dim, i9 = x batch stride (elements), i10 = q rows, i11 = kv rows (k and v each),
//   i12 = KV capacity (positions); p0/p1 = weights (bf16 [N][K]) of segment 0/1, p4 = out,
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

enum GemvEpi { EPI_F32 = 0, EPI_BF16 = 1, EPI_RESID = 2, EPI_SILU_MUL = 3, EPI_QKV_ROPE = 4 };

struct Chunk {
    const uint8_t* src;
    uint32_t bytes;
};

// Streaming plan of one task: up to two contiguous byte ranges, cut into
// ring-stage sized chunks.
struct StreamPlan {
    const uint8_t* base[2];
    long long bytes[2];
    int nseg;

    __device__ int chunks_in(int s) const { return static_cast<int>((bytes[s] + kStageBytes - 1) / kStageBytes); }
    __device__ int total_chunks() const {
        int n = 0;
        for (int s = 0; s < nseg; ++s) n += chunks_in(s);
        return n;
    }
    __device__ Chunk chunk(int idx) const {
        for (int s = 0; s < nseg; ++s) {
            const int n = chunks_in(s);
            if (idx < n) {
                const long long off = static_cast<long long>(idx) * kStageBytes;
                const long long rem = bytes[s] - off;
                return Chunk{base[s] + off, static_cast<uint32_t>(rem < kStageBytes ? rem : kStageBytes)};
            }
            idx -= n;
        }
        return Chunk{nullptr, 0};
    }
};

__device__ __forceinline__ void gemv_rows(const et_op& op, int t, int T, int* r0, int* r1) {
    const int align = op.i[7] > 0 ? op.i[7] : 1;
    const long long units = op.i[0] / align;
    *r0 = static_cast<int>((static_cast<long long>(t) * units) / T) * align;
    *r1 = static_cast<int>((static_cast<long long>(t + 1) * units) / T) * align;
}

// Plan for a task of `call` at row-major `flat` with sample coords `coord`.
__device__ __forceinline__ StreamPlan make_plan(const et_op& op, const int* coord, int T, const long long* binding) {
    StreamPlan pl;
    pl.nseg = 0;
    if (op.kind == ET_OP_GEMV) {
        int r0, r1;
        gemv_rows(op, coord[0], T, &r0, &r1);
        const long long K = op.i[1];
        pl.nseg = op.i[2];
        for (int s = 0; s < pl.nseg; ++s) {
            pl.base[s] = reinterpret_cast<const uint8_t*>(op.p[s]) + static_cast<long long>(r0) * K * 2;
            pl.bytes[s] = static_cast<long long>(r1 - r0) * K * 2;
        }
    } else if (op.kind == ET_OP_ATTN_SPLIT) {
        const int dh = op.i[0], CH = op.i[2], cap = op.i[3];
        const long long s = binding[op.i[4]];
        const int g = coord[0], c = coord[1];
        const long long p0 = static_cast<long long>(c) * CH;
        long long p1 = p0 + CH;
        if (p1 > s) p1 = s;
        if (p1 > p0) {
            const long long off = (static_cast<long long>(g) * cap + p0) * dh * 2;
            pl.nseg = 2;
            pl.base[0] = reinterpret_cast<const uint8_t*>(op.p[1]) + off;
            pl.base[1] = reinterpret_cast<const uint8_t*>(op.p[2]) + off;
            pl.bytes[0] = pl.bytes[1] = (p1 - p0) * dh * 2;
        }
    }
    return pl;
}

}  // namespace etk
