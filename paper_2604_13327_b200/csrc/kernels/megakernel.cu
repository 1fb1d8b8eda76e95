// The persistent Event Tensor megakernel (static scheduler).
//
// One CTA per queue (== per SM).  Warp roles inside a CTA:
//   warps 0..7   consumers: walk the CTA's queue slot by slot doing
//                WAIT* (spin on Event Tensor elements, acquire) -> EXEC (tile body)
//                -> NOTIFY* (release increment), i.e. the instruction sequence of
//                ref sched_static.hpp:13-20 executed as in ref simulate.cpp:183-269;
//   warp 8       producer: walks the same queue ahead of the consumers and streams
//                each task's weights / KV blocks into a 10-stage shared-memory ring
//                with 1-D TMA bulk copies (mbarrier transaction counts).  It never
//                waits on Event Tensors, so weight streaming for the next tasks
//                overlaps the consumers' dependency waits -- the paper's weight
//                prefetch pass (ref simulate.cpp:205-216 models it as PREFETCH
//                overlapping WAIT);
//   warp 9       executes the DMA-class queue (worker 0 only).
//
// Event Tensor elements are stored as "notifies received this step" and
// compared against the element's initial count; the reference's counter value
// is initial - received.  Two buffers alternate between steps; each launch
// zeroes the buffer the next launch will use, so no extra reset launch exists.
// Masking (ref sched_static.cpp:162-171 and simulate.cpp:199-202) is evaluated
// on the device from the binding passed as kernel arguments.
#include <cuda_runtime.h>

#include "megakernel.cuh"
#include "ops.cuh"

#ifndef ET_ATTN_QLO
#define ET_ATTN_QLO 1
#endif
#ifndef ET_ATTN_PLO
#define ET_ATTN_PLO 1
#endif

namespace etk {

__device__ __forceinline__ uint8_t* smem_cta_base() {
    extern __shared__ __align__(1024) uint8_t smem_all[];
    return smem_all;
}
struct SlotInfo {
    int call;
    int rank;
    int coord[kMaxRank];
    int ext0;  // sample extent of dim 0 (GEMV task count)
    bool masked;
    bool lazy;
};

__device__ __forceinline__ long long eval_code(const StaticParams& P, int call, int d) {
    const int b = __ldg(P.grid_code_off + call * 4 + d);
    const int e = __ldg(P.grid_code_off + call * 4 + d + 1);
    long long st[12];
    int sp = 0;
    for (int i = b; i < e; ++i) {
        const int op = __ldg(P.code_op + i);
        const long long a = __ldg(P.code_arg + i);
        if (op == 0) {
            st[sp++] = a;
        } else if (op == 1) {
            st[sp++] = P.binding[a];
        } else {
            const long long y = st[--sp];
            const long long x = st[sp - 1];
            long long r;
            switch (op) {
                case 2: r = x + y; break;
                case 3: r = x * y; break;
                case 4: r = y ? x / y : 0; break;
                case 5: r = y ? x % y : 0; break;
                case 6: r = x < y ? x : y; break;
                default: r = x > y ? x : y; break;
            }
            st[sp - 1] = r;
        }
    }
    return sp ? st[0] : 0;
}

__device__ __forceinline__ SlotInfo slot_info(const StaticParams& P, int s) {
    SlotInfo si;
    si.call = __ldg(P.slot_call + s);
    si.rank = __ldg(P.call_rank + si.call);
    int flat = __ldg(P.slot_flat + s);
    int sext[kMaxRank];
    for (int d = 0; d < kMaxRank; ++d) sext[d] = d < si.rank ? __ldg(P.call_extents + si.call * 4 + d) : 1;
    si.ext0 = sext[0];
    for (int d = si.rank - 1; d >= 0; --d) {
        si.coord[d] = flat % sext[d];
        flat /= sext[d];
    }
    si.masked = false;
    for (int d = 0; d < si.rank; ++d)
        if (si.coord[d] >= eval_code(P, si.call, d)) si.masked = true;
    si.lazy = __ldg(P.call_extent_from + si.call) >= 0;
    return si;
}

// extent_from masking (ref simulate.cpp:199-202): tasks whose row-major index
// in the actual grid is at or beyond the realized count are no-ops.  Only
// valid once the writer of the indptr tensor has finished (after the waits).
__device__ bool extent_masked(const StaticParams& P, int call, const int* coord) {
    const int ef = __ldg(P.call_extent_from + call);
    if (ef < 0 || P.rt_len[ef] <= 0) return false;
    const int rank = __ldg(P.call_rank + call);
    long long aflat = 0;
    for (int d = 0; d < rank; ++d) aflat = aflat * eval_code(P, call, d) + coord[d];
    return aflat >= static_cast<long long>(__ldcg(P.rt[ef] + P.rt_len[ef] - 1));
}

__device__ __forceinline__ void report(DevStatus* st, int code, int worker, int slot, int counter, int value) {
    if (atomicCAS(&st->code, 0, code) == 0) {
        st->worker = worker;
        st->slot = slot;
        st->counter = counter;
        st->value = value;
    }
}

__device__ __forceinline__ bool aborted(const DevStatus* st) {
    return *reinterpret_cast<const volatile int*>(&st->code) != 0;
}

// Status blocks alternate between launches (each launch prepares the other one
// for the next).  Errors are sticky until the host collects them (et_sync): a
// launch that finds its own block already failed (an earlier asynchronous step
// went wrong) copies the error forward and does nothing, and a launch never
// clears a block that holds an error.  Returns true when this launch must exit.
__device__ __forceinline__ bool sticky_status(const StaticParams& P) {
    const bool failed = aborted(P.status);
    if (blockIdx.x == 0 && threadIdx.x < sizeof(DevStatus) / 4) {
        int* other = reinterpret_cast<int*>(P.status_other);
        if (failed) other[threadIdx.x] = reinterpret_cast<const int*>(P.status)[threadIdx.x];
        else if (!aborted(P.status_other)) other[threadIdx.x] = 0;
    }
    return failed;
}

// Spin until every wait element in [b, e) has received its initial count.
// Acquire loads: the producer's data written before its release increment is
// visible to this thread, and to the rest of the CTA after the barrier that
// follows (PTX causality order through bar.sync).
// Acquire polls (debug bit 0x10000: relaxed polls and one acquire fence at the
// end -- measured slower: the fence's MEMBAR sits on the critical path).
__device__ bool wait_range(const StaticParams& P, int b, int e, int s, int worker) {
    const bool relaxed = (P.debug & 0x10000) != 0;
    for (int w = b; w < e; ++w) {
        const int el = __ldg(P.waits + w);
        const uint32_t need = static_cast<uint32_t>(__ldg(P.initial_counts + el));
        uint32_t v = relaxed ? ld_relaxed(P.cnt + el) : ld_acquire(P.cnt + el);
        if (v >= need) continue;
        const uint64_t t0 = globaltimer();
        uint32_t it = 0;
        while ((v = relaxed ? ld_relaxed(P.cnt + el) : ld_acquire(P.cnt + el)) < need) {
            if ((++it & 255u) == 0) {
                if (aborted(P.status)) return false;
                if (globaltimer() - t0 > static_cast<uint64_t>(P.watchdog_ns)) {
                    report(P.status, ET_ERR_DEADLOCK, worker, s, el, static_cast<int>(need - v));
                    return false;
                }
            }
        }
    }
    if (relaxed && e > b) fence_acquire_gpu();
    return true;
}

// Release increments: the consumer warps' writes precede this thread's
// release through the barrier the caller executed just before.
// `first` (>= 0): the element of notify b, read before the slot's waits (the
// wait's acquire invalidates L1, so reading it here would add a round trip).
__device__ bool notify_range(const StaticParams& P, int b, int e, int s, int worker, int first = -1) {
    bool ok = true;
    for (int n = b; n < e; ++n) {
        const int el = (n == b && first >= 0) ? first : __ldg(P.notifies + n);
        const uint32_t old = atom_add_release(P.cnt + el, 1u);
        if (old >= static_cast<uint32_t>(__ldg(P.initial_counts + el))) {
            report(P.status, ET_ERR_UNDERFLOW, worker, s, el, -1);
            ok = false;
        }
    }
    return ok;
}

__device__ __forceinline__ bool wait_slot(const StaticParams& P, int s, int worker) {
    return wait_range(P, __ldg(P.wait_off + s), __ldg(P.wait_off + s + 1), s, worker);
}
__device__ __forceinline__ bool notify_slot(const StaticParams& P, int s, int worker) {
    return notify_range(P, __ldg(P.notify_off + s), __ldg(P.notify_off + s + 1), s, worker);
}

// ---------------------------------------------------------------------------
// Per-CTA slot table in shared memory, filled once per launch: the task loop
// then needs no dependent global loads to find a slot's call, coordinates,
// mask and wait/notify ranges.  Entry = {call | masked<<31 | lazy<<30,
// c0 | c1<<16, wait_off, notify_off}; a sentinel entry closes the ranges.
struct SlotTable {
    const uint4* ent;
    const int* ext0;
    bool valid;
};

struct SlotView {
    int call;
    bool masked;
    bool lazy;  // extent_from call: mask known only after the waits
    int coord[kMaxRank];
    int ext0;
    int wb, we, nb, ne;
};

__device__ __forceinline__ SlotView view_slot(const StaticParams& P, const SlotTable& T, int s, int qb) {
    SlotView v;
    if (T.valid) {
        const uint4 a = T.ent[s - qb];
        const uint4 b = T.ent[s - qb + 1];
        v.call = static_cast<int>(a.x & 0x3fffffffu);
        v.masked = (a.x >> 31) != 0;
        v.lazy = ((a.x >> 30) & 1u) != 0;
        v.coord[0] = static_cast<int>(a.y & 0xffffu);
        v.coord[1] = static_cast<int>(a.y >> 16);
        v.coord[2] = v.coord[3] = 0;
        v.ext0 = T.ext0[v.call];
        v.wb = static_cast<int>(a.z);
        v.we = static_cast<int>(b.z);
        v.nb = static_cast<int>(a.w);
        v.ne = static_cast<int>(b.w);
    } else {
        const SlotInfo si = slot_info(P, s);
        v.call = si.call;
        v.masked = si.masked;
        v.lazy = si.lazy;
        for (int d = 0; d < kMaxRank; ++d) v.coord[d] = si.coord[d];
        v.ext0 = si.ext0;
        v.wb = __ldg(P.wait_off + s);
        v.we = __ldg(P.wait_off + s + 1);
        v.nb = __ldg(P.notify_off + s);
        v.ne = __ldg(P.notify_off + s + 1);
    }
    return v;
}

// ---------------------------------------------------------------------------
// Ring protocol.  The producer fills stages in chunk-sequence order c = 0, 1,
// 2, ... (stage c % kStages, parity (c / kStages) & 1).  Chunk c is owned by
// consumer warp c % kConsumerWarps (== its stage): the owner waits for it and
// releases the stage with one arrive, so each warp has its own stage in flight
// while it computes on another (see kStages).  Every consumer thread tracks the
// same 64-bit sequence number.
struct Ring {
    uint8_t* buf;
    uint64_t* full;
    uint64_t* empty;
    unsigned long long seq;  // sequence number of the next chunk to consume
    DevStatus* status;
    long long watchdog_ns;
    int worker;
    unsigned long long stall = 0;  // ns spent waiting for filled stages (ET_DEBUG bit 2)
    bool dbg = false;
    unsigned long long busy = 0;   // ns between a stage's arrival and its release (ET_DEBUG bit 8)
    unsigned long long xwait = 0;  // tensor-core GEMV: ns the issuer waited for activation pieces
    uint64_t t_ret = 0;

    __device__ __forceinline__ static int stage_of(unsigned long long c) { return static_cast<int>(c % kStages); }
    __device__ __forceinline__ static uint32_t parity_of(unsigned long long c) {
        return static_cast<uint32_t>((c / kStages) & 1ull);
    }
    __device__ __forceinline__ static int owner(unsigned long long c) { return static_cast<int>(c % kConsumerWarps); }
    // Bounded wait: a stage that never fills (protocol bug, aborted producer)
    // reports a deadlock instead of hanging the device.  Returns nullptr then.
    __device__ __forceinline__ const uint8_t* wait(unsigned long long c) {
        const int st = stage_of(c);
        const uint32_t par = parity_of(c);
        const uint64_t t00 = dbg ? globaltimer() : 0;
        if (!mbar_try_wait(&full[st], par)) {
            const uint64_t t0 = globaltimer();
            uint32_t it = 0;
            while (!mbar_try_wait(&full[st], par)) {
                if ((++it & 1023u) == 0) {
                    if (aborted(status)) return nullptr;
                    if (globaltimer() - t0 > static_cast<uint64_t>(watchdog_ns)) {
                        report(status, ET_ERR_DEADLOCK, worker, -1, -2, static_cast<int>(c & 0x7fffffff));
                        return nullptr;
                    }
                }
            }
        }
        if (dbg) {
            const uint64_t now = globaltimer();
            stall += now - t00;
            t_ret = now;
        }
        return buf + st * kStageBytes;
    }
    __device__ __forceinline__ void release(unsigned long long c) {
        if (dbg) busy += globaltimer() - t_ret;
        mbar_arrive(&empty[stage_of(c)]);
    }
};

__device__ __forceinline__ int batch_of(const et_op& op, const StaticParams& P) {
    return op.i[5] >= 0 ? static_cast<int>(P.binding[op.i[5]]) : 1;
}

// A GEMV task's staged activations and accumulators must fit shared memory.
__device__ __forceinline__ bool gemv_fits(const et_op& op, const StaticParams& P) {
    const int nb = batch_of(op, P);
    return nb <= kMaxBatch && nb * op.i[1] * 2 <= kXBytes;
}

// ---------------------------------------------------------------------------
// Tile bodies.  `ctid` in [0, kConsumers); bar id 1 syncs the consumer warps.

__device__ void body_splitk(const StaticParams& P, const et_op& op, const int* coord, int ctid) {
    if (op.kind == ET_OP_SPLITK_PARTIAL) {
        const int L = op.i[0], parts = op.i[1];
        const int row = coord[0], part = coord[1];
        const int* data = reinterpret_cast<const int*>(op.p[0]) + (static_cast<long long>(row) * parts + part) * L;
        int acc = 0;
        for (int i = ctid; i < L; i += kConsumers) acc += __ldcg(data + i);
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        __shared__ int red[kConsumerWarps];
        if ((ctid & 31) == 0) red[ctid >> 5] = acc;
        bar_sync(1, kConsumers);
        if (ctid == 0) {
            int t = 0;
            for (int w = 0; w < kConsumerWarps; ++w) t += red[w];
            reinterpret_cast<int*>(op.p[1])[row * parts + part] = t;
        }
    } else {
        const int parts = op.i[1];
        const int row = coord[0];
        if (ctid == 0) {
            const int* part = reinterpret_cast<const int*>(op.p[1]) + row * parts;
            int t = 0;
            for (int j = 0; j < parts; ++j) t += __ldcg(part + j);
            reinterpret_cast<int*>(op.p[2])[row] = t;
        }
    }
}

// RMSNorm gamma of a GEMV is staged in shared memory right after the bf16
// activations (16-byte aligned) when both fit.
__device__ __forceinline__ int gamma_offset(const et_op& op, const StaticParams& P) {
    return ((batch_of(op, P) * op.i[1] + 7) / 8) * 8;  // in bf16 elements
}
__device__ __forceinline__ bool gemv_gamma_staged(const et_op& op, const StaticParams& P) {
    return op.i[3] == 1 && (gamma_offset(op, P) * 2 + op.i[1] * 4) <= kXBytes;
}

// ---- GEMV main loop (tensor cores).  Weights sit in HBM as m16n8k16
// A-fragment tiles (decode.py `frag16`): tile (t, j) = rows [16t, 16t+16) x
// k-step j is 512 B = 32 lanes x 16 B, lane (g = lane/4, q = lane%4) holding
// its a0..a3.  Inside every 32-wide k block the k order is permuted so that the
// B fragment of lane (g, q) for the k-step pair (2p, 2p+1) is the 16 contiguous
// bytes x[g][32p + 8q, 32p + 8q + 8): one LDS.128 of the activations per two
// MMAs, and one LDS.128 of weights per MMA.  Batch rows are the mma N dimension
// (nb <= 8; x is bf16 [nb][K] in shared memory).  A task's span is a
// contiguous byte range of the tiled matrix (per segment), streamed through the
// ring; each consumer warp owns whole chunks (chunk c -> warp c % 8) and hands
// the 16-row x 8-column partial tile to `flush(seg, row_tile, g, q, d[4])` at
// every row-tile change (d[0] = D[g][2q], d[1] = D[g][2q+1], d[2] = D[g+8][2q],
// d[3] = D[g+8][2q+1]; row tiles count from the span's first tile).
template <typename Flush>
__device__ __forceinline__ void gemv_stream(Ring& ring, int warp, int lane, int nseg, int seg_tiles, int u0, int K,
                                            int nb, const uint16_t* xs, Flush&& flush) {
    const int kst = K / 16;                              // k-steps per row tile (even)
    constexpr int kTilesPerChunk = kStageBytes / 512;    // 40 (even)
    const int g = lane >> 2, q = lane & 3;
    const bool xlane = g < nb;
    const uint16_t* xrow = xs + (xlane ? g : 0) * K + 8 * q;
    const int nch = (seg_tiles + kTilesPerChunk - 1) / kTilesPerChunk;
    const int total = nseg * nch;
    const unsigned long long c0 = ring.seq;
    // this warp's chunks only (c % 8 == warp): no walk over the other warps' chunks
    for (int idx = (warp - static_cast<int>(c0 % kConsumerWarps) + kConsumerWarps) % kConsumerWarps; idx < total;
         idx += kConsumerWarps) {
        const unsigned long long c = c0 + idx;
        const int seg = idx / nch, ch = idx - seg * nch;
        const uint8_t* buf = ring.wait(c);
        if (!buf) continue;  // aborted: the step reports an error
        const int t0 = ch * kTilesPerChunk;
        const int nt = seg_tiles - t0 < kTilesPerChunk ? seg_tiles - t0 : kTilesPerChunk;
        const int tt0 = u0 + t0;  // unit index relative to the span's first tile
        int rtile = tt0 / kst, j = tt0 - rtile * kst;
        int done = 0;
        while (done < nt) {
            const int len = (kst - j < nt - done) ? kst - j : nt - done;
            float d0[4] = {0.f, 0.f, 0.f, 0.f}, d1[4] = {0.f, 0.f, 0.f, 0.f};
            const uint4* ap = reinterpret_cast<const uint4*>(buf + done * 512) + lane;
            const uint16_t* xp = xrow + j * 16;
#pragma unroll 4
            for (int i = 0; i < len; i += 2) {
                const uint4 a0 = lds128(ap + i * 32);
                const uint4 a1 = lds128(ap + (i + 1) * 32);
                const uint4 xv = xlane ? lds128(xp + i * 16) : make_uint4(0u, 0u, 0u, 0u);
                mma_bf16_16816(d0, a0, xv.x, xv.y);
                mma_bf16_16816(d1, a1, xv.z, xv.w);
            }
            const float d[4] = {d0[0] + d1[0], d0[1] + d1[1], d0[2] + d1[2], d0[3] + d1[3]};
            flush(seg, rtile, g, q, d);
            done += len;
            ++rtile;  // the next unit (if any) starts the next row tile
            j = 0;
        }
        __syncwarp();
        if (lane == 0) ring.release(c);
    }
    ring.seq = c0 + total;
}

// Shared-memory mbarrier of the attention-merge prologue's bulk loads (behind the
// tensor-core barriers in the misc area); its phase count is misc[13].
__device__ __forceinline__ uint64_t* merge_bar(uint8_t* smem) {
    return reinterpret_cast<uint64_t*>(smem + kSmemMisc + 464);
}
// Stage `bytes` (16-byte multiple and alignment) of data produced by other CTAs
// (acquired by this task's wait) at smem dst with one bulk copy; every consumer
// thread returns once it landed.  dst must not be read or written by anyone
// else meanwhile (the caller's previous generic accesses are ordered by its last
// consumer barrier).
// The barrier's phase count misc[13] advances once per use, after a consumer
// barrier; the next use is a later task's prologue (further barriers apart).
__device__ __forceinline__ void stage_bulk(const StaticParams&, void* dst, const void* src, uint32_t bytes, int ctid) {
    uint64_t* bar = merge_bar(smem_cta_base());
    volatile int* misc = reinterpret_cast<volatile int*>(smem_cta_base() + kSmemMisc);
    const uint32_t par = static_cast<uint32_t>(misc[13]) & 1u;
    if (ctid == 0) {
        fence_proxy_async_global();
        fence_proxy_async();
        mbar_arrive_expect_tx(bar, bytes);
        bulk_g2s_keep(dst, src, bytes, bar);
    }
    mbar_wait(bar, par);
    bar_sync(1, kConsumers);  // everyone saw this phase before it is reused
    if (ctid == 0) misc[13] = misc[13] + 1;
}

constexpr int kMergeBulkOff = 2048;                      // partials staged at xs + 2 KB ...
constexpr int kMergeBulkMax = kXBytes + kAccFloats * 4 - kMergeBulkOff - 2048;  // ... up to acc's last 2 KB

// Attention-merge prologue of a GEMV (x mode 2, b = 1): activation slice g is the
// merge of kv group g's attention splits, whose unnormalised partials (m, l, o)
// per q head the splits left in p2 (fp32 [heads][i10][kPartHead + dh]; ATTN_SPLIT flags
// bit 10):  x = sum_c e^(m_c - M) o_c / sum_c e^(m_c - M) l_c  (M = max_c m_c),
// so the attention needs no merge task and its consumer no second hop.
// i6 = position slot, i8 = head_dim, i10 = split stride, i11 = CH, i12 = split cap.
// p5 (optional): the group's raw split-K q/k/v accumulators (fp32: q [i9 * G * dh],
// k, v [i9 * dh]; i9 = kv heads), consumed by now -- task t of the group's i13
// zeroes its share for the next step (the splits that read them all arrived).
// kOut outputs per thread (K <= 256 * kOut), kPass splits per batch of loads.
// Out of line: its loads in flight would otherwise crowd the GEMV loop's registers.
template <int kOut, int kPass>
__device__ __noinline__ void gemv_merge_prologue(const StaticParams& P, const et_op& op, int gsel, int tsel,
                                                 uint16_t* xs, float* acc, int ctid, uint64_t* t_probe) {
    const int warp = ctid >> 5, lane = ctid & 31;
    const int K = op.i[1];
    if (op.p[5]) {
        const int dh = op.i[8], G = K / dh, nkv = op.i[9] * dh, nq = op.i[9] * G * dh;
        const int n = G * dh + 2 * dh, per = (n + op.i[13] - 1) / op.i[13];
        float* raw = reinterpret_cast<float*>(op.p[5]);
        for (int i = tsel * per + ctid; i < (tsel + 1) * per && i < n; i += kConsumers) {
            const int off = i < G * dh ? gsel * G * dh + i
                            : i < G * dh + dh ? nq + gsel * dh + (i - G * dh) : nq + nkv + gsel * dh + (i - G * dh - dh);
            raw[off] = 0.f;
        }
    }

    const int dh = op.i[8], G = K / dh, maxs = op.i[10], CH = op.i[11];
    const long long s = P.binding[op.i[6]];
    long long nsl = (s + CH - 1) / CH;
    if (nsl > op.i[12]) nsl = op.i[12];
    const int ns = nsl > 0 ? static_cast<int>(nsl) : 1;
    const float* part = reinterpret_cast<const float*>(op.p[2]) +
                        static_cast<long long>(gsel) * G * maxs * (dh + kPartHead);
    const int row = dh + kPartHead;
    const uint32_t hbytes = static_cast<uint32_t>(ns) * row * 4;  // one head's used splits, contiguous
    if (G * hbytes <= static_cast<uint32_t>(kMergeBulkMax) && 3 * G * ns <= 512) {
        // Bulk path: the group's partials reach shared memory by G bulk copies (the TMA
        // engine keeps far more bytes in flight than 256 threads' loads: 33 KB take one
        // L2 round trip instead of ~3 us of load-slot-limited requests).
        float* ps = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(xs) + kMergeBulkOff);  // [G][ns][row]
        float* ml = acc + kAccFloats - 512;  // [G][ns][2]
        float* wts = ml + 2 * G * ns;        // [G][ns]
        volatile int* misc = reinterpret_cast<volatile int*>(reinterpret_cast<uint8_t*>(xs) - kSmemX + kSmemMisc);
        uint64_t* bar = merge_bar(reinterpret_cast<uint8_t*>(xs) - kSmemX);
        const uint32_t par = static_cast<uint32_t>(misc[13]) & 1u;
        if (ctid == 0) {
            fence_proxy_async_global();  // partials: generic stores of other CTAs, acquired by the wait
            fence_proxy_async();         // xs was last written through the generic proxy
            mbar_arrive_expect_tx(bar, G * hbytes);
            for (int h = 0; h < G; ++h)
                bulk_g2s_keep(ps + h * ns * row, part + static_cast<long long>(h) * maxs * row, hbytes, bar);
        }
        mbar_wait(bar, par);
        if ((P.debug & 0x1000) && ctid == 0) *t_probe = globaltimer();  // partials staged
        for (int i = ctid; i < G * ns; i += kConsumers) {
            ml[2 * i] = ps[i * row];
            ml[2 * i + 1] = ps[i * row + 1];
        }
        bar_sync(1, kConsumers);
        for (int hh = warp; hh < G; hh += kConsumerWarps) {
            float M = -INFINITY;
            for (int c = lane; c < ns; c += 32) M = fmaxf(M, ml[2 * (hh * ns + c)]);
            M = warp_max(M);
            float L = 0.f;
            for (int c = lane; c < ns; c += 32) {
                const float e = __expf(ml[2 * (hh * ns + c)] - M);
                wts[hh * ns + c] = e;
                L += e * ml[2 * (hh * ns + c) + 1];
            }
            const float inv = 1.f / warp_sum(L);
            __syncwarp();
            for (int c = lane; c < ns; c += 32) wts[hh * ns + c] *= inv;
        }
        bar_sync(1, kConsumers);
        if ((P.debug & 0x4000) && ctid == 0) *t_probe = globaltimer();  // weights
        for (int idx = ctid; idx < K; idx += kConsumers) {
            const int hh = idx / dh, d = idx - hh * dh;
            const float* w = wts + hh * ns;
            const float* pc = ps + hh * ns * row + kPartHead + d;
            float o = 0.f, o2 = 0.f;
            int c = 0;
            for (; c + 1 < ns; c += 2) {
                o = fmaf(w[c], pc[c * row], o);
                o2 = fmaf(w[c + 1], pc[(c + 1) * row], o2);
            }
            if (c < ns) o = fmaf(w[c], pc[c * row], o);
            xs[idx] = f2bf(o + o2);
        }
        bar_sync(1, kConsumers);  // ps / ml / wts are done with (acc is zeroed by the caller)
        if (ctid == 0) misc[13] = misc[13] + 1;
        return;
    }
    // more splits than the staging area holds: the same, in rounds of nsr splits
    const int nsr = static_cast<int>(kMergeBulkMax / (static_cast<uint32_t>(G) * row * 4));  // splits per round
    if (nsr >= 1 && 3 * G * ns <= 512) {
        // (m, l) of every split load directly while round 0 lands
        float* ps = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(xs) + kMergeBulkOff);  // [G][round][row]
        float* ml = acc + kAccFloats - 512;  // [G][ns][2]
        float* wts = ml + 2 * G * ns;        // [G][ns]
        volatile int* misc = reinterpret_cast<volatile int*>(reinterpret_cast<uint8_t*>(xs) - kSmemX + kSmemMisc);
        uint64_t* bar = merge_bar(reinterpret_cast<uint8_t*>(xs) - kSmemX);
        const uint32_t ph0 = static_cast<uint32_t>(misc[13]);
        const int rounds = (ns + nsr - 1) / nsr;
        auto issue = [&](int c0) {  // thread 0: splits [c0, c0 + cnt) of every head
            const int cnt = ns - c0 < nsr ? ns - c0 : nsr;
            const uint32_t rb = static_cast<uint32_t>(cnt) * row * 4;
            mbar_arrive_expect_tx(bar, G * rb);
            for (int h = 0; h < G; ++h)
                bulk_g2s_keep(ps + h * cnt * row, part + (static_cast<long long>(h) * maxs + c0) * row, rb, bar);
        };
        if (ctid == 0) {
            fence_proxy_async_global();  // partials: generic stores of other CTAs, acquired by the wait
            fence_proxy_async();         // xs was last written through the generic proxy
            issue(0);
        }
        for (int i = ctid; i < G * ns; i += kConsumers) {
            const float* pr = part + (static_cast<long long>(i / ns) * maxs + i % ns) * row;
            ml[2 * i] = __ldcg(pr);
            ml[2 * i + 1] = __ldcg(pr + 1);
        }
        bar_sync(1, kConsumers);
        for (int hh = warp; hh < G; hh += kConsumerWarps) {
            float M = -INFINITY;
            for (int c = lane; c < ns; c += 32) M = fmaxf(M, ml[2 * (hh * ns + c)]);
            M = warp_max(M);
            float L = 0.f;
            for (int c = lane; c < ns; c += 32) {
                const float e = __expf(ml[2 * (hh * ns + c)] - M);
                wts[hh * ns + c] = e;
                L += e * ml[2 * (hh * ns + c) + 1];
            }
            const float inv = 1.f / warp_sum(L);
            __syncwarp();
            for (int c = lane; c < ns; c += 32) wts[hh * ns + c] *= inv;
        }
        bar_sync(1, kConsumers);
        if ((P.debug & 0x4000) && ctid == 0) *t_probe = globaltimer();  // weights
        float o[kOut], o2[kOut];
#pragma unroll
        for (int j = 0; j < kOut; ++j) o[j] = o2[j] = 0.f;
        for (int r = 0; r < rounds; ++r) {
            const int c0 = r * nsr, cnt = ns - c0 < nsr ? ns - c0 : nsr;
            if (r > 0 && ctid == 0) issue(c0);  // the previous round's readers passed the barrier below
            mbar_wait(bar, (ph0 + static_cast<uint32_t>(r)) & 1u);
            if (r == 0 && (P.debug & 0x1000) && ctid == 0) *t_probe = globaltimer();  // partials staged
#pragma unroll
            for (int j = 0; j < kOut; ++j) {
                const int idx = ctid + j * kConsumers;
                if (idx < K) {
                    const int hh = idx / dh, d = idx - hh * dh;
                    const float* w = wts + hh * ns + c0;
                    const float* pc = ps + hh * cnt * row + kPartHead + d;
                    int c = 0;
                    for (; c + 1 < cnt; c += 2) {
                        o[j] = fmaf(w[c], pc[c * row], o[j]);
                        o2[j] = fmaf(w[c + 1], pc[(c + 1) * row], o2[j]);
                    }
                    if (c < cnt) o[j] = fmaf(w[c], pc[c * row], o[j]);
                }
            }
            bar_sync(1, kConsumers);  // ps is free for the next round (and ml / wts after the last)
        }
#pragma unroll
        for (int j = 0; j < kOut; ++j) {
            const int idx = ctid + j * kConsumers;
            if (idx < K) xs[idx] = f2bf(o[j] + o2[j]);
        }
        if (ctid == 0) misc[13] = static_cast<int>(ph0) + rounds;
        bar_sync(1, kConsumers);  // xs complete (acc is zeroed by the caller)
        return;
    }
    float* ml = acc;              // [G][ns][2] (acc is zeroed after the prologue)
    float* wts = acc + 2 * G * ns;  // [G][ns]
    float ov[kOut][kPass];
#pragma unroll
    for (int j = 0; j < kOut; ++j) {
        const int idx = ctid + j * kConsumers;
        const int hh = idx / dh, d = idx - hh * dh;
#pragma unroll
        for (int c = 0; c < kPass; ++c)
            ov[j][c] = (idx < K && c < ns) ? __ldcg(part + (static_cast<long long>(hh) * maxs + c) * (dh + kPartHead) + kPartHead + d)
                                           : 0.f;
    }
    for (int i = ctid; i < G * ns; i += kConsumers) {
        const float* pr = part + (static_cast<long long>(i / ns) * maxs + i % ns) * (dh + kPartHead);
        ml[2 * i] = __ldcg(pr);
        ml[2 * i + 1] = __ldcg(pr + 1);
    }
    if ((P.debug & 0x1000) && ctid == 0) *t_probe = globaltimer() + (ov[0][0] == 1234.5f ? 1 : 0);  // loads landed
    bar_sync(1, kConsumers);
    if ((P.debug & 0x2000) && ctid == 0) *t_probe = globaltimer();  // every thread's loads landed
    for (int hh = warp; hh < G; hh += kConsumerWarps) {
        float M = -INFINITY;
        for (int c = lane; c < ns; c += 32) M = fmaxf(M, ml[2 * (hh * ns + c)]);
        M = warp_max(M);
        float L = 0.f;
        for (int c = lane; c < ns; c += 32) {
            const float e = __expf(ml[2 * (hh * ns + c)] - M);
            wts[hh * ns + c] = e;
            L += e * ml[2 * (hh * ns + c) + 1];
        }
        const float inv = 1.f / warp_sum(L);
        __syncwarp();
        for (int c = lane; c < ns; c += 32) wts[hh * ns + c] *= inv;
    }
    bar_sync(1, kConsumers);
    if ((P.debug & 0x4000) && ctid == 0) *t_probe = globaltimer();  // weights
#pragma unroll
    for (int j = 0; j < kOut; ++j) {
        const int idx = ctid + j * kConsumers;
        if (idx < K) {
            const int hh = idx / dh, d = idx - hh * dh;
            const float* w = wts + hh * ns;
            float o = 0.f, o2 = 0.f;
#pragma unroll
            for (int c = 0; c < kPass; c += 2) {
                if (c < ns) o = fmaf(w[c], ov[j][c], o);
                if (c + 1 < ns) o2 = fmaf(w[c + 1], ov[j][c + 1], o2);
            }
            for (int c0 = kPass; c0 < ns; c0 += kPass) {  // further splits, one batch of loads at a time
                float pv[kPass];
#pragma unroll
                for (int u = 0; u < kPass; ++u)
                    pv[u] = c0 + u < ns ? __ldcg(part + (static_cast<long long>(hh) * maxs + c0 + u) * (dh + kPartHead) + kPartHead + d)
                                        : 0.f;
#pragma unroll
                for (int u = 0; u < kPass; ++u)
                    if (c0 + u < ns) o = fmaf(w[c0 + u], pv[u], o);
            }
            xs[idx] = f2bf(o + o2);
        }
    }
    for (int idx = ctid + kOut * kConsumers; idx < K; idx += kConsumers) {  // K > 256 * kOut
        const int hh = idx / dh, d = idx - hh * dh;
        float o = 0.f;
        for (int c = 0; c < ns; ++c)
            o = fmaf(wts[hh * ns + c], __ldcg(part + (static_cast<long long>(hh) * maxs + c) * (dh + kPartHead) + kPartHead + d), o);
        xs[idx] = f2bf(o);
    }
    bar_sync(1, kConsumers);  // ml / wts live in acc, zeroed by the caller
}

// Greedy-decoding argmax word: float bits made unsigned-ordered, row complemented
// so that atomicMax prefers the lower row among equal values.
__device__ __forceinline__ unsigned long long argmax_key(float v, int row) {
    uint32_t b = __float_as_uint(v);
    b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    return (static_cast<unsigned long long>(b) << 32) | static_cast<uint32_t>(~row);
}
__device__ __forceinline__ int argmax_row(unsigned long long key) { return static_cast<int>(~static_cast<uint32_t>(key)); }

// Row-range GEMV y[b][r] = sum_k W[r][k] x[b][k] for rows [r0, r1) (multiples
// of 16) of a bf16 weight in mma-fragment tile order (K % 32 == 0).  The
// weight tiles stream through the shared-memory ring; activations are staged
// once per task in shared memory (with the fused RMSNorm when x is the fp32
// residual stream); the epilogue applies the op's fused tail.
// `pre` (static scheduler): shared memory holding the task's constant operands
// staged during its dependency wait (RoPE inverse frequencies; gamma sits behind
// the activations), or nullptr to read them from global memory.
__device__ uint64_t body_gemv(const StaticParams& P, const et_op& op, const SlotView& si, uint16_t* xs, float* acc,
                              float* red, Ring& ring, int ctid, const float* pre = nullptr) {
    const int warp = ctid >> 5, lane = ctid & 31;
    const int N = op.i[0], K = op.i[1], nseg = op.i[2];
    const int nb = batch_of(op, P);
    // flags bit 4: grouped GEMV -- coord 0 selects the group's weight matrix and
    // activation slice, coord 1 the row span among i9 tasks per group
    const bool grouped = (op.flags & 16) != 0;
    uint64_t t_probe = 0;  // debug bits 0x1000 / 0x2000 / 0x4000 / 0x8000: prologue probe points
    if ((P.debug & 0x8000) && ctid == 0) t_probe = globaltimer();  // body entry
    const GemvSpan sp = gemv_span(op, grouped ? si.coord[1] : si.coord[0], grouped ? op.i[13] : si.ext0);
    const int r0 = sp.row0, R = sp.rows;

    // ---- prologue: activations into shared memory (bf16 [nb][K]), accumulators zeroed
    if (op.i[3] == 0) {
        // activation rows are i9 elements apart (0: packed [nb][K]); a grouped GEMV reads slice g
        const uint16_t* x = reinterpret_cast<const uint16_t*>(op.p[2]) + (grouped ? static_cast<long long>(si.coord[0]) * K : 0);
        const int xstride = op.i[9] > 0 ? op.i[9] : K, k8 = K / 8;
        if ((nb == 1 || xstride == K) && (P.debug & 0x20000) == 0) {
            // one bulk copy (the TMA engine keeps the whole row in flight; 256 threads'
            // 16-byte loads are limited by the SM's outstanding-miss slots)
            stage_bulk(P, xs, x, static_cast<uint32_t>(nb) * K * 2, ctid);
        } else {
            for (int v = ctid; v < nb * k8; v += kConsumers) {
                const int bi = v / k8, kk = v - bi * k8;
                reinterpret_cast<uint4*>(xs)[v] = __ldcg(reinterpret_cast<const uint4*>(x + static_cast<long long>(bi) * xstride) + kk);
            }
        }
    } else if (op.i[3] == 2) {
        if (K <= 2 * kConsumers) gemv_merge_prologue<2, 16>(P, op, grouped ? si.coord[0] : 0, grouped ? si.coord[1] : 0, xs, acc, ctid, &t_probe);
        else gemv_merge_prologue<4, 8>(P, op, grouped ? si.coord[0] : 0, grouped ? si.coord[1] : 0, xs, acc, ctid, &t_probe);
    } else {
        // RMSNorm prologue: one pass over the fp32 residual stream held in
        // registers (K <= 8192), sum of squares reduced across the CTA
        const float* h = reinterpret_cast<const float*>(op.p[2]);
        const float* gam = (pre && gemv_gamma_staged(op, P)) ? reinterpret_cast<const float*>(xs + gamma_offset(op, P))
                                                             : reinterpret_cast<const float*>(op.p[3]);
        const int stride = op.i[9];
        constexpr int kMaxPer = 8;  // float4 per thread: K <= 8192
        // (a bulk copy of the fp32 row, as x mode 0 does, measured slower here: the
        // register loads overlap the reduction's first shuffles)
        for (int bi = 0; bi < nb; ++bi) {
            float4 hv[kMaxPer];
            float ss = 0.f;
#pragma unroll
            for (int j = 0; j < kMaxPer; ++j) {
                const int k = (ctid + j * kConsumers) * 4;
                if (k < K) hv[j] = ldcg_f4(h + static_cast<long long>(bi) * stride + k);
            }
#pragma unroll
            for (int j = 0; j < kMaxPer; ++j)
                if ((ctid + j * kConsumers) * 4 < K)
                    ss += hv[j].x * hv[j].x + hv[j].y * hv[j].y + hv[j].z * hv[j].z + hv[j].w * hv[j].w;
            if ((P.debug & 0x1000) && ctid == 0) {
                const float4 z = hv[0];
                t_probe = globaltimer() + (z.x == 12345.f ? 1 : 0);  // after the loads land
            }
            ss = warp_sum(ss);
            if (lane == 0) red[warp] = ss;
            bar_sync(1, kConsumers);
            float t = 0.f;
#pragma unroll
            for (int w = 0; w < kConsumerWarps; ++w) t += red[w];
            const float scale = rsqrtf(t / static_cast<float>(K) + op.f[0]);
            if ((P.debug & 0x2000) && ctid == 0) t_probe = globaltimer();  // after the reduction
#pragma unroll
            for (int j = 0; j < kMaxPer; ++j) {
                const int k = (ctid + j * kConsumers) * 4;
                if (k < K) {
                    const float4 g = *reinterpret_cast<const float4*>(gam + k);
                    uint2 o;
                    o.x = static_cast<uint32_t>(f2bf(hv[j].x * scale * g.x)) |
                          (static_cast<uint32_t>(f2bf(hv[j].y * scale * g.y)) << 16);
                    o.y = static_cast<uint32_t>(f2bf(hv[j].z * scale * g.z)) |
                          (static_cast<uint32_t>(f2bf(hv[j].w * scale * g.w)) << 16);
                    *reinterpret_cast<uint2*>(xs + bi * K + k) = o;
                }
            }
            if ((P.debug & 0x4000) && ctid == 0) t_probe = globaltimer();  // after the bf16 stores
            if (bi + 1 < nb) bar_sync(1, kConsumers);  // red[] is reused
        }
    }
    for (int i = ctid; i < nseg * R * nb; i += kConsumers) acc[i] = 0.f;
    bar_sync(1, kConsumers);
    const uint64_t t_pro = ctid == 0 ? (t_probe ? t_probe : globaltimer()) : 0;

    gemv_stream(ring, warp, lane, nseg, static_cast<int>(sp.u1 - sp.u0),
                static_cast<int>(sp.u0 - static_cast<long long>(r0 / 16) * (K / 16)), K, nb, xs,
                [&](int seg, int rt, int g, int q, const float* d) {
                    const int row = seg * R + rt * 16 + g;
                    if (2 * q < nb) {
                        atomicAdd(&acc[row * nb + 2 * q], d[0]);
                        atomicAdd(&acc[(row + 8) * nb + 2 * q], d[2]);
                    }
                    if (2 * q + 1 < nb) {
                        atomicAdd(&acc[row * nb + 2 * q + 1], d[1]);
                        atomicAdd(&acc[(row + 8) * nb + 2 * q + 1], d[3]);
                    }
                });
    bar_sync(1, kConsumers);

    // ---- epilogue
    const int epi = op.i[4];
    if (epi == EPI_QKV_ROPE) {
        const int dh = op.i[8], nq = op.i[10], nkv = op.i[11], cap = op.i[12];
        const long long pos = P.binding[op.i[6]];
        const float* invf = pre ? pre : reinterpret_cast<const float*>(op.p[8]);  // RoPE inverse frequencies [dh/2]
        float* qout = reinterpret_cast<float*>(op.p[4]);
        uint16_t* kc = reinterpret_cast<uint16_t*>(op.p[6]);
        uint16_t* vc = reinterpret_cast<uint16_t*>(op.p[7]);
        const int G = nq / nkv, grows = (G + 2) * dh;  // flags bit 3: rows grouped by kv head
        for (int pr = ctid; pr < R / 2; pr += kConsumers) {
            int row = r0 + 2 * pr;
            if (op.flags & 8) {  // (q heads of group g, k head g, v head g) -> the global row order
                const int g = row / grows, w = row - g * grows;
                row = w < G * dh ? g * G * dh + w : w < (G + 1) * dh ? nq + g * dh + (w - G * dh)
                                                                    : nq + nkv + g * dh + (w - (G + 1) * dh);
            }
            float a = acc[(2 * pr) * nb], b = acc[(2 * pr + 1) * nb];
            if (row < nq + nkv) {  // q or k: rotate the interleaved pair
                const int d = row % dh;
                const float inv = invf[d / 2];
                float sn, cs;
                sincosf(static_cast<float>(pos) * inv, &sn, &cs);
                const float ra = a * cs - b * sn, rb = a * sn + b * cs;
                a = ra;
                b = rb;
            }
            if (row < nq) {
                qout[row] = a;
                qout[row + 1] = b;
            } else {
                const bool isk = row < nq + nkv;
                const int rr = row - nq - (isk ? 0 : nkv);
                const int head = rr / dh, d = rr % dh;
                uint16_t* dst = (isk ? kc : vc) + (static_cast<long long>(head) * cap + pos) * dh + d;
                *reinterpret_cast<uint32_t*>(dst) =
                    static_cast<uint32_t>(f2bf(a)) | (static_cast<uint32_t>(f2bf(b)) << 16);
            }
        }
    } else {
        for (int idx = ctid; idx < R * nb; idx += kConsumers) {
            const int i = idx / nb, bi = idx % nb;
            const float v = acc[i * nb + bi];
            const long long o = static_cast<long long>(bi) * N + r0 + i;
            if (epi == EPI_F32) {
                reinterpret_cast<float*>(op.p[4])[o] = v;
            } else if (epi == EPI_BF16) {
                reinterpret_cast<uint16_t*>(op.p[4])[o] = f2bf(v);
            } else if (epi == EPI_RESID) {
                reinterpret_cast<float*>(op.p[4])[o] = __ldcg(reinterpret_cast<const float*>(op.p[5]) + o) + v;
            } else if (epi == EPI_ADD) {
                atomicAdd(reinterpret_cast<float*>(op.p[4]) + o, v);
            } else if (epi == EPI_SILU_MUL) {
                const float u = acc[(R + i) * nb + bi];
                const float sv = v / (1.f + __expf(-v));
                reinterpret_cast<uint16_t*>(op.p[4])[o] = f2bf(sv * u);
            }
        }
        if ((op.flags & 32) && epi == EPI_F32 && nb == 1) {
            // flags bit 5 (greedy decoding): fold this task's rows into the step's argmax,
            // one packed 64-bit word (ordered float bits << 32 | ~row: atomicMax keeps the
            // largest logit, the lowest row on ties) at p6, zeroed by the step's embed
            unsigned long long best = 0ull;
            for (int i = ctid; i < R; i += kConsumers) {
                const unsigned long long key = argmax_key(acc[i], r0 + i);
                best = key > best ? key : best;
            }
            for (int o = 16; o > 0; o >>= 1) {
                const unsigned long long x = __shfl_xor_sync(0xffffffffu, best, o);
                best = x > best ? x : best;
            }
            if ((ctid & 31) == 0 && best) atomicMax(reinterpret_cast<unsigned long long*>(op.p[6]), best);
        }
    }
    return t_pro;
}

// ---------------------------------------------------------------------------
// Large-batch GEMV on the 5th-generation tensor cores (ET_OP_GEMV_TC, ops.cuh).
// Shared-memory mbarriers behind the misc words: x slot full [kTcXSlots], x slot
// free [kTcXSlots] (tcgen05.commit), accumulators done [1] (tcgen05.commit).
struct TcState {
    uint32_t tmem;        // TMEM column base (512 columns, allocated at kernel start)
    unsigned int xp;      // activation pieces consumed (issuer thread)
    unsigned int ndone;   // tensor-core tasks completed (phase of the done barrier)
};

__device__ __forceinline__ uint64_t* tc_bars(uint8_t* smem) {
    return reinterpret_cast<uint64_t*>(smem + kSmemMisc + 384);
}

// Bounded mbarrier wait (reports a deadlock instead of hanging; false when aborted).
__device__ __noinline__ bool tc_wait(uint64_t* bar, uint32_t parity, DevStatus* status, long long watchdog_ns,
                                     int worker, int code) {
    if (mbar_try_wait(bar, parity)) return true;
    const uint64_t t0 = globaltimer();
    uint32_t it = 0;
    while (!mbar_try_wait(bar, parity)) {
        if ((++it & 1023u) == 0) {
            if (aborted(status)) return false;
            if (globaltimer() - t0 > static_cast<uint64_t>(watchdog_ns)) {
                report(status, ET_ERR_DEADLOCK, worker, -1, code, 0);
                return false;
            }
        }
    }
    return true;
}

// Sum of the nis issuers' accumulators (cols apart) for 16 columns of this lane.
__device__ __forceinline__ void tc_sum16(uint32_t taddr, int nis, int cols, float* v) {
    tmem_ld16(taddr, v);
    for (int k = 1; k < nis; ++k) {
        float w[16];
        tmem_ld16(taddr + static_cast<uint32_t>(k * cols), w);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] += w[j];
    }
}

// Issuer k (one thread) of a tensor-core GEMV task: for pieces k, k + nis, ...,
// wait for the activation piece, then per weight chunk four K=16 MMAs into its
// own (segment, block) accumulators; each chunk's ring stage is released by
// tcgen05.commit once its MMAs have read it.  Everything lives in registers:
// the mbarrier round trips of one thread bound its streaming rate, so up to
// kTcIssuers threads (in different warps) take alternate pieces.
__device__ __noinline__ void tc_issue(uint8_t* smem, uint32_t tmem, unsigned long long c0, unsigned int xp0, int k,
                                      int nis, int np, int nsb, int cpb, int npad, int kp, unsigned long long* xwait,
                                      DevStatus* status, long long watchdog_ns, int worker) {
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSmemBar);
    uint64_t* empty = full + kStages;
    uint64_t* bars = tc_bars(smem);
    const uint32_t ring0 = smem_u32(smem + kSmemRing);
    const uint32_t idesc = umma_idesc_bf16(npad);
    const uint32_t xbytes = static_cast<uint32_t>(npad * kp * 2);
    const int nxs = tc_xslots(xbytes);
    const int wpp = nsb * cpb;                               // chunks per piece
    const uint64_t xstep = static_cast<uint64_t>(npad * 2);  // one k step of the piece (npad*32 B >> 4)
    for (int p = k; p < np; p += nis) {
        const unsigned int gx = xp0 + static_cast<unsigned int>(p);  // the CTA's piece sequence number
        const int xb = static_cast<int>(gx % nxs);
        const uint64_t tx0 = xwait ? globaltimer() : 0;
        if (!tc_wait(&bars[xb], (gx / nxs) & 1u, status, watchdog_ns, worker, -4)) return;
        if (xwait) xwait[0] += globaltimer() - tx0;
        tc_fence_after();
        const uint64_t xd = umma_desc(smem_u32(smem + kSmemX) + xb * xbytes);
        unsigned long long c = c0 + static_cast<unsigned long long>(p) * wpp;
        uint32_t d = tmem;
        for (int sb = 0; sb < nsb; ++sb, d += npad) {  // (segment, block) accumulators
            uint64_t xk = xd;
            for (int ch = 0; ch < cpb; ++ch, ++c, xk += 4 * xstep) {
                const int st = static_cast<int>(c & (kStages - 1));
                const uint32_t par = static_cast<uint32_t>(c / kStages) & 1u;
                if (!mbar_try_wait(&full[st], par)) {
                    const uint64_t tw0 = xwait ? globaltimer() : 0;
                    if (!tc_wait(&full[st], par, status, watchdog_ns, worker, -2)) return;
                    if (xwait) xwait[1] += globaltimer() - tw0;
                }
                tc_fence_after();
                const uint64_t a = umma_desc(ring0 + st * kStageBytes);
                if (elect_one_sync()) {
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        umma_bf16(d, a + j * 256, xk + j * xstep, idesc, (p != k || ch != 0 || j != 0) ? 1u : 0u);
                    umma_commit(&empty[st]);
                }
                __syncwarp();
            }
        }
        if (elect_one_sync()) umma_commit(&bars[kTcXSlots + xb]);  // the x slot is free once these MMAs complete
        __syncwarp();
    }
    if (elect_one_sync()) umma_commit(&bars[2 * kTcXSlots]);  // one of the kTcIssuers arrivals on the done barrier
    __syncwarp();
}

__device__ __noinline__ uint64_t body_gemv_tc(const StaticParams& P, const et_op& op, const SlotView& si, uint8_t* smem,
                                 Ring& ring, TcState& ts, int ctid) {
    const int warp = ctid >> 5, lane = ctid & 31;
    const int N = op.i[0], nseg = op.i[2], kp = op.i[6];
    const int nb = tc_batch(op, P.binding), npad = tc_npad(nb);
    const bool tiled = tc_tiled(op);  // f4 GEMM tile: (token block, GEMV task) from the coordinates
    int tj = 0, tt = 0;
    if (tiled) tc_tile(op, si.coord, &tj, &tt);
    const TcSpan sp = tiled ? tc_span(op, tt, op.i[12]) : tc_span(op, si.coord[0], si.ext0);
    if (sp.nblk <= 0 || sp.np <= 0) return 0;
    uint64_t* bars = tc_bars(smem);
    const int cpb = kp / 64;                       // 16 KB weight chunks per (piece, block)
    const int wpp = nseg * sp.nblk * cpb;          // weight chunks per piece
    const int cols = nseg * sp.nblk * npad;        // TMEM columns of one issuer's accumulators
    // issuers: lane 0 of warps 0..nis-1 take pieces k, k + nis, ... into their own
    // accumulator columns (the protocol round trips of one thread bound its rate).
    // Parity waits are exact only while no waiter runs two phases ahead of the fills:
    // an issuer's next piece must lie within one ring lap (nis * wpp <= kStages) and
    // one x-slot lap (nis <= slots) of its previous one -- the producer fills in order.
    const int nxs = tc_xslots(static_cast<uint32_t>(npad * kp * 2));
    int nis = kTmemCols / cols;
    nis = nis < kTcIssuers ? nis : kTcIssuers;
    nis = nis < sp.np ? nis : sp.np;
    nis = nis < kStages / wpp ? nis : kStages / wpp;
    nis = nis < nxs ? nis : nxs;
    nis = nis > 1 ? nis : 1;
    const uint64_t t_pro = ctid == 0 ? globaltimer() : 0;
    if (warp < kTcIssuers) {  // whole issuer warps (converged: uniform operands), one elected lane issues
        unsigned long long xw[2] = {0, 0};  // debug: ns waiting for activation pieces / ring stages
        tc_issue(smem, ts.tmem + static_cast<uint32_t>(warp * cols), ring.seq, ts.xp, warp, nis, warp < nis ? sp.np : 0,
                 nseg * sp.nblk, cpb, npad, kp, ring.dbg ? xw : nullptr, P.status, P.watchdog_ns, ring.worker);
        ring.xwait += xw[0];
        ring.stall += xw[1];
    }
    // the other consumer threads block on the named barrier while the issuers run (spinning
    // on the done mbarrier would contend with the issuers' mbarrier traffic)
    bar_sync(1, kConsumers);
    ring.seq += static_cast<unsigned long long>(wpp) * sp.np;
    ts.xp += static_cast<unsigned int>(sp.np);
    const bool done = tc_wait(&bars[2 * kTcXSlots], ts.ndone & 1u, P.status, P.watchdog_ns, ring.worker, -5);
    ++ts.ndone;
    if (!done) return t_pro;
    tc_fence_after();

    // ---- epilogue: warp w reads TMEM lanes 32*(w%4).. (rows of each block); the two
    // warp halves take alternate 16-column (batch) chunks; the issuers' partial
    // accumulators are summed
    const int q = warp & 3, half = warp >> 2;
    const int nchunk = npad / 16, nitems = sp.nblk * nchunk;
    const int epi = op.i[4];
    const int ostride = op.i[8] > 0 ? op.i[8] : N;  // output rows (a padded block's tail rows are dropped)
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    // tiled GEMM: token rows start at block j; EPI_F32 goes to the k-split's partial buffer
    const long long obase = tiled ? static_cast<long long>(tt % (op.i[3] > 0 ? op.i[3] : 1)) * op.i[11] +
                                        static_cast<long long>(tj) * op.i[10] * ostride
                                  : 0;
    for (int it = half; it < nitems; it += 2) {
        const int blk = it / nchunk, n0 = (it - blk * nchunk) * 16;
        float v[16], u[16];
        tc_sum16(ts.tmem + lane_off + static_cast<uint32_t>(blk * npad + n0), nis, cols, v);
        if (epi == EPI_SILU_MUL)
            tc_sum16(ts.tmem + lane_off + static_cast<uint32_t>((sp.nblk + blk) * npad + n0), nis, cols, u);
        const int row = (sp.b0 + blk) * 128 + q * 32 + lane;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int n = n0 + j;
            if (n < nb && row < ostride) {
                const long long o = obase + static_cast<long long>(n) * ostride + row;
                if (epi == EPI_F32) {
                    reinterpret_cast<float*>(op.p[4])[o] = v[j];
                } else if (epi == EPI_ADD) {
                    atomicAdd(reinterpret_cast<float*>(op.p[4]) + o, v[j]);
                } else if (epi == EPI_BF16) {
                    reinterpret_cast<uint16_t*>(op.p[4])[o] = f2bf(v[j]);
                } else if (epi == EPI_RESID) {
                    reinterpret_cast<float*>(op.p[4])[o] = __ldcg(reinterpret_cast<const float*>(op.p[5]) + o) + v[j];
                } else if (epi == EPI_SILU_MUL) {
                    const float sv = v[j] / (1.f + __expf(-v[j]));
                    reinterpret_cast<uint16_t*>(op.p[4])[xb_offset(n, row, npad, op.i[7])] = f2bf(sv * u[j]);
                }
            }
        }
    }
    tc_fence_before();  // the next task's MMAs overwrite these columns after the closing barrier
    return t_pro;
}

// RMSNorm of stream row n into the tensor-core operand layout (ET_OP_NORM).
__device__ __noinline__ void body_norm(const StaticParams& P, const et_op& op, const SlotView& si, float* red, int ctid) {
    const int warp = ctid >> 5, lane = ctid & 31;
    const int n = si.coord[0], nb = batch_of(op, P);
    if (n >= nb) return;
    const int K = op.i[0], kp = op.i[6], npad = tc_npad(nb);
    const float* h = reinterpret_cast<const float*>(op.p[0]) + static_cast<long long>(n) * K;
    const float* gam = reinterpret_cast<const float*>(op.p[1]);
    uint16_t* out = reinterpret_cast<uint16_t*>(op.p[2]);
    constexpr int kMaxPer = 8;  // K <= 8192
    float4 hv[kMaxPer], gv[kMaxPer];
    float ss = 0.f;
    // gamma loads with the row (one L2 round trip: the wait's acquire left L1 cold)
#pragma unroll
    for (int j = 0; j < kMaxPer; ++j) {
        const int k = (ctid + j * kConsumers) * 4;
        if (k < K) {
            hv[j] = ldcg_f4(h + k);
            gv[j] = __ldg(reinterpret_cast<const float4*>(gam + k));
        }
    }
#pragma unroll
    for (int j = 0; j < kMaxPer; ++j)
        if ((ctid + j * kConsumers) * 4 < K)
            ss += hv[j].x * hv[j].x + hv[j].y * hv[j].y + hv[j].z * hv[j].z + hv[j].w * hv[j].w;
    ss = warp_sum(ss);
    if (lane == 0) red[warp] = ss;
    bar_sync(1, kConsumers);
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < kConsumerWarps; ++w) t += red[w];
    const float scale = rsqrtf(t / static_cast<float>(K) + op.f[0]);
#pragma unroll
    for (int j = 0; j < kMaxPer; ++j) {
        const int k = (ctid + j * kConsumers) * 4;
        if (k < K) {
            const float4 g = gv[j];
            uint2 o;
            o.x = static_cast<uint32_t>(f2bf(hv[j].x * scale * g.x)) | (static_cast<uint32_t>(f2bf(hv[j].y * scale * g.y)) << 16);
            o.y = static_cast<uint32_t>(f2bf(hv[j].z * scale * g.z)) | (static_cast<uint32_t>(f2bf(hv[j].w * scale * g.w)) << 16);
            *reinterpret_cast<uint2*>(out + xb_offset(n, k, npad, kp)) = o;
            if (op.p[3])  // also row-major bf16 [b][K] (the MoE expert tiles read their tokens' rows)
                *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(op.p[3]) + static_cast<long long>(n) * K + k) = o;
        }
    }
}

// Qwen3-style per-head RMSNorm (weight w[dh]) followed by the pair rotation at
// position pos, in place on one head vector in shared memory; one warp.
__device__ __noinline__ void qk_norm_rope(float* v, int dh, const float* w, float eps, const float* invf,
                                             long long pos, int lane) {
    float sc = 1.f;
    if (w) {  // nullptr: RoPE only (Llama: no q/k norm)
        float ss = 0.f;
        for (int d = lane; d < dh; d += 32) ss += v[d] * v[d];
        ss = warp_sum(ss);
        sc = rsqrtf(ss / static_cast<float>(dh) + eps);
    }
    for (int j = lane; j < dh / 2; j += 32) {
        const float a = v[2 * j] * sc * (w ? w[2 * j] : 1.f), b = v[2 * j + 1] * sc * (w ? w[2 * j + 1] : 1.f);
        float sn, cs;
        sincosf(static_cast<float>(pos) * invf[j], &sn, &cs);
        v[2 * j] = a * cs - b * sn;
        v[2 * j + 1] = a * sn + b * cs;
    }
    __syncwarp();
}

// Merge of the splits of kv head g's q heads with the new token at position s
// (K/V row s of the cache):
//   O = (sum_c e^(m_c-M) o_c + e^(s_new-M) v_new) / (sum_c e^(m_c-M) l_c + e^(s_new-M)).
// q (RoPE applied) is in shared memory (qs, row stride qstride).  Every global
// operand -- split statistics, the new K/V row and this thread's o partials
// (in registers, up to 16 splits per pass) -- is requested before the first
// use, so a pass costs one L2 round trip.
// kWide: G * dh <= 1024 (MoE instantiation: 8 q heads per kv head), else G * dh
// <= 512 -- the register footprint of the dense kernel stays spill-free.
// kTcLayout (tensor-core instantiations): operand-layout output (i9) and swizzled cache rows.
template <bool kWide, bool kTcLayout = false>
__device__ __noinline__ void attn_merge_group(const StaticParams& P, const et_op& op, int gi, const float* qs,
                                              int qstride, float* scr, int ctid) {
    constexpr int kPass = kWide ? 8 : 16, kOut = kWide ? 4 : 2;  // splits in registers; outputs per thread
    const int warp = ctid >> 5, lane = ctid & 31;
    const int dh = op.i[0], G = op.i[1], CH = op.i[2], cap = op.i[3], kvh = op.i[6];
    const int maxs = kTcLayout ? attn_part_stride(op) : op.i[5];
    const int g = gi % kvh, bq = gi / kvh;  // kv head, sequence of the batch
    const long long s = P.binding[op.i[4]];
    const int nspl = kTcLayout ? attn_splits_with_data(op, P.binding) : attn_splits_base(op, P.binding);
    const float scale = op.f[0];
    const float* part = reinterpret_cast<const float*>(op.p[3]) + static_cast<long long>(gi) * G * maxs * (dh + kPartHead);
    const long long cb = static_cast<long long>(bq) * op.i[8];  // this sequence's cache
    const uint16_t* kn = reinterpret_cast<const uint16_t*>(op.p[1]) + cb + (static_cast<long long>(g) * cap + s) * dh;
    const uint16_t* vn = reinterpret_cast<const uint16_t*>(op.p[2]) + cb + (static_cast<long long>(g) * cap + s) * dh;
    // i9 > 0 (tensor-core instantiation): the output goes to the operand layout of the
    // next GEMV (piece length i9, batch from symbol slot i10)
    const int kxb = kTcLayout ? op.i[9] : 0;
    const int xnp = kxb ? tc_npad(op.i[10] >= 0 ? static_cast<int>(P.binding[op.i[10]]) : 1) : 0;
    uint16_t* out = reinterpret_cast<uint16_t*>(op.p[4]) +
                    (kxb ? 0 : static_cast<long long>(bq) * kvh * G * dh + static_cast<long long>(g) * G * dh);
    float* ml = scr;                    // [G][nspl][2]
    float* wts = ml + 2 * G * nspl;     // [G][nspl]
    float* hs = wts + G * nspl;         // [G]: weight of the new token
    float* kns = hs + G;                // [dh]
    // flags bit 8 (tensor-core instantiations): cache rows hold their 16-byte chunks
    // XOR-swizzled by position % 8, so row-strided tensor-core reads are bank-conflict free
    const int csw = (kTcLayout && (op.flags & 256)) ? static_cast<int>(s & 7) : 0;
    float ov[kOut][kPass];
    float vv[kOut];
#pragma unroll
    for (int j = 0; j < kOut; ++j) {
        const int idx = ctid + j * kConsumers;
        const int hh = idx / dh, d = idx - hh * dh;
        vv[j] = idx < G * dh ? bf2f(__ldcg(vn + ((((d >> 3) ^ csw)) << 3) + (d & 7))) : 0.f;
#pragma unroll
        for (int c = 0; c < kPass; ++c)
            ov[j][c] = (idx < G * dh && c < nspl) ? __ldcg(part + (static_cast<long long>(hh) * maxs + c) * (dh + kPartHead) + kPartHead + d)
                                                 : 0.f;
    }
    for (int i = ctid; i < G * nspl; i += kConsumers) {
        const float* pr = part + (static_cast<long long>(i / nspl) * maxs + i % nspl) * (dh + kPartHead);
        ml[2 * i] = __ldcg(pr);
        ml[2 * i + 1] = __ldcg(pr + 1);
    }
    for (int d = ctid; d < dh; d += kConsumers) kns[d] = bf2f(__ldcg(kn + ((((d >> 3) ^ csw)) << 3) + (d & 7)));
    bar_sync(1, kConsumers);
    for (int hh = warp; hh < G; hh += kConsumerWarps) {
        float dot = 0.f;
        for (int d = lane; d < dh; d += 32) dot += qs[hh * qstride + d] * kns[d];
        const float snew = warp_sum(dot) * scale;
        float M = snew;
        for (int c = lane; c < nspl; c += 32) M = fmaxf(M, ml[2 * (hh * nspl + c)]);
        M = warp_max(M);
        float L = 0.f;
        for (int c = lane; c < nspl; c += 32) {
            const float e = __expf(ml[2 * (hh * nspl + c)] - M);
            wts[hh * nspl + c] = e;
            L += e * ml[2 * (hh * nspl + c) + 1];
        }
        const float en = __expf(snew - M);
        L = warp_sum(L) + en;
        const float inv = 1.f / L;
        for (int c = lane; c < nspl; c += 32) wts[hh * nspl + c] *= inv;
        __syncwarp();
        if (lane == 0) hs[hh] = en * inv;
    }
    bar_sync(1, kConsumers);
#pragma unroll
    for (int j = 0; j < kOut; ++j) {
        const int idx = ctid + j * kConsumers;
        if (idx >= G * dh) break;
        const int hh = idx / dh, d = idx - hh * dh;
        const float* w = wts + hh * nspl;
        float o = hs[hh] * vv[j], o2 = 0.f;
#pragma unroll
        for (int c = 0; c < kPass; c += 2) {
            if (c < nspl) o = fmaf(w[c], ov[j][c], o);
            if (c + 1 < nspl) o2 = fmaf(w[c + 1], ov[j][c + 1], o2);
        }
        // long contexts: the remaining splits, their loads batched eight at a time (one L2
        // round trip per batch instead of per split)
        for (int c0 = kPass; c0 < nspl; c0 += 8) {
            float pv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                pv[u] = c0 + u < nspl ? __ldcg(part + (static_cast<long long>(hh) * maxs + c0 + u) * (dh + kPartHead) + kPartHead + d)
                                      : 0.f;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (c0 + u < nspl) o = fmaf(w[c0 + u], pv[u], o);
        }
        out[kxb ? xb_offset(bq, g * G * dh + idx, xnp, kxb) : idx] = f2bf(o + o2);
    }
    if constexpr (kWide) {
        if ((op.flags & 33) == 33) {
            // split-K q/k/v projection (flags bit 5): its fp32 accumulators of this group are
            // consumed (every split arrived, split 0 appended k/v) -- zero them for the next step
            const long long rb = static_cast<long long>(bq) * op.i[7];  // this sequence's projection row
            float* q = reinterpret_cast<float*>(op.p[0]) + rb + static_cast<long long>(g) * G * dh;
            float* kr = reinterpret_cast<float*>(op.p[8]) + rb + static_cast<long long>(g) * dh;
            float* vr = kr + static_cast<long long>(kvh) * dh;
            for (int i = ctid; i < G * dh; i += kConsumers) q[i] = 0.f;
            for (int i = ctid; i < dh; i += kConsumers) {
                kr[i] = 0.f;
                vr[i] = 0.f;
            }
        }
    }
}

// Single-split group (fused merge, one split per (sequence, kv head): large batches)
// finished in shared memory: the split's folded (M, L, O) per q head (sc: mW [8 warps][8],
// lW, oacc [G][dh]) plus the new token (its k / v, appended by this task, at
// sc + kAttnSoloKv) give the attention output directly, written in the next GEMV's
// operand layout -- no partials round trip through L2, no arrival atomic, no merge.
// The raw q/k/v accumulators of the group are zeroed for the next step (flags 33), as
// attn_merge_group does.
__device__ __noinline__ void attn_solo_finish(const StaticParams& P, const et_op& op, int gi, const float* qs,
                                              int qstride, float* sc, int ctid) {
    const int warp = ctid >> 5, lane = ctid & 31;
    const int dh = op.i[0], G = op.i[1], kvh = op.i[6];
    const int g = gi % kvh, bq = gi / kvh;
    const float* mW = sc;
    const float* lW = sc + 64;
    const float* oacc = sc + 128;
    const float* kv = sc + kAttnSoloKv;  // [2][dh] new k, v (bf16-rounded, as cached)
    float* hw = sc + kAttnSoloKv + 2 * dh;  // [G][2]: weight of the folded O, weight of v_new
    for (int h = warp; h < G; h += kConsumerWarps) {
        float dot = 0.f;
        for (int d = lane; d < dh; d += 32) dot += qs[h * qstride + d] * kv[d];
        const float snew = warp_sum(dot) * op.f[0];
        if (lane == 0) {
            float M = -INFINITY;
            for (int w = 0; w < kConsumerWarps; ++w) M = fmaxf(M, mW[w * 8 + h]);
            float L = 0.f;
            if (M != -INFINITY)
                for (int w = 0; w < kConsumerWarps; ++w) {
                    const float mw = mW[w * 8 + h];
                    if (mw != -INFINITY) L += lW[w * 8 + h] * __expf(mw - M);
                }
            const float Mn = fmaxf(M, snew);
            const float a = M == -INFINITY ? 0.f : __expf(M - Mn), en = __expf(snew - Mn);
            const float inv = 1.f / (L * a + en);
            hw[2 * h] = a * inv;
            hw[2 * h + 1] = en * inv;
        }
    }
    bar_sync(1, kConsumers);
    const int kxb = op.i[9];
    const int xnp = tc_npad(op.i[10] >= 0 ? static_cast<int>(P.binding[op.i[10]]) : 1);
    uint16_t* out = reinterpret_cast<uint16_t*>(op.p[4]);
    for (int idx = ctid; idx < G * dh; idx += kConsumers) {
        const int h = idx / dh, d = idx - h * dh;
        const float o = oacc[idx] * hw[2 * h] + kv[dh + d] * hw[2 * h + 1];
        out[xb_offset(bq, g * G * dh + idx, xnp, kxb)] = f2bf(o);
    }
    if ((op.flags & 33) == 33) {  // the split-K q/k/v accumulators of this group: consumed
        const long long rb = static_cast<long long>(bq) * op.i[7];
        float* q = reinterpret_cast<float*>(op.p[0]) + rb + static_cast<long long>(g) * G * dh;
        float* kr = reinterpret_cast<float*>(op.p[8]) + rb + static_cast<long long>(g) * dh;
        float* vr = kr + static_cast<long long>(kvh) * dh;
        for (int i = ctid; i < G * dh; i += kConsumers) q[i] = 0.f;
        for (int i = ctid; i < dh; i += kConsumers) {
            kr[i] = 0.f;
            vr[i] = 0.f;
        }
    }
}

// Tensor-core form of a split's block loop (tensor-core instantiations: the batch
// path), split along positions: warp w owns the 16-position tile (w % 4) of every
// block of parity (w / 4) -- warps 0-3 take blocks 0, 2, 4, ..., warps 4-7 blocks
// 1, 3, 5, ... -- and keeps its own online softmax (m, l per head) and O^T
// accumulators in registers, so a block needs no CTA barrier: per tile,
// S^T = K Q^T (mma.sync m16n8k16, positions x q heads, q split bf16 hi + lo), the
// running max / sum by shuffles over the tile's 16 positions, P^T transposed
// through a per-warp scratch, then O^T += V^T P^T for every 16-dim tile of the
// head (V^T by ldmatrix.trans, P split hi + lo).  The four warps of a block meet
// on a named barrier only to release its two ring stages.  At the end the 8 warp
// partials are folded in shared memory into the split's partial (or, with flags
// bit 9 and a single split, left as 8 sub-splits for the group merge).
// G <= 8, dh % 16 == 0, dh <= 128, CH == 64 (checked on the host).
__device__ __noinline__ bool attn_split_mma(const StaticParams& P, const et_op& op, int gi, int c, const AttnBlocks ab,
                                            long long s, const float* qs, int qstride, float* sc, float* st, Ring& ring,
                                            int ctid) {
    const int warp = ctid >> 5, lane = ctid & 31, g8 = lane >> 2, q4 = lane & 3;
    const int dh = op.i[0], G = op.i[1], CH = op.i[2], maxs = attn_part_stride(op);
    const float scale = op.f[0];
    const int nks = dh / 16, half = warp >> 2, tile = warp & 3;
    const bool swz = (op.flags & 256) != 0;  // cache rows chunk-swizzled by position % 8
    // Q^T fragments (k = dim, n = head g8) and the bf16 remainders q - bf16(q) (ET_ATTN_QLO: a
    // second MMA per k step), likewise P split hi + lo for P.V (ET_ATTN_PLO).  Without the
    // remainders the batched step is 6-10% faster (b=64: 9.01 -> 8.48 ms at s=1024, 21.8 ->
    // 19.5 ms at s=8192) but the MoE tensor-core logits leave the 2e-3 tolerance
    // (tests/test_gpu_moe.py: 5.2e-3; P alone: 4.5e-3), so both stay on.
    // The fragments live in shared memory, [k step][lane] x {hi0, hi1, lo0, lo1} (the same
    // for every warp; one 16-byte load per k step): held in registers they took 32 of the
    // 168 and left the block loop one temporary, serialising every ldmatrix -> mma pair.
    uint32_t* qfr = reinterpret_cast<uint32_t*>(sc + kAttnQFrag);
    {
        const int fks = ctid >> 5, fl = ctid & 31, fg = fl >> 2, fq = fl & 3;  // 256 threads = 8 x 32
        uint4 f = make_uint4(0u, 0u, 0u, 0u);
        if (fks < nks && fg < G) {
            const float* qv = qs + fg * qstride + fks * 16 + 2 * fq;
            split_bf16x2(qv[0], qv[1], f.x, f.z);
            split_bf16x2(qv[8], qv[9], f.y, f.w);
        }
        reinterpret_cast<uint4*>(qfr)[ctid] = f;
    }
    bar_sync(1, kConsumers);
    const int h0 = 2 * q4;                       // this thread's two head columns
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    float o[8][4];                               // O^T per 16-dim tile: (d, h0) (d, h0+1) (d+8, h0) (d+8, h0+1)
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
    float* pw = sc + warp * 16 * 9;              // per-warp P scratch [16 positions][8 heads] (+1 pad)
    const unsigned long long seq0 = ring.seq;
    ring.seq += 2ull * ab.nblk;
    for (int blk = half; blk < ab.nblk; blk += 2) {
        const long long pb = ab.p0 + static_cast<long long>(blk) * CH;
        const int np = static_cast<int>(pb + CH < s ? CH : s - pb);
        const unsigned long long ck = seq0 + 2ull * blk, cv = ck + 1;
        const uint8_t* kb = ring.wait(ck);
        if (!kb) return false;
        const int t0 = 16 * tile;                // the tile's first position in the block
        if (t0 < np) {
            float d[4] = {0.f, 0.f, 0.f, 0.f}, e[4] = {0.f, 0.f, 0.f, 0.f};
            // K tile as the A operand by ldmatrix: lane l addresses row (l & 7) of matrix
            // l >> 3 = (rows +8 if odd, k chunk +1 if >= 2); row r's chunks are swizzled by r % 8
            // chunk (2 ks + hi) ^ sw = (2 ks ^ (sw & 6)) | ((hi ^ sw) & 1): the k step's byte
            // offset is (ks << 5) ^ ((sw & 6) << 4) past the row's odd-chunk bit (two
            // registers instead of eight precomputed offsets)
            const int km = lane >> 3, kr = lane & 7;
            const int ksw = swz ? kr : 0;
            const uint32_t kaddr = smem_u32(kb + (t0 + ((km & 1) << 3) + kr) * dh * 2) +
                                   static_cast<uint32_t>((((km >> 1) ^ ksw) & 1) << 4);
            const uint32_t kx = static_cast<uint32_t>((ksw & 6) << 4);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                if (ks < nks) {
                    const uint4 a = ldsm_x4_addr(kaddr + (static_cast<uint32_t>(ks << 5) ^ kx));
                    const uint4 qf = reinterpret_cast<const uint4*>(qfr)[ks * 32 + lane];
                    mma_bf16_16816(d, a, qf.x, qf.y);
                    if (ET_ATTN_QLO) mma_bf16_16816(e, a, qf.z, qf.w);
                }
            }
            // scores of positions t0+g8 / t0+g8+8 for heads h0, h0+1 (invalid -> -inf)
            const bool v0 = t0 + g8 < np, v1 = t0 + g8 + 8 < np;
            const float s00 = v0 ? (d[0] + e[0]) * scale : -INFINITY, s01 = v0 ? (d[1] + e[1]) * scale : -INFINITY;
            const float s10 = v1 ? (d[2] + e[2]) * scale : -INFINITY, s11 = v1 ? (d[3] + e[3]) * scale : -INFINITY;
            float mx0 = fmaxf(s00, s10), mx1 = fmaxf(s01, s11);
#pragma unroll
            for (int off = 4; off < 32; off <<= 1) {  // over g8 (lanes with the same q4)
                mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
                mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
            }
            const float n0 = fmaxf(m0, mx0), n1 = fmaxf(m1, mx1);  // finite: the tile has a valid position
            const float a0 = __expf(m0 - n0), a1 = __expf(m1 - n1);
            const float p00 = __expf(s00 - n0), p01 = __expf(s01 - n1), p10 = __expf(s10 - n0), p11 = __expf(s11 - n1);
            float r0s = p00 + p10, r1s = p01 + p11;
#pragma unroll
            for (int off = 4; off < 32; off <<= 1) {
                r0s += __shfl_xor_sync(0xffffffffu, r0s, off);
                r1s += __shfl_xor_sync(0xffffffffu, r1s, off);
            }
            m0 = n0;
            m1 = n1;
            l0 = l0 * a0 + r0s;
            l1 = l1 * a1 + r1s;
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
                o[mt][0] *= a0;
                o[mt][1] *= a1;
                o[mt][2] *= a0;
                o[mt][3] *= a1;
            }
            // P^T fragments need (positions 2q4.., head g8): transpose through the warp scratch
            pw[g8 * 9 + h0] = p00;
            pw[g8 * 9 + h0 + 1] = p01;
            pw[(g8 + 8) * 9 + h0] = p10;
            pw[(g8 + 8) * 9 + h0 + 1] = p11;
            __syncwarp();
            const float q00 = g8 < G ? pw[(2 * q4) * 9 + g8] : 0.f, q01 = g8 < G ? pw[(2 * q4 + 1) * 9 + g8] : 0.f;
            const float q10 = g8 < G ? pw[(2 * q4 + 8) * 9 + g8] : 0.f, q11 = g8 < G ? pw[(2 * q4 + 9) * 9 + g8] : 0.f;
            __syncwarp();
            uint32_t bh0, bl0, bh1, bl1;
            split_bf16x2(q00, q01, bh0, bl0);
            split_bf16x2(q10, q11, bh1, bl1);
            const uint8_t* vb = ring.wait(cv);
            if (!vb) return false;
            // this lane's V row; rows past the block's valid positions (the partial
            // last block) hold stale stage bytes that need not be finite, and their
            // P is 0 but 0 * Inf = NaN: read the tile's first (valid) row instead
            const int mi = lane >> 3, prow0 = t0 + ((mi & 2) ? 8 : 0) + (lane & 7);
            const int prow = prow0 < np ? prow0 : t0;
            const uint8_t* vrow = vb + prow * dh * 2;
            const int csw = swz ? (prow & 7) : 0;                                  // chunk swizzle of that row
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
                if (mt < nks) {
                    const uint4 a = ldsm_x4_trans(vrow + ((2 * mt + (mi & 1)) ^ csw) * 16);  // V^T: dims x positions
                    mma_bf16_16816(o[mt], a, bh0, bh1);
                    if (ET_ATTN_PLO) mma_bf16_16816(o[mt], a, bl0, bl1);
                }
            }
        } else {
            if (!ring.wait(cv)) return false;
        }
        // the block's four warps are done with its K and V stages: the first warp of the
        // four waits for the others and releases them; the other three only arrive and go
        // on to their next block.  A warp runs at most one group step ahead of the slowest
        // (step i + 2 reuses step i's stages, released after step i's barrier), so two
        // barrier ids per group, alternating by step, keep the phases apart.
        const int bid = 2 + half + (((blk >> 1) & 1) << 1);
        if ((ctid & 127) < 32) {
            bar_sync(bid, 128);
            if ((ctid & 127) == 0) {
                ring.release(ck);
                ring.release(cv);
            }
        } else {
            bar_arrive(bid, 128);
        }
    }
    const bool solo = attn_solo(op, P.binding);
    if (solo || !attn_warp_partials(op, P.binding)) {
        // fold the 8 warps' partials in shared memory: M = max_w m_w, L = sum_w l_w e^(m_w - M),
        // O = sum_w e^(m_w - M) O_w (red.shared.add), one partial per split
        bar_sync(1, kConsumers);  // every warp is past its P scratch
        float* mW = sc;           // [8 warps][8 heads]
        float* lW = sc + 64;
        float* oacc = sc + 128;   // [G][dh]
        if (g8 == 0) {
            mW[warp * 8 + h0] = m0;
            mW[warp * 8 + h0 + 1] = m1;
            lW[warp * 8 + h0] = l0;
            lW[warp * 8 + h0 + 1] = l1;
        }
        for (int i = ctid; i < G * dh; i += kConsumers) oacc[i] = 0.f;
        bar_sync(1, kConsumers);
        float M0 = -INFINITY, M1 = -INFINITY;
#pragma unroll
        for (int w = 0; w < kConsumerWarps; ++w) {
            M0 = fmaxf(M0, mW[w * 8 + h0]);
            M1 = fmaxf(M1, mW[w * 8 + h0 + 1]);
        }
        const float f0 = m0 == -INFINITY ? 0.f : __expf(m0 - M0), f1 = m1 == -INFINITY ? 0.f : __expf(m1 - M1);
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
            if (mt < nks) {
                const int d0 = 16 * mt + g8;
                if (h0 < G) {
                    atomicAdd(&oacc[h0 * dh + d0], o[mt][0] * f0);
                    atomicAdd(&oacc[h0 * dh + d0 + 8], o[mt][2] * f0);
                }
                if (h0 + 1 < G) {
                    atomicAdd(&oacc[(h0 + 1) * dh + d0], o[mt][1] * f1);
                    atomicAdd(&oacc[(h0 + 1) * dh + d0 + 8], o[mt][3] * f1);
                }
            }
        }
        bar_sync(1, kConsumers);
        if (solo) {
            attn_solo_finish(P, op, gi, qs, qstride, sc, ctid);
            return true;
        }
        float* part = reinterpret_cast<float*>(op.p[3]);
        for (int i = ctid; i < G * dh; i += kConsumers) {
            const int h = i / dh, d = i - h * dh;
            part[((static_cast<long long>(gi) * G + h) * maxs + c) * (dh + kPartHead) + kPartHead + d] = oacc[i];
        }
        if (ctid < G) {
            float M = -INFINITY, L = 0.f;
            for (int w = 0; w < kConsumerWarps; ++w) M = fmaxf(M, mW[w * 8 + ctid]);
            for (int w = 0; w < kConsumerWarps; ++w) {
                const float mw = mW[w * 8 + ctid];
                if (mw != -INFINITY) L += lW[w * 8 + ctid] * __expf(mw - M);
            }
            float* pr = part + ((static_cast<long long>(gi) * G + ctid) * maxs + c) * (dh + kPartHead);
            pr[0] = M;
            pr[1] = L;
        }
        return true;
    }
    // this warp's partial: sub-split c * 8 + warp
    float* part = reinterpret_cast<float*>(op.p[3]);
    const int sub = c * 8 + warp;
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
        if (mt < nks) {
            const int d0 = 16 * mt + g8;
            if (h0 < G) {
                float* pr = part + ((static_cast<long long>(gi) * G + h0) * maxs + sub) * (dh + kPartHead);
                pr[kPartHead + d0] = o[mt][0];
                pr[kPartHead + 8 + d0] = o[mt][2];
            }
            if (h0 + 1 < G) {
                float* pr = part + ((static_cast<long long>(gi) * G + h0 + 1) * maxs + sub) * (dh + kPartHead);
                pr[kPartHead + d0] = o[mt][1];
                pr[kPartHead + 8 + d0] = o[mt][3];
            }
        }
    }
    if (g8 == 0) {  // lanes 0..3: (m, l) of heads h0, h0+1
        if (h0 < G) {
            float* pr = part + ((static_cast<long long>(gi) * G + h0) * maxs + sub) * (dh + kPartHead);
            pr[0] = m0;
            pr[1] = l0;
        }
        if (h0 + 1 < G) {
            float* pr = part + ((static_cast<long long>(gi) * G + h0 + 1) * maxs + sub) * (dh + kPartHead);
            pr[0] = m1;
            pr[1] = l1;
        }
    }
    return true;
}

template <bool kQK, bool kMMA = false>
__device__ void body_attn_split(const StaticParams& P, const et_op& op, const SlotView& si, float* scratch, Ring& ring,
                                int ctid, uint64_t* t_split = nullptr) {
    // Flash-decoding split c of kv head g: its run of CH-position K/V blocks
    // (attn_blocks) arrives through the ring interleaved K0 V0 K1 V1 ...; each
    // block updates an online softmax (scores one (position, head) dot product per
    // thread; per-head running max / sum by one warp; P.V accumulated in registers
    // by the thread owning (head, dim pair)).  The unnormalised partial (m, l, o)
    // per q head goes to the partials buffer; the merge combines the splits.
    constexpr int kOutMax = kQK ? 2 : 1;  // (head, dim pair) outputs per thread: G * dh / 2 <= 256 * kOutMax
    const int warp = ctid >> 5, lane = ctid & 31;
    // i13 = HS > 1 (scalar split with the output projection's merge, flags bit 10): the q heads
    // of a kv head are shared by HS tasks per split (dim 0 of the grid = group * HS + part),
    // each scoring its G / HS heads against the same K/V blocks -- wide groups (Qwen3: 8 q
    // heads per kv head) get HS times the tasks at 1/HS the arithmetic each
    const int HS = (!kMMA && op.i[13] > 1) ? op.i[13] : 1;
    const int dh = op.i[0], Gf = op.i[1], G = Gf / HS, CH = op.i[2], maxs = op.i[5], kvh = op.i[6];
    const long long s = P.binding[op.i[4]];
    int gi = si.coord[0] / HS, c = si.coord[1];  // gi = sequence * kv_heads + kv head, c = split
    const int hb = (si.coord[0] - gi * HS) * G;  // first q head (within the group) of this task
    if constexpr (kMMA) attn_coord(op, si.coord, P.binding, &gi, &c);  // flat batch-dependent grid
    const int g = gi % kvh, bq = gi / kvh;
    const long long rb = static_cast<long long>(bq) * op.i[7];  // this sequence's q / projection row
    const AttnBlocks ab = attn_blocks(op, c, P.binding);
    const int qstride = dh + 4;          // padded rows: heads land on different banks
    const int nvec = dh / 8;             // 16-byte vectors per K/V row
    const int half = dh / 2;
    float* qs = scratch;                 // [G][dh+4]
    float* sc = scratch + G * qstride;   // [G][CH]
    float* st = sc + G * CH;             // [G][4]: running max, running sum, block rescale
    const float* q = reinterpret_cast<const float*>(op.p[0]) + rb + static_cast<long long>(g * Gf + hb) * dh;
    // flags bit 10 (no merge task): the group's last split also folds in the new token
    // -- cache row s, appended by the q/k/v projection this task waited on -- so the
    // partials alone make the attention output and the group's consumer (the output
    // projection's prologue, gemv_merge_prologue) merges them.  Its k/v rows load with q:
    // every load of the prologue is issued before its shared-memory stores (a store
    // through a generic pointer could alias them as far as the compiler knows, and each
    // load would then wait for the previous store -- one L2 round trip apiece).
    const int nsl = attn_splits_base(op, P.binding);
    const bool fold = !kMMA && (op.flags & 1024) && c == (nsl > 0 ? nsl : 1) - 1;
    float* kv_new = st + 4 * G + 8;  // [2][dh] new k, v
    const bool fold_kv = fold && !(kQK && (op.flags & 1));  // (q/k-norm mode: normalised from the raw projection below)
    const long long krow = static_cast<long long>(bq) * op.i[8] + (static_cast<long long>(g) * op.i[3] + s) * dh;
    const uint16_t* kn = reinterpret_cast<const uint16_t*>(op.p[1]) + krow;
    const uint16_t* vn = reinterpret_cast<const uint16_t*>(op.p[2]) + krow;
    const bool kv1 = fold_kv && ctid < dh;  // dh <= kConsumers: one new k / v element per thread
    const float kn0 = kv1 ? bf2f(__ldcg(kn + ctid)) : 0.f, vn0 = kv1 ? bf2f(__ldcg(vn + ctid)) : 0.f;
    // q/k-norm mode (flags bit 0): the norm weights, RoPE frequencies and the raw new k / v of
    // this thread's dimension, loaded with q as well (used below)
    const bool qkm = kQK && (op.flags & 1) != 0;
    const bool knew = qkm && (((op.flags & 2) && c == 0) || fold);  // this task appends the new k / v
    const bool nw = (op.flags & 64) == 0;
    float wq0 = 0.f, wk0 = 0.f, fr0 = 0.f, kr0 = 0.f, vr0 = 0.f;
    const float* kraw = reinterpret_cast<const float*>(op.p[8]) + rb + static_cast<long long>(g) * dh;
    if (qkm && ctid < dh) {
        if (nw) {
            wq0 = __ldg(reinterpret_cast<const float*>(op.p[(op.flags & 2) ? 9 : 5]) + ctid);
            wk0 = __ldg(reinterpret_cast<const float*>(op.p[6]) + ctid);
        }
        if (ctid < dh / 2) fr0 = __ldg(reinterpret_cast<const float*>(op.p[7]) + ctid);
        if (knew) {
            kr0 = __ldcg(kraw + ctid);
            vr0 = __ldcg(kraw + static_cast<long long>(kvh) * dh + ctid);
        }
    }
    for (int i0 = ctid; i0 < G * dh; i0 += 2 * kConsumers) {  // both loads ahead of the stores
        const int i1 = i0 + kConsumers;
        const float a = __ldcg(q + i0), b = i1 < G * dh ? __ldcg(q + i1) : 0.f;
        qs[(i0 / dh) * qstride + i0 % dh] = a;
        if (i1 < G * dh) qs[(i1 / dh) * qstride + i1 % dh] = b;
    }
    if (kv1) {
        kv_new[ctid] = kn0;
        kv_new[dh + ctid] = vn0;
    }
    if (fold_kv)
        for (int d = ctid + kConsumers; d < dh; d += kConsumers) {  // dh > kConsumers (not used by the models)
            kv_new[d] = bf2f(__ldcg(kn + d));
            kv_new[dh + d] = bf2f(__ldcg(vn + d));
        }
    if (ctid < G) {
        st[4 * ctid] = -INFINITY;
        st[4 * ctid + 1] = 0.f;
    }
    if constexpr (kQK) {
        if (op.flags & 1) {  // q-norm + RoPE applied here (q is the raw projection)
            // the q / k norm weights and the RoPE frequencies loaded with q above (one L2
            // round trip; the wait's acquire left L1 cold)
            float* wqs = kv_new + 2 * dh;  // [dh] q-norm, [dh] k-norm, [dh/2] inverse frequencies
            if (ctid < dh) {
                if (nw) {
                    wqs[ctid] = wq0;
                    wqs[dh + ctid] = wk0;
                }
                if (ctid < dh / 2) wqs[2 * dh + ctid] = fr0;
            }
            // fused merge: split 0 also normalises + rotates the new k and appends the
            // new k/v (bf16) to the cache row s before it arrives, so the merger reads
            // them like any cached row
            // no merge task (flags bit 10): the last split does it and keeps them for its fold
            // [2][dh]: sc is scratch before the blocks use it; the tensor-core split keeps them
            // past its per-warp P scratch (attn_solo_finish reads them after the blocks)
            float* kv = fold ? kv_new : kMMA ? sc + kAttnSoloKv : sc;
            if (knew && ctid < dh) {
                kv[ctid] = kr0;
                kv[dh + ctid] = vr0;
            }
            bar_sync(1, kConsumers);
            for (int h = warp; h < G + (knew ? 1 : 0); h += kConsumerWarps)
                qk_norm_rope(h < G ? qs + h * qstride : kv, dh, (op.flags & 64) ? nullptr : wqs + (h < G ? 0 : dh),
                             op.f[1], wqs + 2 * dh, s, lane);
            if (knew) {
                bar_sync(1, kConsumers);
                const long long cb = static_cast<long long>(bq) * op.i[8];
                uint16_t* kc = reinterpret_cast<uint16_t*>(op.p[1]) + cb + (static_cast<long long>(g) * op.i[3] + s) * dh;
                uint16_t* vc = reinterpret_cast<uint16_t*>(op.p[2]) + cb + (static_cast<long long>(g) * op.i[3] + s) * dh;
                const int sw = (op.flags & 256) ? static_cast<int>(s & 7) : 0;  // cache row chunk swizzle
                for (int d = ctid; d < dh; d += kConsumers) {
                    const int dp = ((((d >> 3) ^ sw)) << 3) | (d & 7);
                    const uint16_t kb = f2bf(kv[d]), vb = f2bf(kv[dh + d]);
                    kc[dp] = kb;
                    vc[dp] = vb;
                    kv[d] = bf2f(kb);  // the fold uses the cached (bf16) row, like every later step
                    kv[dh + d] = bf2f(vb);
                }
            }
        }
    }
    bar_sync(1, kConsumers);
    if ((P.debug & 0x1000) && t_split && ctid == 0) *t_split = globaltimer();  // probe: q staged
    if constexpr (kMMA) {
        if (!attn_split_mma(P, op, gi, c, ab, s, qs, qstride, sc, st, ring, ctid)) return;
    } else {
        const float scale = op.f[0];
        float o0[kOutMax], o1[kOutMax];
    #pragma unroll
        for (int j = 0; j < kOutMax; ++j) o0[j] = o1[j] = 0.f;
        for (int blk = 0; blk < ab.nblk; ++blk) {
            const long long pb = ab.p0 + static_cast<long long>(blk) * CH;
            const int np = static_cast<int>(pb + CH < s ? CH : s - pb);
            const unsigned long long ck = ring.seq, cv = ring.seq + 1;
            ring.seq += 2;
            // scores; each position starts its walk over the row at a different 16-byte
            // vector (bank rotation)
            const uint8_t* kb = ring.wait(ck);
            if (!kb) return;
            for (int t = ctid; t < G * np; t += kConsumers) {
                const int h = t % G, p = t / G;
                const uint8_t* kr = kb + p * dh * 2;
                const float* qh = qs + h * qstride;
                float a0 = 0.f, a1 = 0.f;
                for (int v = 0; v < nvec; ++v) {
                    const int vv = (v + p) & (nvec - 1);
                    const uint4 k8 = lds128(kr + vv * 16);
                    const float4 qa = *reinterpret_cast<const float4*>(qh + vv * 8);
                    const float4 qb = *reinterpret_cast<const float4*>(qh + vv * 8 + 4);
                    a0 = fmaf(bf16lo(k8.x), qa.x, a0);
                    a1 = fmaf(bf16hi(k8.x), qa.y, a1);
                    a0 = fmaf(bf16lo(k8.y), qa.z, a0);
                    a1 = fmaf(bf16hi(k8.y), qa.w, a1);
                    a0 = fmaf(bf16lo(k8.z), qb.x, a0);
                    a1 = fmaf(bf16hi(k8.z), qb.y, a1);
                    a0 = fmaf(bf16lo(k8.w), qb.z, a0);
                    a1 = fmaf(bf16hi(k8.w), qb.w, a1);
                }
                sc[h * CH + p] = (a0 + a1) * scale;
            }
            bar_sync(1, kConsumers);
            if ((P.debug & 0x2000) && blk == 0 && t_split && ctid == 0) *t_split = globaltimer();  // probe: scores
            if (ctid == Ring::owner(ck) * 32) ring.release(ck);
            // online softmax statistics per head (warp h), probabilities in place
            for (int h = warp; h < G; h += kConsumerWarps) {
                float m = -INFINITY;
                for (int p = lane; p < np; p += 32) m = fmaxf(m, sc[h * CH + p]);
                m = warp_max(m);
                const float mo = st[4 * h], mn = fmaxf(mo, m);
                float l = 0.f;
                for (int p = lane; p < np; p += 32) {
                    const float e = __expf(sc[h * CH + p] - mn);
                    sc[h * CH + p] = e;
                    l += e;
                }
                l = warp_sum(l);
                if (lane == 0) {
                    const float alpha = __expf(mo - mn);  // 0 on the first block (mo = -inf)
                    st[4 * h] = mn;
                    st[4 * h + 1] = st[4 * h + 1] * alpha + l;
                    st[4 * h + 2] = alpha;
                }
            }
            bar_sync(1, kConsumers);
            // o = alpha * o + P V: one (head, dim pair) per thread (two when G * dh > 512)
            const uint8_t* vb = ring.wait(cv);
            if (!vb) return;
            const uint32_t* v2 = reinterpret_cast<const uint32_t*>(vb);
    #pragma unroll
            for (int j = 0; j < kOutMax; ++j) {
                const int idx = ctid + j * kConsumers;
                if (idx >= G * half) break;
                const int h = idx / half, dp = idx - h * half;
                const float* ph = sc + h * CH;
                const float alpha = st[4 * h + 2];
                float a0 = o0[j] * alpha, a1 = o1[j] * alpha, a2 = 0.f, a3 = 0.f;
                int p = 0;
    #pragma unroll 4
                for (; p + 2 <= np; p += 2) {
                    const uint32_t va = v2[p * half + dp], vb2 = v2[(p + 1) * half + dp];
                    const float wa = ph[p], wb = ph[p + 1];
                    a0 = fmaf(wa, bf16lo(va), a0);
                    a1 = fmaf(wa, bf16hi(va), a1);
                    a2 = fmaf(wb, bf16lo(vb2), a2);
                    a3 = fmaf(wb, bf16hi(vb2), a3);
                }
                if (p < np) {
                    const uint32_t va = v2[p * half + dp];
                    a0 = fmaf(ph[p], bf16lo(va), a0);
                    a1 = fmaf(ph[p], bf16hi(va), a1);
                }
                o0[j] = a0 + a2;
                o1[j] = a1 + a3;
            }
            bar_sync(1, kConsumers);  // sc / st are reused by the next block
            if (ctid == Ring::owner(cv) * 32) ring.release(cv);
        }
        // flags bit 10 (no merge task): the group's last split also folds in the new
        // token -- cache row s, appended by the q/k/v projection this task waited on --
        // so the partials alone make the attention output and the consumer of the
        // group (the output projection's prologue) merges them
        const int nsl = attn_splits_base(op, P.binding);
        if ((P.debug & 0x4000) && t_split && ctid == 0) *t_split = globaltimer();  // probe: blocks done
        if (fold) {
            for (int h = warp; h < G; h += kConsumerWarps) {
                float dot = 0.f;
                for (int d = lane; d < dh; d += 32) dot += qs[h * qstride + d] * kv_new[d];
                const float snew = warp_sum(dot) * scale;
                if (lane == 0) {
                    const float mo = st[4 * h], mn = fmaxf(mo, snew);
                    const float alpha = __expf(mo - mn), en = __expf(snew - mn);
                    st[4 * h] = mn;
                    st[4 * h + 1] = st[4 * h + 1] * alpha + en;
                    st[4 * h + 2] = alpha;
                    st[4 * h + 3] = en;
                }
            }
            bar_sync(1, kConsumers);
    #pragma unroll
            for (int j = 0; j < kOutMax; ++j) {
                const int idx = ctid + j * kConsumers;
                if (idx >= G * half) break;
                const int h = idx / half, dp = idx - h * half;
                const float alpha = st[4 * h + 2], en = st[4 * h + 3];
                o0[j] = fmaf(en, kv_new[dh + 2 * dp], o0[j] * alpha);
                o1[j] = fmaf(en, kv_new[dh + 2 * dp + 1], o1[j] * alpha);
            }
        }
        // the unnormalised partial (m, l, o) of every q head of the group
        float* part = reinterpret_cast<float*>(op.p[3]);
    #pragma unroll
        for (int j = 0; j < kOutMax; ++j) {
            const int idx = ctid + j * kConsumers;
            if (idx >= G * half) break;
            const int h = idx / half, dp = idx - h * half;
            float* pr = part + ((static_cast<long long>(gi) * Gf + hb + h) * maxs + c) * (dh + kPartHead);
            pr[kPartHead + 2 * dp] = o0[j];
            pr[kPartHead + 1 + 2 * dp] = o1[j];
            if (dp == 0) {
                pr[0] = st[4 * h];
                pr[1] = st[4 * h + 1];
            }
        }
    }
    if ((P.debug & 0x7000) == 0 && t_split && ctid == 0) *t_split = globaltimer();  // split work done (trace: prologue stamp)
    if ((op.flags & 2) && !(kMMA && attn_solo(op, P.binding))) {  // fused merge: the split of group g that arrives last merges it
        volatile int* flag = reinterpret_cast<volatile int*>(st + 4 * G);
        bar_sync(1, kConsumers);
        if (ctid == 0) {
            int* arrive = reinterpret_cast<int*>(op.p[5]) + gi;
            // release: this split's partial (CTA writes ordered by the bar above) before
            // the arrival; acquire: the other splits' partials after it
            const int ntask = kMMA ? attn_tasks(op, P.binding) : attn_splits_base(op, P.binding);  // max(splits, 1)
            const bool last = atom_add_acq_rel(arrive, 1) == (ntask > 0 ? ntask : 1) - 1;
            if (last) *reinterpret_cast<volatile int*>(arrive) = 0;  // every split of this step arrived
            *flag = last ? 1 : 0;
        }
        bar_sync(1, kConsumers);
        if (*flag) {
            if ((P.debug & 16) && ctid == 0) ring.stall = globaltimer() - *t_split;  // arrival round trip
            attn_merge_group<kQK, kMMA>(P, op, gi, qs, qstride, st + 4 * G + 4, ctid);
        }
    }
}

// Merge of the splits of one kv head's q heads with the new token at s:
//   O = (sum_c e^(m_c-M) o_c + e^(s_new-M) v_new) / (sum_c e^(m_c-M) l_c + e^(s_new-M)).
// Split statistics are staged in shared memory with independent loads, then
// every (head, dim) output is one thread's dot product over the splits.
template <bool kQK>
__device__ void body_attn_merge(const StaticParams& P, const et_op& op, const SlotView& si, float* scratch, int ctid) {
    const int warp = ctid >> 5, lane = ctid & 31;
    const int dh = op.i[0], G = op.i[1], CH = op.i[2], cap = op.i[3], maxs = attn_part_stride(op);
    const long long s = P.binding[op.i[4]];
    const int nspl = attn_splits_with_data(op, P.binding);
    const int g = si.coord[0];
    const float scale = op.f[0];
    const float* part = reinterpret_cast<const float*>(op.p[3]) + static_cast<long long>(g) * G * maxs * (dh + kPartHead);
    const uint16_t* kn = reinterpret_cast<const uint16_t*>(op.p[1]) + (static_cast<long long>(g) * cap + s) * dh;
    const uint16_t* vn = reinterpret_cast<const uint16_t*>(op.p[2]) + (static_cast<long long>(g) * cap + s) * dh;
    uint16_t* out = reinterpret_cast<uint16_t*>(op.p[4]) + static_cast<long long>(g) * G * dh;
    float* ml = scratch;                // [G][nspl][2]
    float* wts = ml + 2 * G * nspl;     // [G][nspl]
    float* hs = wts + G * nspl;         // [G]: s_new, then e^(s_new-M)/L
    for (int idx = ctid; idx < G * nspl; idx += kConsumers) {
        const float* pr = part + (static_cast<long long>(idx / nspl) * maxs + idx % nspl) * (dh + kPartHead);
        ml[2 * idx] = __ldcg(pr);
        ml[2 * idx + 1] = __ldcg(pr + 1);
    }
    if (kQK && (op.flags & 1)) {
        // Qwen3 mode: q, k, v of the new token are raw projections.  q and k get
        // the per-head RMSNorm + RoPE here; k and v are appended to the cache
        // (bf16) for later steps and read back below like any cached row.
        float* qn = hs + G;  // [G][dh] then [dh] for k
        const float* q = reinterpret_cast<const float*>(op.p[0]) + static_cast<long long>(g) * G * dh;
        const float* kr = reinterpret_cast<const float*>(op.p[8]) + static_cast<long long>(g) * dh;
        const float* vr = kr + static_cast<long long>(op.i[6]) * dh;
        for (int i = ctid; i < (G + 1) * dh; i += kConsumers) qn[i] = i < G * dh ? __ldcg(q + i) : __ldcg(kr + i - G * dh);
        bar_sync(1, kConsumers);
        for (int hh = warp; hh <= G; hh += kConsumerWarps)
            qk_norm_rope(qn + hh * dh, dh, reinterpret_cast<const float*>(op.p[hh < G ? 5 : 6]), op.f[1],
                         reinterpret_cast<const float*>(op.p[7]), s, lane);
        bar_sync(1, kConsumers);
        uint16_t* kc = const_cast<uint16_t*>(kn);
        uint16_t* vc = const_cast<uint16_t*>(vn);
        for (int d = ctid; d < dh; d += kConsumers) {
            kc[d] = f2bf(qn[G * dh + d]);
            vc[d] = f2bf(__ldcg(vr + d));
        }
        bar_sync(1, kConsumers);
        for (int hh = warp; hh < G; hh += kConsumerWarps) {
            float dot = 0.f;
            for (int d = lane; d < dh; d += 32) dot += qn[hh * dh + d] * bf2f(__ldcg(kn + d));
            dot = warp_sum(dot);
            if (lane == 0) hs[hh] = dot * scale;
        }
    } else {
        for (int hh = warp; hh < G; hh += kConsumerWarps) {
            const float* q = reinterpret_cast<const float*>(op.p[0]) + (static_cast<long long>(g) * G + hh) * dh;
            float dot = 0.f;
            for (int d = lane; d < dh; d += 32) dot += __ldcg(q + d) * bf2f(__ldcg(kn + d));
            dot = warp_sum(dot);
            if (lane == 0) hs[hh] = dot * scale;
        }
    }
    bar_sync(1, kConsumers);
    for (int hh = warp; hh < G; hh += kConsumerWarps) {
        const float snew = hs[hh];
        float M = snew;
        for (int c = lane; c < nspl; c += 32) M = fmaxf(M, ml[2 * (hh * nspl + c)]);
        M = warp_max(M);
        float L = 0.f;
        for (int c = lane; c < nspl; c += 32) {
            const float e = __expf(ml[2 * (hh * nspl + c)] - M);
            wts[hh * nspl + c] = e;
            L += e * ml[2 * (hh * nspl + c) + 1];
        }
        const float en = __expf(snew - M);
        L = warp_sum(L) + en;
        const float inv = 1.f / L;
        for (int c = lane; c < nspl; c += 32) wts[hh * nspl + c] *= inv;
        __syncwarp();
        if (lane == 0) hs[hh] = en * inv;
    }
    bar_sync(1, kConsumers);
    for (int idx = ctid; idx < G * dh; idx += kConsumers) {
        const int hh = idx / dh, d = idx % dh;
        const float* ph = part + static_cast<long long>(hh) * maxs * (dh + kPartHead) + kPartHead + d;
        const float* w = wts + hh * nspl;
        float o = hs[hh] * bf2f(__ldcg(vn + d));
#pragma unroll 8
        for (int c = 0; c < nspl; ++c) o = fmaf(w[c], __ldcg(ph + static_cast<long long>(c) * (dh + kPartHead)), o);
        out[idx] = f2bf(o);
    }
}

// ---------------------------------------------------------------------------
// MoE.  Router: the GEMV above on E/16 tasks (logits, RMSNorm prologue), then
// the last task to arrive turns the logits into the routing runtime tensors
// that drive the data-dependent Event Tensors of the layer (ref
// workloads.cpp:81-150: topk, expert_counts, exp_indptr; plus task_indptr,
// eoff and elist for the expert call).  Everything is written before this
// task's NOTIFY (release), and the dynamic scheduler reveals the counts when
// the whole writer call has finished (ref simulate.cpp:632-649).
__device__ __forceinline__ void body_moe_route_impl(const StaticParams& P, const et_op& op, const SlotView& si, uint16_t* xs, float* acc,
                               float* red, Ring& ring, int ctid, uint64_t* t_pro) {
    // flags bit 1: the router logits were accumulated by a tensor-core GEMV (large batch)
    // into p1 (fp32 [b][E], split-K adds): one route task copies them to p4 and zeroes p1
    const bool pre = (op.flags & 2) != 0;
    const int warp = ctid >> 5, lane = ctid & 31;
    const int E = op.i[0], H = op.i[1], K = op.i[6], RS = op.i[12], TS = op.i[13];
    const int nb = batch_of(op, P);
    if (pre) {
        float* lacc = reinterpret_cast<float*>(op.p[1]);
        for (int i = ctid; i < nb * E; i += kConsumers) {
            reinterpret_cast<float*>(op.p[4])[i] = __ldcg(lacc + i);
            lacc[i] = 0.f;
        }
        bar_sync(1, kConsumers);
    } else {
        *t_pro = body_gemv(P, op, si, xs, acc, red, ring, ctid);
        if (si.coord[0] == 0)  // the normalised activations feed the experts
            for (int v = ctid; v < nb * H / 8; v += kConsumers)
                reinterpret_cast<uint4*>(op.p[5])[v] = reinterpret_cast<const uint4*>(xs)[v];
    }
    volatile int* flag = reinterpret_cast<volatile int*>(red + kConsumerWarps);
    const bool single = !pre && si.ext0 == 1;  // one route task: no arrival, logits still in shared memory
    if (!single && !pre) {
        bar_sync(1, kConsumers);
        if (ctid == 0) {
            int* arrive = reinterpret_cast<int*>(op.p[7]);
            const bool last = atom_add_acq_rel(arrive, 1) == si.ext0 - 1;
            if (last) *reinterpret_cast<volatile int*>(arrive) = 0;
            *flag = last ? 1 : 0;
        }
        bar_sync(1, kConsumers);
        if (!*flag) return;
    }

    const int rb = op.i[10];  // the layer's routing tensors: topk, cnt, ind, tind, elist, eoff
    int* topk = P.rt[rb];
    int* cnt = P.rt[rb + 1];
    int* ind = P.rt[rb + 2];
    int* tind = P.rt[rb + 3];
    int* elist = P.rt[rb + 4];
    int* eoff = P.rt[rb + 5];
    const float* logits = reinterpret_cast<const float*>(op.p[4]);
    float* wslot = reinterpret_cast<float*>(op.p[6]);
    int4* tinfo = reinterpret_cast<int4*>(op.p[8]);   // [tiles] (expert, first slot, tokens)
    int* scnt = reinterpret_cast<int*>(acc + (single ? E * nb : 0));  // [E] counts (single: logits in acc[0, E*nb))
    int* stop = scnt + 256;                           // [nb*K] experts per slot
    float* sw = reinterpret_cast<float*>(stop + 256);  // [nb*K] routing weight per slot
    int* tfirst = reinterpret_cast<int*>(sw + 256);    // [E] first tile of a one-token expert, else -1
    for (int e = ctid; e < E; e += kConsumers) scnt[e] = 0;
    bar_sync(1, kConsumers);
    // one warp per token: softmax over E (<= 256), top-K by repeated warp argmax
    constexpr int kPer = 8;
    for (int t = warp; t < nb; t += kConsumerWarps) {
        float lg[kPer];
        float m = -INFINITY;
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int e = lane + 32 * u;
            lg[u] = e < E ? (single ? acc[e * nb + t] : __ldcg(logits + static_cast<long long>(t) * E + e)) : -INFINITY;
            m = fmaxf(m, lg[u]);
        }
        m = warp_max(m);
        float z = 0.f;
#pragma unroll
        for (int u = 0; u < kPer; ++u)
            if (lane + 32 * u < E) z += __expf(lg[u] - m);
        z = warp_sum(z);
        for (int j = 0; j < K; ++j) {
            int e;
            if (op.flags & 1) {  // injected routing (host-written topk)
                e = __ldcg(topk + t * K + j);
            } else {  // selection on the raw logits: larger wins, the lower expert index on ties
                // each lane's best remaining candidate, then two warp reductions (redux.sync):
                // the largest order-preserving key, and the lowest expert index holding it
                float bv = -INFINITY;
                int bi = 1 << 30;
#pragma unroll
                for (int u = 0; u < kPer; ++u)
                    if (lane + 32 * u < E && (lg[u] > bv || bi == (1 << 30))) {
                        bv = lg[u];
                        bi = lane + 32 * u;
                    }
                uint32_t key = __float_as_uint(bv + 0.f);  // -0 -> +0: equal logits tie on the index
                key = (key & 0x80000000u) ? ~key : (key | 0x80000000u);
                const uint32_t kmax = __reduce_max_sync(0xffffffffu, key);
                e = static_cast<int>(__reduce_min_sync(0xffffffffu, key == kmax ? static_cast<uint32_t>(bi) : 0xffffffffu));
                if ((e & 31) == lane) {  // taken: drop it from the candidates
#pragma unroll
                    for (int u = 0; u < kPer; ++u)
                        if (u == (e >> 5)) lg[u] = -INFINITY;
                }
                // the selected logit (sw holds it until the slot's weight replaces it below)
                if (lane == 0) sw[t * K + j] = __uint_as_float((kmax & 0x80000000u) ? (kmax & 0x7fffffffu) : ~kmax);
            }
            if (lane == 0) stop[t * K + j] = e;
        }
        __syncwarp();
        // weights p_e / sum of the selected p, from the selected logits (injected routing:
        // loaded)
        const int ej = lane < K ? stop[t * K + lane] : 0;
        const float lj = lane >= K              ? 0.f
                         : !(op.flags & 1)      ? sw[t * K + lane]
                         : single               ? acc[ej * nb + t]
                                                : __ldcg(logits + static_cast<long long>(t) * E + ej);
        const float wj = lane < K ? __expf(lj - m) / z : 0.f;
        const float wsum = warp_sum(wj);
        if (lane < K) {
            const int slot = t * K + lane;
            if (!(op.flags & 1)) topk[slot] = ej;
            wslot[slot] = wj / wsum;
            sw[slot] = wj / wsum;
            atomicAdd(&scnt[ej], 1);
        }
    }
    bar_sync(1, kConsumers);
    if (warp == 0) {  // exclusive scans over E <= 256 experts (8 per lane)
        int c8[kPer], tiles = 0, toks = 0;
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int e = lane * kPer + u;
            c8[u] = e < E ? scnt[e] : 0;
            tiles += (c8[u] + TS - 1) / TS;
            toks += c8[u];
        }
        int it = tiles, io = toks;  // inclusive warp scans
        for (int o = 1; o < 32; o <<= 1) {
            const int a = __shfl_up_sync(0xffffffffu, it, o), b = __shfl_up_sync(0xffffffffu, io, o);
            if (lane >= o) {
                it += a;
                io += b;
            }
        }
        int tp = it - tiles, op_ = io - toks;
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int e = lane * kPer + u;
            if (e < E) {
                cnt[e] = c8[u];
                ind[e] = tp;
                tind[e] = tp * RS;
                eoff[e] = op_;
                tfirst[e] = c8[u] == 1 ? tp : -1;
                scnt[e] = op_;  // cursor for elist
                for (int i = 0; i * TS < c8[u]; ++i)  // direct tile table for the expert tasks
                    tinfo[tp + i] = make_int4(e, op_ + i * TS, c8[u] - i * TS < TS ? c8[u] - i * TS : TS, 0);
            }
            tp += (c8[u] + TS - 1) / TS;
            op_ += c8[u];
        }
        if (lane == 31) {
            ind[E] = tp;
            tind[E] = tp * RS;
            eoff[E] = op_;
        }
    }
    bar_sync(1, kConsumers);
    if (ctid == 0)  // slots grouped by expert, stable in slot order
        for (int sl = 0; sl < nb * K; ++sl) {
            const int e = stop[sl];
            elist[scnt[e]++] = sl;
            // a one-token tile carries its slot's routing weight (int4 .w, float bits): its
            // expert tasks skip the elist / weight lookups (one L2 round trip instead of three)
            if (tfirst[e] >= 0) tinfo[tfirst[e]].w = __float_as_int(sw[sl]);
        }
    // The selected experts' weights cannot be streamed before this point (their ids
    // exist only now); start pulling them into L2 while the expert tasks get
    // released.  (Plain writes above are published by the task's NOTIFY release.)
    if (op.p[9]) {
        const long long mat = static_cast<long long>(op.i[8]) * H * 2;  // one expert matrix: I x H bf16
        for (int i = ctid; i < 3 * E; i += kConsumers) {
            const int e = i / 3, m = i - 3 * e;
            if (cnt[e] > 0) {
                const uint8_t* base = reinterpret_cast<const uint8_t*>(op.p[9 + m]) + e * mat;
                for (long long off = 0; off < mat; off += (1 << 20))
                    bulk_prefetch_l2(base + off, static_cast<uint32_t>(mat - off < (1 << 20) ? mat - off : (1 << 20)));
            }
        }
    }
}

// Inlined into the MoE kernels (its registers are free there); out of line in the
// MoE + tensor-core kernels, whose other bodies already fill the register budget.
template <bool kOutOfLine>
__device__ __forceinline__ void body_moe_route(const StaticParams& P, const et_op& op, const SlotView& si, uint16_t* xs,
                                               float* acc, float* red, Ring& ring, int ctid, uint64_t* t_pro) {
    body_moe_route_impl(P, op, si, xs, acc, red, ring, ctid, t_pro);
}
template <>
__device__ __noinline__ void body_moe_route<true>(const StaticParams& P, const et_op& op, const SlotView& si,
                                                  uint16_t* xs, float* acc, float* red, Ring& ring, int ctid,
                                                  uint64_t* t_pro) {
    body_moe_route_impl(P, op, si, xs, acc, red, ring, ctid, t_pro);
}

// Routed expert task (see expert_task): gate/up rows of its row split for the
// tile's tokens, SiLU-mul, then the matching column block of the down
// projection, added into the residual stream with the routing weight.
__device__ uint64_t body_moe_expert(const StaticParams& P, const et_op& op, const SlotView& si, uint16_t* xs,
                                    float* acc, Ring& ring, int ctid) {
    const int warp = ctid >> 5, lane = ctid & 31;
    const int I = op.i[0], H = op.i[1], RS = op.i[2], K = op.i[8];
    const int IR = I / RS;
    int* stok = reinterpret_cast<int*>(acc + kAccFloats - 16);     // [8] token of each tile row
    float* swt = acc + kAccFloats - 8;                             // [8] its routing weight
    int nb;
    const uint16_t* xn = reinterpret_cast<const uint16_t*>(op.p[3]);
    if (op.i[9] < 0) {
        // one sequence (i9 = -1): every tile is token 0 with one slot, whose routing weight the
        // route task left in the tile record -- the record and the activations load together
        const int4 info = __ldcg(reinterpret_cast<const int4*>(op.p[6]) + si.coord[0] / op.i[2]);
        for (int v = ctid; v < H / 8; v += kConsumers)
            reinterpret_cast<uint4*>(xs)[v] = __ldcg(reinterpret_cast<const uint4*>(xn) + v);
        nb = 1;
        if (ctid == 0) {
            stok[0] = 0;
            swt[0] = __int_as_float(info.w);
        }
        bar_sync(1, kConsumers);
    } else {
        {
            const ExpertTask t = expert_task(op, si.coord[0], P.rt);
            nb = t.ntok;
            if (ctid < nb) {
                stok[ctid] = t.slot[ctid] / K;
                swt[ctid] = __ldcg(reinterpret_cast<const float*>(op.p[4]) + t.slot[ctid]);
            }
        }
        bar_sync(1, kConsumers);
        for (int v = ctid; v < nb * H / 8; v += kConsumers) {
            const int j = v / (H / 8), k8 = v - j * (H / 8);
            reinterpret_cast<uint4*>(xs)[v] =
                __ldcg(reinterpret_cast<const uint4*>(xn + static_cast<long long>(stok[j]) * H) + k8);
        }
    }
    for (int i = ctid; i < 2 * IR * nb; i += kConsumers) acc[i] = 0.f;
    bar_sync(1, kConsumers);
    const uint64_t t_pro = ctid == 0 ? globaltimer() : 0;
    gemv_stream(ring, warp, lane, 2, (IR / 16) * (H / 16), 0, H, nb, xs,
                [&](int seg, int rt, int g, int q, const float* d) {
                    const int row = seg * IR + rt * 16 + g;
                    if (2 * q < nb) {
                        atomicAdd(&acc[row * nb + 2 * q], d[0]);
                        atomicAdd(&acc[(row + 8) * nb + 2 * q], d[2]);
                    }
                    if (2 * q + 1 < nb) {
                        atomicAdd(&acc[row * nb + 2 * q + 1], d[1]);
                        atomicAdd(&acc[(row + 8) * nb + 2 * q + 1], d[3]);
                    }
                });
    bar_sync(1, kConsumers);
    uint16_t* xa = reinterpret_cast<uint16_t*>(acc + 2 * IR * 8);  // act [nb][IR] bf16
    for (int idx = ctid; idx < IR * nb; idx += kConsumers) {
        const int i = idx / nb, j = idx - i * nb;
        const float gv = acc[i * nb + j], uv = acc[(IR + i) * nb + j];
        xa[j * IR + i] = f2bf(gv / (1.f + __expf(-gv)) * uv);
    }
    bar_sync(1, kConsumers);
    float* h = reinterpret_cast<float*>(op.p[5]);
    gemv_stream(ring, warp, lane, 1, (H / 16) * (IR / 16), 0, IR, nb, xa,
                [&](int, int rt, int g, int q, const float* d) {
                    const int row = rt * 16 + g;
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const int j = 2 * q + c;
                        if (j < nb) {
                            const float w = swt[j];
                            float* hr = h + static_cast<long long>(stok[j]) * H;
                            atomicAdd(hr + row, w * d[c]);
                            atomicAdd(hr + row + 8, w * d[2 + c]);
                        }
                    }
                });
    return t_pro;
}

// ---------------------------------------------------------------------------
// Tensor-parallel allreduce task (row-parallel output projection / down
// projection).  Every rank wrote its partial product of the stage into its own
// `part` slot (EPI_F32); this task adds the partials of all TP ranks into rows
// [r0, r1) of the local residual stream.  The cross-GPU dependency is an Event
// Tensor element per (stage slot, source rank) living in each destination
// rank's memory: the first allreduce task of a rank to run (its local stage is
// complete -- the task waited on it) stores the step epoch into that element
// on every rank with st.release.sys; every task spins with ld.acquire.sys until
// all TP sources reached the epoch, then reads the peers' partials over NVLink.
// Epochs (the step id, identical on all ranks) make resets unnecessary.
__device__ void body_allreduce(const StaticParams& P, const et_op& op, const SlotView& si, int ctid, int worker) {
    const int H = op.i[0], TP = op.i[1], rank = op.i[2], slot = op.i[3];
    const uint32_t epoch = static_cast<uint32_t>(P.step_id);
    float* h = reinterpret_cast<float*>(op.p[0]);
    uint32_t* flags = reinterpret_cast<uint32_t*>(op.p[1]);          // local [slots][TP]
    uint32_t* once = reinterpret_cast<uint32_t*>(op.p[2]);           // local [slots]
    const unsigned long long* peers = reinterpret_cast<const unsigned long long*>(op.p[3]);  // [TP][2]: part, flags
    if (ctid == 0 && atomicMax(once + slot, epoch) < epoch) {
        for (int p = 0; p < TP; ++p) {
            uint32_t* pf = reinterpret_cast<uint32_t*>(__ldg(peers + 2 * p + 1)) + slot * TP + rank;
            st_release_sys(pf, epoch);
        }
    }
    if (ctid < TP) {
        const uint32_t* f = flags + slot * TP + ctid;
        const uint64_t t0 = globaltimer();
        uint32_t it = 0;
        while (static_cast<int>(ld_relaxed_sys(f) - epoch) < 0) {
            if ((++it & 255u) == 0) {
                if (aborted(P.status)) break;
                if (globaltimer() - t0 > static_cast<uint64_t>(P.watchdog_ns)) {
                    report(P.status, ET_ERR_DEADLOCK, worker, -5, slot * TP + ctid, static_cast<int>(epoch));
                    break;
                }
            }
        }
        fence_acquire_sys();
    }
    bar_sync(1, kConsumers);
    const int T = si.ext0, t = si.coord[0];
    const int n4 = H / 4;
    const int a = static_cast<int>(static_cast<long long>(t) * n4 / T), b = static_cast<int>(static_cast<long long>(t + 1) * n4 / T);
    for (int i = a + ctid; i < b; i += kConsumers) {
        float4 acc = ldcg_f4(h + 4 * i);
        for (int p = 0; p < TP; ++p) {
            const float* part = reinterpret_cast<const float*>(__ldg(peers + 2 * p)) + static_cast<long long>(slot) * H;
            const float4 v = ld_cv_f4(part + 4 * i);
            acc.x += v.x;
            acc.y += v.y;
            acc.z += v.z;
            acc.w += v.w;
        }
        *reinterpret_cast<float4*>(h + 4 * i) = acc;
    }
}

__device__ void body_embed(const StaticParams& P, const et_op& op, int ctid) {
    const int H = op.i[0];
    const int nb = op.i[1] >= 0 ? static_cast<int>(P.binding[op.i[1]]) : 1;
    // flags bit 0: this step's greedy-argmax words (p3, one per sequence) start at 0; every
    // lm_head task waits on this task through the layer chain
    if ((op.flags & 1) && ctid < nb) reinterpret_cast<unsigned long long*>(op.p[3])[ctid] = 0ull;
    const uint4* __restrict__ table = reinterpret_cast<const uint4*>(op.p[0]);
    const int* tok = reinterpret_cast<const int*>(op.p[1]);
    float4* __restrict__ out = reinterpret_cast<float4*>(op.p[2]);
    // 16-byte vectors (8 bf16 -> 8 fp32) over (sequence, vector); restrict lets the loads of
    // later vectors issue ahead of earlier stores -- element-wise loads each waited behind the
    // previous store, a memory round trip per element (12 us on the critical path at H = 4096)
    const int hv = H / 8, nv = nb * hv;  // H % 8 == 0
#pragma unroll 2
    for (int v = ctid; v < nv; v += kConsumers) {
        const int bi = v / hv;
        const uint4 w = __ldg(table + static_cast<long long>(__ldcg(tok + bi)) * hv + (v - bi * hv));
        out[2 * v] = make_float4(bf16lo(w.x), bf16hi(w.x), bf16lo(w.y), bf16hi(w.y));
        out[2 * v + 1] = make_float4(bf16lo(w.z), bf16hi(w.z), bf16lo(w.w), bf16hi(w.w));
    }
}

// ET_OP_ARGMAX: task (0): the greedy token of each sequence from the argmax words the
// lm_head epilogue (GEMV flags bit 5) left at p0 -> int32 p1[b] (and, when p2 is set,
// the next step's token input), words re-zeroed.  i0 = batch symbol slot (-1: 1).
__device__ void body_argmax(const StaticParams& P, const et_op& op, int ctid) {
    const int nb = op.i[0] >= 0 ? static_cast<int>(P.binding[op.i[0]]) : 1;
    if (ctid < nb) {
        unsigned long long* w = reinterpret_cast<unsigned long long*>(op.p[0]);
        const int tok = argmax_row(__ldcg(w + ctid));
        reinterpret_cast<int*>(op.p[1])[ctid] = tok;
        if (op.p[2]) reinterpret_cast<int*>(op.p[2])[ctid] = tok;
        w[ctid] = 0ull;
    }
}

// ET_OP_REDUCE (f4, GEMM + reduce-scatter): output tile (token block j, row group g) =
// the sum of the k-split partial buffers, once every split's GEMM tile of it notified.
__device__ void body_reduce(const StaticParams&, const et_op& op, const int* coord, int ctid) {
    const int N = op.i[0], TB = op.i[1], parts = op.i[2], RG = op.i[4];
    const long long pstride = static_cast<long long>(op.i[3]);
    const int j = coord[0], g = coord[1];
    const float* part = reinterpret_cast<const float*>(op.p[0]);
    const int per_row = RG / 4;  // float4 per token row of the tile
    for (int v = ctid; v < TB * per_row; v += kConsumers) {
        const int n = v / per_row, c4 = v - n * per_row;
        const long long o = (static_cast<long long>(j) * TB + n) * N + static_cast<long long>(g) * RG + c4 * 4;
        float4 acc = ldcg_f4(part + o);
        for (int r = 1; r < parts; ++r) {
            const float4 x = ldcg_f4(part + r * pstride + o);
            acc.x += x.x;
            acc.y += x.y;
            acc.z += x.z;
            acc.w += x.w;
        }
        if (op.i[5] == 1) {
            uint2 b;
            b.x = static_cast<uint32_t>(f2bf(acc.x)) | (static_cast<uint32_t>(f2bf(acc.y)) << 16);
            b.y = static_cast<uint32_t>(f2bf(acc.z)) | (static_cast<uint32_t>(f2bf(acc.w)) << 16);
            *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(op.p[1]) + o) = b;
        } else {
            *reinterpret_cast<float4*>(reinterpret_cast<float*>(op.p[1]) + o) = acc;
        }
    }
}

// ET_OP_COPY (f4, all-gather + GEMM; DMA-class tasks, one warp): chunk t of i0 bytes
// (16-byte multiple) from p0 + t * i0 to p1 + t * i0 (flags bit 0: source chunk t at p2[t],
// a table of per-rank source addresses -- the peers' buffers).
// flags bit 1 (pull-based all-gather): no copy -- the consumers' TMA loads read the chunk
// in place (over NVLink on a TP node); this task only pulls it into L2 ahead of them
// (bulk L2 prefetches, 1 MB each) and releases its arrival element.
__device__ void body_copy(const et_op& op, int t, int lane) {
    const long long bytes = op.i[0];
    if (op.flags & 2) {
        const uint8_t* src = (op.flags & 1)
                                 ? reinterpret_cast<const uint8_t*>(reinterpret_cast<const unsigned long long*>(op.p[2])[t])
                                 : reinterpret_cast<const uint8_t*>(op.p[0]) + t * bytes;
        for (long long off = static_cast<long long>(lane) << 20; off < bytes; off += 32ll << 20)
            bulk_prefetch_l2(src + off, static_cast<uint32_t>(bytes - off < (1 << 20) ? bytes - off : (1 << 20)));
        return;
    }
    const uint4* src = reinterpret_cast<const uint4*>(
        (op.flags & 1) ? reinterpret_cast<const uint8_t*>(reinterpret_cast<const unsigned long long*>(op.p[2])[t])
                       : reinterpret_cast<const uint8_t*>(op.p[0]) + t * bytes);
    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(op.p[1]) + t * bytes);
    const long long n = bytes / 16;
    long long i = lane;
    for (; i + 96 < n; i += 128) {  // four 16-byte loads in flight per lane
        const uint4 a = __ldcg(src + i), b = __ldcg(src + i + 32), c = __ldcg(src + i + 64), d = __ldcg(src + i + 96);
        dst[i] = a;
        dst[i + 32] = b;
        dst[i + 64] = c;
        dst[i + 96] = d;
    }
    for (; i < n; i += 32) dst[i] = __ldcg(src + i);
}

// ---------------------------------------------------------------------------

__device__ __forceinline__ bool op_streams(int kind) {
    return kind == ET_OP_GEMV || kind == ET_OP_ATTN_SPLIT || kind == ET_OP_MOE_ROUTE || kind == ET_OP_MOE_EXPERT ||
           kind == ET_OP_GEMV_TC;
}

// kMoE: the MoE bodies are compiled into this instantiation.  The dense
// instantiation keeps them out of the register allocation of the GEMV loop.
template <bool kMoE, bool kTC>
__device__ void consumer_loop(const StaticParams& P, int worker, uint8_t* smem, const SlotTable& T) {
    const int ctid = threadIdx.x;
    TcState ts{kTC ? reinterpret_cast<volatile uint32_t*>(smem + kSmemMisc)[8] : 0u, 0u, 0u};
    uint16_t* xs = reinterpret_cast<uint16_t*>(smem + kSmemX);
    float* acc = reinterpret_cast<float*>(smem + kSmemAcc);
    volatile int* misc = reinterpret_cast<volatile int*>(smem + kSmemMisc);
    float* red = reinterpret_cast<float*>(smem + kSmemMisc + 64);
    Ring ring{smem + kSmemRing, reinterpret_cast<uint64_t*>(smem + kSmemBar),
              reinterpret_cast<uint64_t*>(smem + kSmemBar) + kStages, 0ull, P.status, P.watchdog_ns, worker};
    ring.dbg = (P.debug & 522) != 0 && P.record;
    const int qb = __ldg(P.queue_off + worker), qe = __ldg(P.queue_off + worker + 1);
    unsigned long long executed = 0, noops = 0;
    for (int s = qb; s < qe; ++s) {
        uint64_t t_begin = 0, t_wait = 0, t_pro = 0, t_exec = 0;
        if (ctid == 0) t_begin = globaltimer();
        SlotView v = view_slot(P, T, s, qb);
        // The op record is copied into shared memory while thread 0 spins on the
        // dependency: the acquire that ends the wait invalidates L1, and every
        // body reads its op fields first (an L2 round trip on the critical path).
        const et_op& opg = P.ops[v.call];
        if (ctid >= 32 && ctid < 32 + static_cast<int>(sizeof(et_op) / 4))
            reinterpret_cast<int*>(smem + kSmemOp)[ctid - 32] = reinterpret_cast<const int*>(&opg)[ctid - 32];
        // likewise the constant operands of a GEMV: RMSNorm gamma (behind the staged
        // activations) and the RoPE inverse frequencies
        if (opg.kind == ET_OP_GEMV && !v.masked && ctid > 0) {
            if (gemv_gamma_staged(opg, P)) {
                const int K = opg.i[1];
                float4* dst = reinterpret_cast<float4*>(xs + gamma_offset(opg, P));
                const float4* src = reinterpret_cast<const float4*>(opg.p[3]);
                for (int i = ctid - 1; i < K / 4; i += kConsumers - 1) dst[i] = __ldg(src + i);
            }
            if (opg.i[4] == EPI_QKV_ROPE)
                for (int i = ctid - 1; i < opg.i[8] / 2; i += kConsumers - 1)
                    reinterpret_cast<float*>(smem + kSmemPre)[i] = __ldg(reinterpret_cast<const float*>(opg.p[8]) + i);
        }
        const et_op& op = *reinterpret_cast<const et_op*>(smem + kSmemOp);
        int first_notify = -1;
        if (ctid == 0) {
            if (v.ne > v.nb) first_notify = __ldg(P.notifies + v.nb);
            misc[12] = s;  // the wait episode (L2 run-ahead)
            misc[2] = 1;  // consumers blocked on an Event Tensor: HBM idles, the producer may fill L2
            bool ok = (P.debug & 1) ? true : wait_range(P, v.wb, v.we, s, worker);
            misc[2] = 0;
            if (ok && P.step_limit > 0 &&
                atomicAdd(&P.status->executed, 1ull) >= static_cast<unsigned long long>(P.step_limit)) {
                report(P.status, ET_ERR_STEP_LIMIT, worker, s, -1, 0);
                ok = false;
            }
            misc[0] = ok ? 0 : 1;
            misc[1] = s + 1;  // releases the producer when prefetch is off
            t_wait = globaltimer();
        }
        bar_sync(1, kConsumers);
        if (misc[0]) break;
        if (v.lazy && !v.masked) v.masked = extent_masked(P, v.call, v.coord);
        if (v.masked) {
            ++noops;
        } else {
            ++executed;
            switch (op.kind) {
                case ET_OP_NONE:
                    if (ctid == 0 && P.tick_ns > 0 && P.slot_duration) {
                        const uint64_t until = t_wait + static_cast<uint64_t>(__ldg(P.slot_duration + s)) *
                                                            static_cast<uint64_t>(P.tick_ns);
                        while (globaltimer() < until) {
                        }
                    }
                    break;
                case ET_OP_SPLITK_PARTIAL:
                case ET_OP_SPLITK_FINAL: body_splitk(P, op, v.coord, ctid); break;
                case ET_OP_GEMV:
                    if (!gemv_fits(op, P)) {
                        if (ctid == 0) report(P.status, ET_ERR_INVALID, worker, s, -1, batch_of(op, P));
                        break;
                    }
                    t_pro = body_gemv(P, op, v, xs, acc, red, ring, ctid, reinterpret_cast<const float*>(smem + kSmemPre));
                    break;
                case ET_OP_ATTN_SPLIT:
                    body_attn_split<kMoE || kTC, kTC>(P, op, v, reinterpret_cast<float*>(xs), ring, ctid, &t_pro);
                    break;
                case ET_OP_ATTN_MERGE: body_attn_merge<kMoE || kTC>(P, op, v, reinterpret_cast<float*>(xs), ctid); break;
                case ET_OP_GEMV_TC:
                    if constexpr (kTC) t_pro = body_gemv_tc(P, op, v, smem, ring, ts, ctid);
                    break;
                case ET_OP_NORM:
                    if constexpr (kTC) body_norm(P, op, v, red, ctid);
                    break;
                case ET_OP_EMBED: body_embed(P, op, ctid); break;
                case ET_OP_ARGMAX: body_argmax(P, op, ctid); break;
                case ET_OP_REDUCE: body_reduce(P, op, v.coord, ctid); break;
                case ET_OP_COPY:  // copies are DMA-class tasks (dma_loop)
                    if (ctid == 0) report(P.status, ET_ERR_INVALID, worker, -1, -7, op.kind);
                    break;
                case ET_OP_ALLREDUCE: body_allreduce(P, op, v, ctid, worker); break;
                case ET_OP_MOE_ROUTE:
                    if constexpr (kMoE) body_moe_route<kTC>(P, op, v, xs, acc, red, ring, ctid, &t_pro);
                    break;
                case ET_OP_MOE_EXPERT:
                    if constexpr (kMoE) t_pro = body_moe_expert(P, op, v, xs, acc, ring, ctid);
                    break;
                default: break;
            }
        }
        bar_sync(1, kConsumers);
        if (ctid == 0) {
            t_exec = globaltimer();
            notify_range(P, v.nb, v.ne, s, worker, first_notify);
            if (P.record) {
                et_trace_rec r;
                r.t_push = 0;
                r.t_begin = static_cast<int64_t>(t_begin);
                r.t_wait_end = static_cast<int64_t>(t_wait);
                r.t_prologue = static_cast<int64_t>(t_pro);
                r.t_exec_end = static_cast<int64_t>(t_exec);
                r.t_notify_end = static_cast<int64_t>(globaltimer());
                r.worker = worker;
                r.flags = v.masked ? 1 : 0;
                r.task = s;
                r.pad = (P.debug & 512) ? static_cast<int>(ring.xwait)
                        : (P.debug & 8) ? static_cast<int>(ring.busy)
                        : (P.debug & 18) ? static_cast<int>(ring.stall) : 0;
                ring.stall = 0;
                ring.busy = 0;
                ring.xwait = 0;
                P.trace[s] = r;
            }
        }
    }
    if (ctid == 0) {
        misc[11] = 1;  // queue done: the L2 run-ahead warp exits
        if (P.step_limit <= 0) atomicAdd(&P.status->executed, executed);
        atomicAdd(&P.status->noops, noops);
    }
}

// Producer side of a tensor-core GEMV task: per piece p, the activation piece X(p)
// into x slot xq % nxs (once the issuer freed it) and the weight chunks of every
// (segment, block) into the ring; piece 0 streams up to kStages weight chunks
// before X(0), which -- produced upstream -- may only load once the task's waits
// passed (dep 0: static slot `key` done waiting, misc[1] > key; dep 1: dynamic
// task generation `key`, misc[6] == key).  Pointer walks only: this thread's
// scalar work is on the streaming critical path.
__device__ __noinline__ bool tc_produce(const StaticParams& P, uint8_t* smem, const StreamPlan& pl,
                                        volatile int* misc, int dep, int key, unsigned long long& cseq,
                                        unsigned int& xq, int worker, uint64_t pol) {
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSmemBar);
    uint64_t* empty = full + kStages;
    uint64_t* bars = tc_bars(smem);
    // the plan's fields in registers (the plan itself sits in local memory)
    const uint8_t* const base0 = pl.base[0];
    const uint8_t* const base1 = pl.nseg > 1 ? pl.base[1] : pl.base[0];
    const long long pstride = pl.tc_pstride;
    const uint8_t* const xsrc = pl.tc_x;
    const uint32_t xbytes = pl.tc_xbytes;
    const int np = pl.tc_np, tw = pl.tc_w, pre = pl.tc_pre, nseg = pl.nseg;
    const int nxs = tc_xslots(xbytes);
    const int per_seg = static_cast<int>(pl.bytes[0] >> 14);  // 16 KB chunks per segment and piece
    const bool fast = (P.debug & 4) != 0, xfast = (P.debug & 256) != 0;
    const uint32_t ring0 = smem_u32(smem + kSmemRing);
    bool fenced = false;
    for (int p = 0; p < np; ++p) {
        int w = 0;
        const uint8_t* src = base0 + p * pstride;
        int sg = 0, left = per_seg;
        for (int half = 0; half < 2; ++half) {
            const int stop = half ? tw : (p == 0 ? pre : 0);
            for (; w < stop; ++w) {
                const int stage = static_cast<int>(cseq % kStages);
                const uint32_t phase = static_cast<uint32_t>((cseq / kStages) & 1ull);
                ++cseq;
                uint32_t spins = 0;
                uint64_t t0 = 0;
                while (!mbar_try_wait(&empty[stage], phase ^ 1u)) {
                    if ((++spins & 1023u) == 0) {
                        if (aborted(P.status)) return false;
                        if (t0 == 0) t0 = globaltimer();
                        else if (globaltimer() - t0 > static_cast<uint64_t>(P.watchdog_ns)) {
                            report(P.status, ET_ERR_DEADLOCK, worker, -1, -3, w);
                            return false;
                        }
                    }
                }
                if (fast) {
                    mbar_arrive(&full[stage]);
                } else {
                    mbar_arrive_expect_tx(&full[stage], kTcChunk);
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, "
                        "[%3], %4;" ::"r"(ring0 + stage * kStageBytes),
                        "l"(src), "r"(kTcChunk), "r"(smem_u32(&full[stage])), "l"(pol)
                        : "memory");
                }
                src += kTcChunk;
                if (--left == 0 && ++sg < nseg) {
                    src = base1 + p * pstride;
                    left = per_seg;
                }
            }
            if (half) break;
            // X(p)
            if (!fenced) {
                for (uint32_t it = 0; dep == 0 ? misc[1] <= key : misc[6] != key;)
                    if ((++it & 1023u) == 0 && aborted(P.status)) return false;
                __threadfence();             // the pieces were written by other CTAs before the waits passed
                fence_proxy_async_global();  // ... with generic stores; the bulk copy reads through the async proxy
                fenced = true;
            }
            const int b = static_cast<int>(xq % nxs);
            const uint32_t par = ((xq / nxs) & 1u) ^ 1u;
            uint32_t spins = 0;
            uint64_t t0 = 0;
            while (!mbar_try_wait(&bars[kTcXSlots + b], par)) {
                if ((++spins & 1023u) == 0) {
                    if (aborted(P.status)) return false;
                    if (t0 == 0) t0 = globaltimer();
                    else if (globaltimer() - t0 > static_cast<uint64_t>(P.watchdog_ns)) {
                        report(P.status, ET_ERR_DEADLOCK, worker, -1, -6, static_cast<int>(xq));
                        return false;
                    }
                }
            }
            if (xfast) {  // timing experiment: x slots "fill" instantly
                mbar_arrive(&bars[b]);
            } else {
                mbar_arrive_expect_tx(&bars[b], xbytes);
                bulk_g2s_keep(smem + kSmemX + b * xbytes, xsrc + static_cast<long long>(p) * xbytes, xbytes, &bars[b]);
            }
            ++xq;
        }
    }
    return true;
}

__device__ void producer_loop(const StaticParams& P, int worker, uint8_t* smem, const SlotTable& T) {
    if ((threadIdx.x & 31) != 0) return;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSmemBar);
    uint64_t* empty = full + kStages;
    volatile int* misc = reinterpret_cast<volatile int*>(smem + kSmemMisc);
    const uint64_t pol = policy_evict_first();
    const int qb = __ldg(P.queue_off + worker), qe = __ldg(P.queue_off + worker + 1);
    unsigned long long cseq = 0;  // chunks issued to the ring
    unsigned int xq = 0;          // activation pieces issued to the tensor-core x buffers
    long long pcum = 0;           // bytes of non-lazy chunks issued (the L2 run-ahead warp's reference)
    for (int s = qb; s < qe; ++s) {
        SlotView v = view_slot(P, T, s, qb);
        if (v.masked) continue;
        const et_op& op = P.ops[v.call];
        if (!op_streams(op.kind)) continue;
        if (!P.prefetch || v.lazy) {
            // data-dependent extents are known only once the slot's waits pass
            for (uint32_t it = 0; misc[1] <= s;) {
                if ((++it & 1023u) == 0 && aborted(P.status)) return;  // (a global load: not every spin)
                __nanosleep(32);  // routed slots wait microseconds: leave the issue slots to the consumers
            }
            if (v.lazy && extent_masked(P, v.call, v.coord)) continue;
        }
        const StreamPlan pl = make_plan(op, v.coord, v.ext0, P.binding, P.rt);
        if (pl.tc_np) {  // tensor-core GEMV: weight chunks + activation pieces (gated on the waits)
            // tiled GEMM (f4): every token block re-reads the weights -- keep them in L2
            // (evict_last) instead of streaming them through it (debug bit 0x400000: evict_first)
            const uint64_t wpol = (tc_tiled(op) && !(P.debug & 0x400000)) ? policy_evict_last() : pol;
            if (!tc_produce(P, smem, pl, misc, 0, s, cseq, xq, worker, wpol)) return;
            continue;
        }
        const int n = pl.total_chunks();
        for (int c = 0; c < n; ++c, ++cseq) {
            const int stage = static_cast<int>(cseq % kStages);
            const uint32_t phase = static_cast<uint32_t>((cseq / kStages) & 1ull);
            uint32_t spins = 0;
            uint64_t t0 = 0;
            while (!mbar_try_wait(&empty[stage], phase ^ 1u)) {
                if ((++spins & 1023u) == 0) {
                    if (aborted(P.status)) return;
                    if (t0 == 0) t0 = globaltimer();
                    else if (globaltimer() - t0 > static_cast<uint64_t>(P.watchdog_ns)) {
                        report(P.status, ET_ERR_DEADLOCK, worker, s, -3, c);
                        return;
                    }
                }
            }
            const Chunk ch = pl.chunk(c);
            misc[9] = s;
            misc[10] = c;
            if (!v.lazy) {
                pcum += ch.bytes;
                reinterpret_cast<volatile long long*>(misc)[7] = pcum;
            }
            if (P.debug & 4) {  // timing experiment: stages "fill" instantly (no HBM traffic)
                mbar_arrive(&full[stage]);
            } else {
                mbar_arrive_expect_tx(&full[stage], ch.bytes);
                bulk_g2s(smem + kSmemRing + stage * kStageBytes, ch.src, ch.bytes, &full[stage], pol);
            }
        }
    }
}

// L2 run-ahead by warp 9 (static scheduler, workers without a DMA queue).  While
// the consumers sit in an Event Tensor wait (misc[2]) the prefetch warp walks
// the slots ahead of the producer and prefetches their bytes into L2 with
// prefetch.global.L2 (one 128-byte line per lane per instruction), keeping at
// most P.l2_ahead bytes in front of the producer's ring position.  Positions
// are compared as cumulative bytes of the non-lazy streaming chunks: the
// producer publishes its count (misc64[7]) and its (slot, chunk) (misc[9],
// misc[10]); a prefetch cursor that fell behind jumps to the producer.  The
// LSU path keeps the prefetches out of the TMA unit, so the ring's own bulk
// copies never queue behind them.  Data-dependent (lazy) slots are skipped
// (debug bit 32: the walk stops at them instead).
__device__ void l2_ahead_loop(const StaticParams& P, int worker, uint8_t* smem, const SlotTable& T) {
    volatile int* misc = reinterpret_cast<volatile int*>(smem + kSmemMisc);
    volatile long long* pbytes = reinterpret_cast<volatile long long*>(smem + kSmemMisc) + 7;
    const int lane = threadIdx.x & 31;
    const int qb = __ldg(P.queue_off + worker), qe = __ldg(P.queue_off + worker + 1);
    const bool stop_lazy = (P.debug & 32) != 0;
    int slot = qb, chunk = 0, n = -1;
    long long fbytes = 0;  // cumulative bytes up to the cursor
    StreamPlan pl;
    for (uint32_t it = 0; misc[11] == 0 && slot < qe;) {
        if ((++it & 1023u) == 0 && aborted(P.status)) return;
        const long long pb = *pbytes;
        if (pb > fbytes) {  // behind the producer: continue from its position
            const int ps = misc[9], pc = misc[10];
            if (ps != slot) n = -1;
            slot = ps < qb ? qb : ps;
            chunk = pc + 1;
            fbytes = pb;
        }
        if (misc[2] == 0 || fbytes - pb >= P.l2_ahead) {
            __nanosleep(64);
            continue;
        }
        if (n < 0) {
            const SlotView v = view_slot(P, T, slot, qb);
            const et_op& op = P.ops[v.call];
            if (v.lazy && stop_lazy) {
                __nanosleep(64);
                continue;
            }
            if (v.masked || v.lazy || !op_streams(op.kind)) {
                ++slot;
                chunk = 0;
                continue;
            }
            pl = make_plan(op, v.coord, v.ext0, P.binding, P.rt);
            n = pl.tc_np ? 0 : pl.total_chunks();
        }
        if (chunk < n) {
            const Chunk ch = pl.chunk(chunk++);
            for (uint32_t off = lane * 128u; off < ch.bytes; off += 32u * 128u)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(ch.src + off));
            fbytes += ch.bytes;
        } else {
            ++slot;
            chunk = 0;
            n = -1;
        }
    }
}

// DMA-class queue: synthetic bodies only (copies are modelled by duration).
__device__ void dma_loop(const StaticParams& P) {
    // the whole warp walks the DMA queue: lane 0 waits / notifies, every lane copies
    const int lane = threadIdx.x & 31;
    const int q = P.num_queues;
    const int qb = __ldg(P.queue_off + q), qe = __ldg(P.queue_off + q + 1);
    for (int s = qb; s < qe; ++s) {
        const SlotInfo si = slot_info(P, s);
        const uint64_t t_begin = globaltimer();
        int ok = 1;
        if (lane == 0) {
            ok = wait_slot(P, s, q);
            if (ok && P.step_limit > 0 &&
                atomicAdd(&P.status->executed, 1ull) >= static_cast<unsigned long long>(P.step_limit)) {
                report(P.status, ET_ERR_STEP_LIMIT, q, s, -1, 0);
                ok = 0;
            }
        }
        if (!__shfl_sync(0xffffffffu, ok, 0)) return;
        const uint64_t t_wait = globaltimer();
        const bool masked = si.masked || (si.lazy && extent_masked(P, si.call, si.coord));
        const et_op& op = P.ops[si.call];
        if (!masked && op.kind == ET_OP_COPY) {
            body_copy(op, si.coord[0], lane);
            __syncwarp();  // every lane's stores precede lane 0's release notify
        } else if (!masked && lane == 0 && P.tick_ns > 0 && P.slot_duration) {
            const uint64_t until = t_wait + static_cast<uint64_t>(__ldg(P.slot_duration + s)) * P.tick_ns;
            while (globaltimer() < until) {
            }
        }
        if (lane != 0) continue;
        const uint64_t t_exec = globaltimer();
        notify_slot(P, s, q);
        if (P.step_limit <= 0 && !masked) atomicAdd(&P.status->executed, 1ull);
        if (masked) atomicAdd(&P.status->noops, 1ull);
        if (P.record) {
            et_trace_rec r;
            r.t_push = 0;
            r.t_begin = static_cast<int64_t>(t_begin);
            r.t_wait_end = static_cast<int64_t>(t_wait);
            r.t_prologue = 0;
            r.t_exec_end = static_cast<int64_t>(t_exec);
            r.t_notify_end = static_cast<int64_t>(globaltimer());
            r.worker = q;
            r.flags = masked ? 1 : 0;
            r.task = s;
            r.pad = 0;
            P.trace[s] = r;
        }
    }
}

// Tensor-core instantiations: TMEM (512 columns) held for the whole launch and
// the x-buffer / done mbarriers initialised.
__device__ __forceinline__ void tc_setup(uint8_t* smem) {
    if (threadIdx.x == 0) {
        uint64_t* b = tc_bars(smem);
        for (int i = 0; i < 2 * kTcXSlots; ++i) mbar_init(&b[i], 1);
        mbar_init(&b[2 * kTcXSlots], kTcIssuers);  // done: one commit per issuer
        fence_mbar_init();
    }
    if ((threadIdx.x >> 5) == 0) tmem_alloc(reinterpret_cast<uint32_t*>(smem + kSmemMisc + 32), kTmemCols);
    tc_fence_before();
}

__device__ __forceinline__ void tc_teardown(uint8_t* smem) {
    tc_fence_before();
    bar_sync(1, kConsumers);
    tc_fence_after();
    if ((threadIdx.x >> 5) == 0) tmem_dealloc(reinterpret_cast<volatile uint32_t*>(smem + kSmemMisc)[8], kTmemCols);
}

template <bool kMoE, bool kTC>
__global__ void __launch_bounds__(kThreads, 1) et_static_kernel(const __grid_constant__ StaticParams P) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int worker = blockIdx.x;
    if (sticky_status(P)) return;
    // zero this CTA's slice of the other-parity counters (used by the next step)
    for (int i = worker * blockDim.x + threadIdx.x; i < P.cnt_capacity; i += gridDim.x * blockDim.x)
        P.cnt_other[i] = 0u;
    if (threadIdx.x == 0) {
        uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSmemBar);
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&full[kStages + i], 1);
        }
        mbar_init(merge_bar(smem), 1);
        fence_mbar_init();
        volatile int* misc = reinterpret_cast<volatile int*>(smem + kSmemMisc);
        misc[0] = 0;
        misc[1] = 0;
        misc[2] = 0;
        misc[9] = -1;
        misc[10] = 0;
        misc[11] = 0;
        misc[12] = -1;
        misc[13] = 0;
        reinterpret_cast<volatile long long*>(misc)[7] = 0;
    }
    // slot table for this CTA's queue
    SlotTable T;
    T.ent = reinterpret_cast<const uint4*>(smem + kSmemTable);
    T.ext0 = reinterpret_cast<const int*>(smem + kSmemExt0);
    const int qb = __ldg(P.queue_off + worker), qe = __ldg(P.queue_off + worker + 1);
    T.valid = P.table_ok && (qe - qb) <= kMaxTableSlots && P.num_calls <= kMaxTableCalls;
    if (T.valid) {
        uint4* ent = reinterpret_cast<uint4*>(smem + kSmemTable);
        int* ext0 = reinterpret_cast<int*>(smem + kSmemExt0);
        for (int c = threadIdx.x; c < P.num_calls; c += blockDim.x) ext0[c] = __ldg(P.call_extents + c * 4);
        for (int i = threadIdx.x; i <= qe - qb; i += blockDim.x) {
            const int s = qb + i;
            uint4 e;
            if (i < qe - qb) {
                const SlotInfo si = slot_info(P, s);
                e.x = static_cast<uint32_t>(si.call) | (si.masked ? 0x80000000u : 0u) | (si.lazy ? 0x40000000u : 0u);
                e.y = static_cast<uint32_t>(si.coord[0] & 0xffff) |
                      (static_cast<uint32_t>(si.rank > 1 ? si.coord[1] & 0xffff : 0) << 16);
            } else {
                e.x = e.y = 0u;
            }
            e.z = static_cast<uint32_t>(__ldg(P.wait_off + s));
            e.w = static_cast<uint32_t>(__ldg(P.notify_off + s));
            ent[i] = e;
        }
    }
    if constexpr (kTC) tc_setup(smem);
    __syncthreads();
    if constexpr (kTC) tc_fence_after();
    const int warp = threadIdx.x >> 5;
    if (warp < kConsumerWarps) {
        consumer_loop<kMoE, kTC>(P, worker, smem, T);
        if constexpr (kTC) tc_teardown(smem);
    } else if (warp == kProducerWarp) {
        producer_loop(P, worker, smem, T);
    } else if (warp == kDmaWarp && worker == 0 && P.has_dma) {
        dma_loop(P);
    } else if (warp == kDmaWarp && P.prefetch && P.l2_ahead > 0 && (P.debug & 128) == 0) {
        l2_ahead_loop(P, worker, smem, T);
    }
}

// ===========================================================================
// Dynamic scheduler (Algorithm 2 of the paper; ref simulate.cpp:303-668).
//
// A device-resident ready queue per resource class: a slot array with an
// atomic tail (push) and head (pop); a slot holds task+1 once published with a
// release store, so a pop never reads an unpublished slot.  Workers pop, wait
// on armed Event Tensor waits, execute, and notify; a notify that completes an
// element pushes its consumers (consumer CSR built on the host for static
// maps; range-trigger consumers read from the device-resident indptr).  With
// early push, consumers are pushed when all producers have *started*
// (dispatch counters) and their waits are armed.  Data-dependent counters
// take their initial value from the counts tensor written on the device and
// become visible when the writer call finishes (reveal).  All per-step state
// is double-buffered; every launch resets the other parity for the next step.

__device__ __forceinline__ void fence_sc_gpu() { asm volatile("fence.sc.gpu;" ::: "memory"); }

__device__ __forceinline__ uint32_t dyn_init(const StaticParams& P, const DynParams& D, int el) {
    const int4 info = __ldg(D.el_info + el);
    if (info.z < 0) return static_cast<uint32_t>(info.w);
    return static_cast<uint32_t>(__ldcg(P.rt[D.dd_counts_rt[info.z]] + (el - D.dd_base[info.z])));
}

__device__ __forceinline__ bool dyn_visible(const DynParams& D, int el) {
    const int t = __ldg(D.el_dd + el);
    if (t < 0) return true;
    if (ld_relaxed(reinterpret_cast<const uint32_t*>(&D.ctl->revealed[t])) == 0u) return false;
    fence_acquire_gpu();  // the revealed counts / indptr are read next
    return true;
}

// Ready-queue slot word: (call << 21) | (task + 1) -- the popper starts loading the
// call's op record in the same round trip as the task's own records.  Call 511 =
// not encoded (more than 511 calls): the popper reads it from task_desc.
constexpr int kSlotTaskBits = 21;
constexpr uint32_t kSlotNoCall = 511u;
__device__ __forceinline__ uint32_t slot_word(int task, int call) {
    const uint32_t c = (call >= 0 && call < static_cast<int>(kSlotNoCall)) ? static_cast<uint32_t>(call) : kSlotNoCall;
    return (c << kSlotTaskBits) | static_cast<uint32_t>(task + 1);
}
// consumers[] entries: task in bits 0..20, its call in 21..29 (511: unknown), bit 30 =
// DMA class, bit 31 = this element is the consumer's only pending wait
__device__ __forceinline__ int cons_task(int e) { return e & ((1 << kSlotTaskBits) - 1); }
__device__ __forceinline__ int cons_call(int e) {
    const int c = (e >> kSlotTaskBits) & 511;
    return c == static_cast<int>(kSlotNoCall) ? -1 : c;
}

__device__ void dyn_push(const StaticParams& P, const DynParams& D, int task, int call = -1) {
    const int cls = __ldg(D.task_class + task);
    const unsigned int i = atomicAdd(&D.ctl->tail[cls], 1u);
    if (P.record) D.push_time[task] = globaltimer();
    st_release(reinterpret_cast<uint32_t*>(D.slots + static_cast<long long>(cls) * D.num_tasks + i), slot_word(task, call));
    atomicAdd(&P.status->pushes, 1ull);
}

__device__ void dyn_fire(const StaticParams& P, const DynParams& D, int el) {
    if (atomicExch(&D.fired[el], 1u) != 0u) return;
    for (int k = __ldg(D.consumer_off + el), e = __ldg(D.consumer_off + el + 1); k < e; ++k) {
        const int ce = __ldg(D.consumers + k), c = cons_task(ce);
        if (ce < 0 || atomicSub(&D.rem[c], 1) == 1) dyn_push(P, D, c, cons_call(ce));
    }
    const int t = __ldg(D.el_dd + el);
    if (t >= 0 && D.dd_range_call[t] >= 0) {
        const int call = D.dd_range_call[t];
        const int* ip = P.rt[__ldg(D.call_range_rt + call)];
        const int g = el - D.dd_base[t];
        const int first = __ldg(D.call_first_task + call);
        for (int f = __ldcg(ip + g), hi = __ldcg(ip + g + 1); f < hi; ++f)
            if (atomicSub(&D.rem[first + f], 1) == 1) dyn_push(P, D, first + f, call);
    }
}

__device__ void dyn_reveal(const StaticParams& P, const DynParams& D, int t) {
    st_release(reinterpret_cast<uint32_t*>(&D.ctl->revealed[t]), 1u);
    fence_sc_gpu();
    const int rc = D.dd_range_call[t];
    if (rc >= 0) {  // range-call tasks at or beyond indptr[last] never exist
        const int* ip = P.rt[__ldg(D.call_range_rt + rc)];
        const int live = __ldcg(ip + D.dd_count[t]);
        long long worst = 1;
        for (int d = 0, r = __ldg(P.call_rank + rc); d < r; ++d) worst *= __ldg(P.call_extents + rc * 4 + d);
        const int first = __ldg(D.call_first_task + rc);
        const int cls = __ldg(D.task_class + first);
        atomicSub(&D.ctl->total[cls], static_cast<int>(worst - live));
    }
    for (int el = D.dd_base[t], e = D.dd_base[t] + D.dd_count[t]; el < e; ++el) {
        const uint32_t have = D.early_push ? ld_acquire(D.disp + el) : ld_acquire(P.cnt + el);
        if (have >= dyn_init(P, D, el)) dyn_fire(P, D, el);
    }
}

// element produced by a routed notify of task (call, flat), or -1
__device__ __forceinline__ int dyn_routed_el(const StaticParams& P, const DynParams& D, int call, int flat) {
    const int r = __ldg(D.call_routed_rt + call);
    if (r < 0) return -1;
    return __ldg(D.call_routed_base + call) + __ldcg(P.rt[r] + flat);
}

// counts one finished notify (or dispatch under early push) of element el
__device__ void dyn_count(const StaticParams& P, const DynParams& D, unsigned int* ctr, int el, bool may_fire, int worker,
                          int task) {
    const uint32_t old = atom_add_release(ctr + el, 1u);
    const uint32_t need = dyn_init(P, D, el);
    if (ctr == P.cnt && old >= need) report(P.status, ET_ERR_UNDERFLOW, worker, task, el, -1);
    if (may_fire && old + 1 == need) {
        fence_sc_gpu();
        if (dyn_visible(D, el)) dyn_fire(P, D, el);
    }
}

// ---- warp-cooperative completion (the consumer CTAs' warp 0).  A notify that
// completes an element releases its consumers lane-strided over the warp and
// pushes the ready ones with one tail reservation per warp (a 148-way fan-out
// costs ~5 serial atomics instead of ~300).  Lane 0 owns the counter atomics.
__device__ __forceinline__ void dyn_push_warp(const StaticParams& P, const DynParams& D, int task, bool ready, int lane,
                                              int known_cls = -1, int call = -1) {
    const unsigned any = __ballot_sync(0xffffffffu, ready);
    if (!any) return;
    const int cls = !ready ? 0 : known_cls >= 0 ? known_cls : __ldg(D.task_class + task);
    for (int c = 0; c < 2; ++c) {
        const unsigned m = __ballot_sync(0xffffffffu, ready && cls == c);
        if (!m) continue;
        const int leader = __ffs(m) - 1;
        unsigned int base = 0;
        if (lane == leader) base = atomicAdd(&D.ctl->tail[c], static_cast<unsigned int>(__popc(m)));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (ready && cls == c) {
            const unsigned int i = base + __popc(m & ((1u << lane) - 1u));
            if (P.record) D.push_time[task] = globaltimer();
            st_release(reinterpret_cast<uint32_t*>(D.slots + static_cast<long long>(c) * D.num_tasks + i),
                       slot_word(task, call));
        }
    }
    if (lane == 0) atomicAdd(&P.status->pushes, static_cast<unsigned long long>(__popc(any)));
}

// info: the element's record when the caller has it; e_first: this lane's entry of
// its first 32 consumers, preloaded by the caller (or pass have_first = false).
__device__ __noinline__ void dyn_fire_warp(const StaticParams& P, const DynParams& D, int el, int lane,
                                           const int4* pinfo = nullptr, int e_first = 0, bool have_first = false) {
    const int4 info = pinfo ? *pinfo : __ldg(D.el_info + el);  // (consumers begin, end, dd tensor, initial count)
    if (info.z >= 0) {  // a data-dependent element can be fired by its count and by the reveal
        int first = 0;
        if (lane == 0) first = atomicExch(&D.fired[el], 1u) == 0u;
        if (!__shfl_sync(0xffffffffu, first, 0)) return;
    }
    const int cb = info.x, ce = info.y;
    for (int k0 = cb; k0 < ce; k0 += 32) {
        const int k = k0 + lane;
        const int e = k < ce ? ((k0 == cb && have_first) ? e_first : __ldg(D.consumers + k)) : 0;
        const int c = cons_task(e);
        // bit 31: this element is the consumer's only pending wait -> ready now; bit 30: DMA class
        const bool ready = k < ce && (e < 0 || atomicSub(&D.rem[c], 1) == 1);
        dyn_push_warp(P, D, c, ready, lane, (e >> 30) & 1, cons_call(e));
    }
    const int t = info.z;
    if (t >= 0 && D.dd_range_call[t] >= 0) {
        const int call = D.dd_range_call[t];
        const int* ip = P.rt[__ldg(D.call_range_rt + call)];
        const int g = el - D.dd_base[t];
        const int first_task = __ldg(D.call_first_task + call);
        const int lo = __ldcg(ip + g), hi = __ldcg(ip + g + 1);
        for (int f0 = lo; f0 < hi; f0 += 32) {
            const int f = f0 + lane;
            const bool ready = f < hi && atomicSub(&D.rem[first_task + f], 1) == 1;
            dyn_push_warp(P, D, first_task + f, ready, lane, -1, call);
        }
    }
}

__device__ void dyn_count_warp(const StaticParams& P, const DynParams& D, unsigned int* ctr, int el, bool may_fire,
                               int worker, int task, int lane);
__device__ void dyn_count_n_warp(const StaticParams& P, const DynParams& D, unsigned int* ctr, int el, uint32_t n,
                                 bool may_fire, int task, int lane);

__device__ void dyn_reveal_warp(const StaticParams& P, const DynParams& D, int t, int lane) {
    if (lane == 0) {
        st_release(reinterpret_cast<uint32_t*>(&D.ctl->revealed[t]), 1u);
        fence_sc_gpu();
        const int rc = D.dd_range_call[t];
        if (rc >= 0) {  // range-call tasks at or beyond indptr[last] never exist
            const int* ip = P.rt[__ldg(D.call_range_rt + rc)];
            const int live = __ldcg(ip + D.dd_count[t]);
            long long worst = 1;
            for (int d = 0, r = __ldg(P.call_rank + rc); d < r; ++d) worst *= __ldg(P.call_extents + rc * 4 + d);
            const int first = __ldg(D.call_first_task + rc);
            const int cls = __ldg(D.task_class + first);
            atomicSub(&D.ctl->total[cls], static_cast<int>(worst - live));
        }
    }
    __syncwarp();
    // Every element of the tensor, 4 per lane with all their loads in flight at once
    // (one pass of L2 round trips for up to 128 elements instead of one per 32).
    const int rcw = D.dd_range_call[t];
    const int* ipw = rcw >= 0 ? P.rt[__ldg(D.call_range_rt + rcw)] : nullptr;
    const int* cntw = P.rt[D.dd_counts_rt[t]];
    const unsigned int* havew = D.early_push ? D.disp : P.cnt;
    for (int e0 = D.dd_base[t], e1 = D.dd_base[t] + D.dd_count[t]; e0 < e1; e0 += 128) {
        int4 info[4];
        uint32_t need[4], have[4];
        int r0[4], r1[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int el = e0 + lane + 32 * u;
            const bool in = el < e1;
            info[u] = in ? __ldg(D.el_info + el) : make_int4(0, 0, -1, 0);
            need[u] = in ? static_cast<uint32_t>(__ldcg(cntw + (el - D.dd_base[t]))) : 0u;
            r0[u] = in && ipw ? __ldcg(ipw + (el - D.dd_base[t])) : 0;
            r1[u] = in && ipw ? __ldcg(ipw + (el - D.dd_base[t]) + 1) : 0;
            have[u] = in ? ld_relaxed(havew + el) : 0u;
        }
        fence_acquire_gpu();  // the counts above were written before the notifies they count
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int el = e0 + lane + 32 * u;
            // an element that releases nothing (no static consumers, empty range) never needs to fire
            const bool releases = info[u].y > info[u].x || r1[u] > r0[u];
            const bool f = el < e1 && releases && have[u] >= need[u];
            unsigned m = __ballot_sync(0xffffffffu, f);
            while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                dyn_fire_warp(P, D, e0 + b + 32 * u, lane);
            }
        }
    }
    // Range-call tasks at or beyond indptr[last] never exist (extent_from): the
    // static-map notifies the sample's worst-case counts expect from them are
    // credited here, once the live count is known (the reference instantiates the
    // actual grid instead, ref materialize.cpp:166-174).
    const int rcall = D.dd_range_call[t];
    if (rcall >= 0) {
        const int live = __ldcg(P.rt[__ldg(D.call_range_rt + rcall)] + D.dd_count[t]);
        long long worst = 1;
        for (int d = 0, r = __ldg(P.call_rank + rcall); d < r; ++d) worst *= __ldg(P.call_extents + rcall * 4 + d);
        const int first = __ldg(D.call_first_task + rcall);
        const int uel = D.dd_range_uniform_el[t];
        if (uel >= 0 && worst > live) {
            // every tail task notifies the same single element: credit them with one add each
            // counter (one atomic per task took ~1.4 ms per MoE layer at batch 32)
            const uint32_t n = static_cast<uint32_t>(worst - live);
            if (D.early_push) dyn_count_n_warp(P, D, D.disp, uel, n, true, first + static_cast<int>(live), lane);
            dyn_count_n_warp(P, D, P.cnt, uel, n, !D.early_push, first + static_cast<int>(live), lane);
        } else {
            for (long long f = live; f < worst; ++f) {
                const int task = first + static_cast<int>(f);
                const int4 rg = __ldg(D.task_rng + task);
                for (int n = rg.z; n < rg.w; ++n) {
                    const int el = __ldg(D.task_notifies + n);
                    if (D.early_push) dyn_count_warp(P, D, D.disp, el, true, -1, task, lane);
                    dyn_count_warp(P, D, P.cnt, el, !D.early_push, -1, task, lane);
                }
            }
        }
    }
}

__device__ void dyn_count_warp(const StaticParams& P, const DynParams& D, unsigned int* ctr, int el, bool may_fire,
                               int worker, int task, int lane) {
    int fire = 0;
    int4 info = make_int4(0, 0, 0, 0);
    if (lane == 0) {
        info = __ldg(D.el_info + el);  // in flight together with the atomic
        const uint32_t old = atom_add_release(ctr + el, 1u);
        const uint32_t need = info.z < 0 ? static_cast<uint32_t>(info.w) : dyn_init(P, D, el);
        if (ctr == P.cnt && old >= need) report(P.status, ET_ERR_UNDERFLOW, worker, task, el, -1);
        if (may_fire && old + 1 == need) {
            if (info.z < 0) {
                fire = 1;  // static element: only this notify can complete it
            } else {
                fence_sc_gpu();  // ordered against the reveal of the data-dependent tensor
                fire = dyn_visible(D, el);
            }
        }
    }
    if (__shfl_sync(0xffffffffu, fire, 0)) {
        info.x = __shfl_sync(0xffffffffu, info.x, 0);
        info.y = __shfl_sync(0xffffffffu, info.y, 0);
        info.z = __shfl_sync(0xffffffffu, info.z, 0);
        info.w = __shfl_sync(0xffffffffu, info.w, 0);
        dyn_fire_warp(P, D, el, lane, &info);
    }
}

// n notifies of element el at once (the reveal's credit for never-instantiated tail tasks)
__device__ void dyn_count_n_warp(const StaticParams& P, const DynParams& D, unsigned int* ctr, int el, uint32_t n,
                                 bool may_fire, int task, int lane) {
    int fire = 0;
    int4 info = make_int4(0, 0, 0, 0);
    if (lane == 0) {
        info = __ldg(D.el_info + el);
        const uint32_t old = atom_add_release(ctr + el, n);
        const uint32_t need = info.z < 0 ? static_cast<uint32_t>(info.w) : dyn_init(P, D, el);
        if (ctr == P.cnt && old + n > need) report(P.status, ET_ERR_UNDERFLOW, -1, task, el, -1);
        if (may_fire && old < need && old + n == need) {
            if (info.z < 0) {
                fire = 1;
            } else {
                fence_sc_gpu();
                fire = dyn_visible(D, el);
            }
        }
    }
    if (__shfl_sync(0xffffffffu, fire, 0)) {
        info.x = __shfl_sync(0xffffffffu, info.x, 0);
        info.y = __shfl_sync(0xffffffffu, info.y, 0);
        info.z = __shfl_sync(0xffffffffu, info.z, 0);
        info.w = __shfl_sync(0xffffffffu, info.w, 0);
        dyn_fire_warp(P, D, el, lane, &info);
    }
}

__device__ bool dyn_wait_el(const StaticParams& P, const DynParams& D, int el, int worker, int task) {
    const uint64_t t0 = globaltimer();
    uint32_t it = 0;
    while (!dyn_visible(D, el)) {  // data-dependent element: its count exists once revealed
        if ((++it & 255u) == 0) {
            if (aborted(P.status)) return false;
            if (globaltimer() - t0 > static_cast<uint64_t>(P.watchdog_ns)) {
                report(P.status, ET_ERR_DEADLOCK, worker, task, el, -1);
                return false;
            }
        }
    }
    const uint32_t need = dyn_init(P, D, el);
    while (ld_relaxed(P.cnt + el) < need) {
        if ((++it & 255u) == 0) {
            if (aborted(P.status)) return false;
            if (globaltimer() - t0 > static_cast<uint64_t>(P.watchdog_ns)) {
                report(P.status, ET_ERR_DEADLOCK, worker, task, el,
                       static_cast<int>(dyn_init(P, D, el) - ld_relaxed(P.cnt + el)));
                return false;
            }
        }
    }
    fence_acquire_gpu();
    return true;
}

// Pops one task of class cls: -1 when every task of the class has been taken.
__device__ int dyn_pop(const StaticParams& P, const DynParams& D, int cls, int worker) {
    const unsigned int i = atomicAdd(&D.ctl->head[cls], 1u);
    const uint32_t* slot = reinterpret_cast<const uint32_t*>(D.slots + static_cast<long long>(cls) * D.num_tasks + i);
    const uint64_t t0 = globaltimer();
    uint32_t it = 0;
    for (;;) {
        if (static_cast<int>(i) < D.num_tasks) {
            const uint32_t v = ld_relaxed(slot);
            if (v) {
                fence_acquire_gpu();
                atomicAdd(&P.status->pops, 1ull);
                return static_cast<int>(v);  // slot_word: the caller decodes task and call
            }
        }
        if (static_cast<int>(i) >= *reinterpret_cast<volatile int*>(&D.ctl->total[cls])) return -1;
        if ((++it & 255u) == 0) {
            if (aborted(P.status)) return -1;
            if (globaltimer() - t0 > static_cast<uint64_t>(P.watchdog_ns)) {
                report(P.status, ET_ERR_DEADLOCK, worker, -1, -4, static_cast<int>(i));
                return -1;
            }
        }
    }
}

// A task's slot view from its packed records; masking compares the coordinates
// with the call's grid extents at this launch's binding (shared-memory table
// filled at kernel start when the graph has <= kMaxCallExt calls of rank <= 2).
__device__ SlotView dyn_view(const StaticParams& P, const DynParams& D, int task, const int4* cext = nullptr) {
    SlotView v;
    const int4 d = __ldg(D.task_desc + task);
    const int4 r = __ldg(D.task_rng + task);
    v.call = d.x;
    v.coord[0] = d.y;
    v.coord[1] = d.z;
    v.coord[2] = v.coord[3] = 0;
    v.ext0 = d.w;
    if (cext) {
        const int4 e = cext[v.call];
        v.masked = v.coord[0] >= e.x || v.coord[1] >= e.y;
    } else {
        const int rank = __ldg(P.call_rank + v.call);
        v.masked = false;
        for (int k = 0; k < rank && k < 2; ++k)
            if (v.coord[k] >= eval_code(P, v.call, k)) v.masked = true;
    }
    v.lazy = false;
    v.wb = r.x;
    v.we = r.y;
    v.nb = r.z;
    v.ne = r.w;
    return v;
}

// WAITs of a popped task (armed slots only, ref simulate.cpp:497-515), then the
// early-push dispatch (ref simulate.cpp:600-618).
__device__ bool dyn_prepare(const StaticParams& P, const DynParams& D, const SlotView& v, int task, int worker,
                            bool dispatch = true) {
    for (int w = v.wb; w < v.we; ++w)
        if (__ldg(D.task_wait_armed + w) && !dyn_wait_el(P, D, __ldg(D.task_waits + w), worker, task)) return false;
    const int rr = __ldg(D.call_range_rt + v.call);
    if (rr >= 0 && __ldg(D.call_range_armed + v.call)) {
        const int* ip = P.rt[rr];
        const int flat = __ldg(D.task_flat + task);
        int g = 0;
        for (bool found = false; !found; g += 8) {  // 8 loads in flight per probe round
            int v8[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v8[u] = __ldcg(ip + g + u + 1);
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (!found && v8[u] > flat) {
                    found = true;
                    g += u - 8;
                }
        }
        if (!dyn_wait_el(P, D, __ldg(D.call_range_base + v.call) + g, worker, task)) return false;
    }
    if (D.early_push && dispatch) {
        for (int n = v.nb; n < v.ne; ++n) dyn_count(P, D, D.disp, __ldg(D.task_notifies + n), true, worker, task);
        const int rel = v.masked ? -1 : dyn_routed_el(P, D, v.call, __ldg(D.task_flat + task));  // masked: no routing
        if (rel >= 0) dyn_count(P, D, D.disp, rel, true, worker, task);
    }
    return true;
}

// Completion: reveal data-dependent tensors written by this call (before the
// notifies, so consumers released by them see visible counters), then NOTIFY.
__device__ void dyn_finish(const StaticParams& P, const DynParams& D, const SlotView& v, int task, int worker) {
    for (int t = 0; t < D.num_dd; ++t)
        if (D.dd_writer_call[t] == v.call && atomicSub(&D.ctl->writer_rem[t], 1) == 1) dyn_reveal(P, D, t);
    const bool fire = !D.early_push;
    for (int n = v.nb; n < v.ne; ++n) dyn_count(P, D, P.cnt, __ldg(D.task_notifies + n), fire, worker, task);
    const int rel = v.masked ? -1 : dyn_routed_el(P, D, v.call, __ldg(D.task_flat + task));  // masked: no routing
    if (rel >= 0) dyn_count(P, D, P.cnt, rel, fire, worker, task);
}

// Warp-0 versions used by the consumer CTAs (the DMA warp keeps the scalar ones).
__device__ void dyn_dispatch_warp(const StaticParams& P, const DynParams& D, const SlotView& v, int task, int worker,
                                  int lane) {
    for (int n = v.nb; n < v.ne; ++n) dyn_count_warp(P, D, D.disp, __ldg(D.task_notifies + n), true, worker, task, lane);
    const int rel = v.masked ? -1 : dyn_routed_el(P, D, v.call, __ldg(D.task_flat + task));  // masked: no routing
    if (rel >= 0) dyn_count_warp(P, D, D.disp, rel, true, worker, task, lane);
}

__device__ void dyn_finish_warp(const StaticParams& P, const DynParams& D, const SlotView& v, int task, int worker,
                                int lane, int4 note = make_int4(-1, 0, 0, 0), const int4* cext = nullptr) {
    if ((P.debug & 0x100000) && lane == 0) D.push_time[task] = globaltimer();  // probe: finish entry
    // data-dependent tensors this call writes: from the shared-memory call table (an
    // indexed walk over the kernel parameters costs ~4 us of constant-cache misses)
    const int t_lo = cext ? cext[v.call].z : 0, t_hi = cext ? (cext[v.call].z < 0 ? 0 : cext[v.call].z + cext[v.call].w)
                                                       : D.num_dd;
    for (int t = t_lo < 0 ? 0 : t_lo; t < t_hi; ++t) {
        if (D.dd_writer_call[t] != v.call) continue;
        int last = 0;
        if (lane == 0) last = atomicSub(&D.ctl->writer_rem[t], 1) == 1;
        if (__shfl_sync(0xffffffffu, last, 0)) dyn_reveal_warp(P, D, t, lane);
    }
    if ((P.debug & 0x200000) && lane == 0) D.push_time[task] = globaltimer();  // probe: after the writer loop
    const bool fire = !D.early_push;
    int n0 = v.nb;
    if (note.x >= 0 && v.ne > v.nb) {
        // the first notify's element record came with the task (task_note): its consumer
        // entries load together with the count's atomic -- one round trip, then the push
        const int k = note.y + lane;
        const int e = k < note.z ? __ldg(D.consumers + k) : 0;
        int go = 0;
        if (lane == 0) {
            const uint32_t old = atom_add_release(P.cnt + note.x, 1u);
            if (old >= static_cast<uint32_t>(note.w)) report(P.status, ET_ERR_UNDERFLOW, worker, task, note.x, -1);
            go = fire && old + 1 == static_cast<uint32_t>(note.w);
        }
        if ((P.debug & 0x40000) && lane == 0) D.push_time[task] = globaltimer();  // probe: count returned
        if (__shfl_sync(0xffffffffu, go, 0)) {
            const int4 info = make_int4(note.y, note.z, -1, note.w);
            dyn_fire_warp(P, D, note.x, lane, &info, e, true);
        }
        if ((P.debug & 0x80000) && lane == 0) D.push_time[task] = globaltimer();  // probe: fired
        n0 = v.nb + 1;
    }
    for (int n = n0; n < v.ne; ++n) dyn_count_warp(P, D, P.cnt, __ldg(D.task_notifies + n), fire, worker, task, lane);
    const int rel = v.masked ? -1 : dyn_routed_el(P, D, v.call, __ldg(D.task_flat + task));  // masked: no routing
    if (rel >= 0) dyn_count_warp(P, D, P.cnt, rel, fire, worker, task, lane);
}

__device__ void dyn_record(const StaticParams& P, const DynParams& D, int task, int worker, bool masked, uint64_t tb,
                           uint64_t tw, uint64_t tp, uint64_t te) {
    if (!P.record) return;
    et_trace_rec r;
    r.t_push = static_cast<int64_t>(D.push_time[task]);
    r.t_begin = static_cast<int64_t>(tb);
    r.t_wait_end = static_cast<int64_t>(tw);
    r.t_prologue = static_cast<int64_t>(tp);
    r.t_exec_end = static_cast<int64_t>(te);
    r.t_notify_end = static_cast<int64_t>(globaltimer());
    r.worker = worker;
    r.flags = masked ? 1 : 0;
    r.task = task;
    r.pad = P.step_id;
    P.trace[task] = r;
}

template <bool kMoE, bool kTC>
__device__ void dyn_consumer_loop(const StaticParams& P, const DynParams& D, int worker, uint8_t* smem) {
    const int ctid = threadIdx.x;
    TcState ts{kTC ? reinterpret_cast<volatile uint32_t*>(smem + kSmemMisc)[8] : 0u, 0u, 0u};
    const int4* cext = P.num_calls <= kMaxCallExt ? reinterpret_cast<const int4*>(smem + kSmemCallExt) : nullptr;
    uint16_t* xs = reinterpret_cast<uint16_t*>(smem + kSmemX);
    float* acc = reinterpret_cast<float*>(smem + kSmemAcc);
    volatile int* misc = reinterpret_cast<volatile int*>(smem + kSmemMisc);
    float* red = reinterpret_cast<float*>(smem + kSmemMisc + 64);
    Ring ring{smem + kSmemRing, reinterpret_cast<uint64_t*>(smem + kSmemBar),
              reinterpret_cast<uint64_t*>(smem + kSmemBar) + kStages, 0ull, P.status, P.watchdog_ns, worker};
    unsigned long long executed = 0, noops = 0;
    for (;;) {
        uint64_t tb = 0, tw = 0, tp = 0, te = 0;
        if (ctid == 0) {
            const int word = dyn_pop(P, D, 0, worker);
            tb = globaltimer();
            const int task = word < 0 ? -1 : (word & ((1 << kSlotTaskBits) - 1)) - 1;
            const uint32_t wc = word < 0 ? kSlotNoCall : static_cast<uint32_t>(word) >> kSlotTaskBits;
            misc[3] = task;
            misc[7] = wc == kSlotNoCall ? -1 : static_cast<int>(wc);
            misc[4] = task;  // hand the task to the producer warp (streams during the waits)
            __threadfence_block();
            misc[5] = misc[5] + 1;
        }
        bar_sync(1, kConsumers);
        const int task = misc[3];
        if (task < 0) break;
        const int wcall = misc[7];  // the call, when the slot word carried it
        // the op record's copy starts with the task's own records (same round trip)
        const et_op* opp = wcall >= 0 ? P.ops + wcall : nullptr;
        int opw = 0;
        if (opp && ctid >= 32 && ctid < 32 + static_cast<int>(sizeof(et_op) / 4))
            opw = reinterpret_cast<const int*>(opp)[ctid - 32];
        int4 note = make_int4(-1, 0, 0, 0);
        if (ctid < 32) note = __ldg(D.task_note + task);  // used by warp 0 at the task's end
        SlotView v = dyn_view(P, D, task, cext);
        if (opp) {
            if (ctid >= 32 && ctid < 32 + static_cast<int>(sizeof(et_op) / 4))
                reinterpret_cast<int*>(smem + kSmemOp)[ctid - 32] = opw;
        }
        const et_op& opg = P.ops[v.call];  // shared-memory copy, as in the static loop
        if (!opp && ctid >= 32 && ctid < 32 + static_cast<int>(sizeof(et_op) / 4))
            reinterpret_cast<int*>(smem + kSmemOp)[ctid - 32] = reinterpret_cast<const int*>(&opg)[ctid - 32];
        const et_op& op = *reinterpret_cast<const et_op*>(smem + kSmemOp);
        if (ctid < 32) {
            int ok = 1;
            if (ctid == 0) {
                // Without early push a task is pushed only once every wait element (armed or
                // not, range trigger included) has fired, so its armed waits hold already: no
                // device round trips to re-check them (early push: dispatched tasks wait here).
                ok = D.early_push ? dyn_prepare(P, D, v, task, worker, false) : true;
                if (ok && P.step_limit > 0 &&
                    atomicAdd(&P.status->executed, 1ull) >= static_cast<unsigned long long>(P.step_limit)) {
                    report(P.status, ET_ERR_STEP_LIMIT, worker, task, -1, 0);
                    ok = 0;
                }
            }
            ok = __shfl_sync(0xffffffffu, ok, 0);
            if (ok && D.early_push) dyn_dispatch_warp(P, D, v, task, worker, ctid);
            if (ctid == 0) {
                misc[0] = ok ? 0 : 1;
                misc[6] = misc[5];  // waits passed: the producer may stream this task's activations
                tw = globaltimer();
            }
        }
        bar_sync(1, kConsumers);
        if (misc[0]) break;
        if (v.masked) {
            ++noops;
        } else {
            ++executed;
            switch (op.kind) {
                case ET_OP_NONE:
                    if (ctid == 0 && P.tick_ns > 0 && D.task_duration) {
                        const uint64_t until = tw + static_cast<uint64_t>(__ldg(D.task_duration + task)) *
                                                        static_cast<uint64_t>(P.tick_ns);
                        while (globaltimer() < until) {
                        }
                    }
                    break;
                case ET_OP_SPLITK_PARTIAL:
                case ET_OP_SPLITK_FINAL: body_splitk(P, op, v.coord, ctid); break;
                case ET_OP_GEMV:
                    if (!gemv_fits(op, P)) {
                        if (ctid == 0) report(P.status, ET_ERR_INVALID, worker, task, -1, batch_of(op, P));
                        break;
                    }
                    tp = body_gemv(P, op, v, xs, acc, red, ring, ctid);
                    break;
                case ET_OP_ATTN_SPLIT:
                    body_attn_split<kMoE || kTC, kTC>(P, op, v, reinterpret_cast<float*>(xs), ring, ctid);
                    break;
                case ET_OP_ATTN_MERGE: body_attn_merge<kMoE || kTC>(P, op, v, reinterpret_cast<float*>(xs), ctid); break;
                case ET_OP_GEMV_TC:
                    if constexpr (kTC) tp = body_gemv_tc(P, op, v, smem, ring, ts, ctid);
                    break;
                case ET_OP_NORM:
                    if constexpr (kTC) body_norm(P, op, v, red, ctid);
                    break;
                case ET_OP_EMBED: body_embed(P, op, ctid); break;
                case ET_OP_ARGMAX: body_argmax(P, op, ctid); break;
                case ET_OP_REDUCE: body_reduce(P, op, v.coord, ctid); break;
                case ET_OP_COPY:  // copies are DMA-class tasks (dma_loop)
                    if (ctid == 0) report(P.status, ET_ERR_INVALID, worker, -1, -7, op.kind);
                    break;
                case ET_OP_MOE_ROUTE:
                    if constexpr (kMoE) body_moe_route<kTC>(P, op, v, xs, acc, red, ring, ctid, &tp);
                    break;
                case ET_OP_MOE_EXPERT:
                    if constexpr (kMoE) tp = body_moe_expert(P, op, v, xs, acc, ring, ctid);
                    break;
                default: break;
            }
        }
        bar_sync(1, kConsumers);
        if (ctid < 32) {
            if (ctid == 0) te = globaltimer();
            dyn_finish_warp(P, D, v, task, worker, ctid, note, cext);
            if (ctid == 0) dyn_record(P, D, task, worker, v.masked, tb, tw, tp, te);
        }
    }
    if (ctid == 0) {
        misc[4] = -1;
        __threadfence_block();
        misc[5] = misc[5] + 1;
        if (P.step_limit <= 0) atomicAdd(&P.status->executed, executed);
        atomicAdd(&P.status->noops, noops);
    }
}

__device__ void dyn_producer_loop(const StaticParams& P, const DynParams& D, int worker, uint8_t* smem) {
    if ((threadIdx.x & 31) != 0) return;
    const int4* cext = P.num_calls <= kMaxCallExt ? reinterpret_cast<const int4*>(smem + kSmemCallExt) : nullptr;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSmemBar);
    uint64_t* empty = full + kStages;
    volatile int* misc = reinterpret_cast<volatile int*>(smem + kSmemMisc);
    const uint64_t pol = policy_evict_first();
    unsigned long long cseq = 0;
    unsigned int xq = 0;
    int gen = 0;
    for (;;) {
        for (uint32_t it = 0; misc[5] == gen;)
            if ((++it & 1023u) == 0 && aborted(P.status)) return;
        gen = misc[5];
        const int task = misc[4];
        if (task < 0) return;
        const SlotView v = dyn_view(P, D, task, cext);
        if (v.masked) continue;
        const et_op& op = P.ops[v.call];
        if (!op_streams(op.kind)) continue;
        const StreamPlan pl = make_plan(op, v.coord, v.ext0, P.binding, P.rt);
        if (pl.tc_np) {  // tensor-core GEMV: activation pieces once the task's (armed) waits pass
            if (!tc_produce(P, smem, pl, misc, 1, gen, cseq, xq, worker, pol)) return;
            continue;
        }
        const int n = pl.total_chunks();
        for (int c = 0; c < n; ++c, ++cseq) {
            const int stage = static_cast<int>(cseq % kStages);
            const uint32_t phase = static_cast<uint32_t>((cseq / kStages) & 1ull);
            uint32_t spins = 0;
            while (!mbar_try_wait(&empty[stage], phase ^ 1u)) {
                if ((++spins & 1023u) == 0 && aborted(P.status)) return;
            }
            const Chunk ch = pl.chunk(c);
            mbar_arrive_expect_tx(&full[stage], ch.bytes);
            bulk_g2s(smem + kSmemRing + stage * kStageBytes, ch.src, ch.bytes, &full[stage], pol);
        }
    }
}

// DMA-class tasks: popped from their own queue by worker 0's DMA warp.
__device__ void dyn_dma_loop(const StaticParams& P, const DynParams& D, const int4* cext) {
    if ((threadIdx.x & 31) != 0) return;
    const int worker = P.num_queues;
    for (;;) {
        const int word = dyn_pop(P, D, 1, worker);
        if (word < 0) return;
        const int task = (word & ((1 << kSlotTaskBits) - 1)) - 1;
        const uint64_t tb = globaltimer();
        const SlotView v = dyn_view(P, D, task, cext);
        if (!dyn_prepare(P, D, v, task, worker)) return;
        const uint64_t tw = globaltimer();
        if (!v.masked && P.tick_ns > 0 && D.task_duration) {
            const uint64_t until = tw + static_cast<uint64_t>(__ldg(D.task_duration + task)) * P.tick_ns;
            while (globaltimer() < until) {
            }
        }
        const uint64_t te = globaltimer();
        dyn_finish(P, D, v, task, worker);
        atomicAdd(v.masked ? &P.status->noops : &P.status->executed, 1ull);
        dyn_record(P, D, task, worker, v.masked, tb, tw, 0, te);
    }
}

// (Re)initialises one parity of the dynamic state; block-strided over `nblk` blocks.
__device__ void dyn_reset_state(const StaticParams& P, const DynParams& D, DynCtl* ctl, int* rem, int* slots,
                                unsigned int* fired, unsigned int* disp, uint32_t* cnt, int blk, int nblk) {
    const int tid = blk * blockDim.x + threadIdx.x, stride = nblk * blockDim.x;
    for (int i = tid; i < D.num_tasks; i += stride) {
        rem[i] = __ldg(D.task_rem_init + i);
        // the ready seeds occupy the first slots of each class queue (id order)
        if (i < D.num_ready[0]) {
            const int t = __ldg(D.ready + i);
            slots[i] = static_cast<int>(slot_word(t, __ldg(D.task_call + t)));
        } else {
            slots[i] = 0;
        }
        if (i < D.num_ready[1]) {
            const int t = __ldg(D.ready + D.num_ready[0] + i);
            slots[D.num_tasks + i] = static_cast<int>(slot_word(t, __ldg(D.task_call + t)));
        } else {
            slots[D.num_tasks + i] = 0;
        }
    }
    for (int i = tid; i < P.cnt_capacity; i += stride) {
        fired[i] = 0u;
        disp[i] = 0u;
        cnt[i] = 0u;
    }
    if (blk == 0 && threadIdx.x == 0) {
        for (int c = 0; c < 2; ++c) {
            ctl->head[c] = 0u;
            ctl->tail[c] = static_cast<unsigned int>(D.num_ready[c]);
            ctl->total[c] = D.class_total[c];
        }
        for (int t = 0; t < kMaxDd; ++t) {
            ctl->writer_rem[t] = t < D.num_dd ? D.writer_tasks[t] : 0;
            ctl->revealed[t] = 0;
        }
    }
}

template <bool kMoE, bool kTC>
__global__ void __launch_bounds__(kThreads, 1)
    et_dynamic_kernel(const __grid_constant__ StaticParams P, const __grid_constant__ DynParams D) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int worker = blockIdx.x;
    if (sticky_status(P)) return;
    // the other parity is rebuilt for the next launch (same sample)
    dyn_reset_state(P, D, D.ctl_other, D.rem_other, D.slots_other, D.fired_other, D.disp_other, P.cnt_other, worker,
                    gridDim.x);
    if (threadIdx.x == 0) {
        uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSmemBar);
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&full[kStages + i], 1);
        }
        mbar_init(merge_bar(smem), 1);
        fence_mbar_init();
        volatile int* misc = reinterpret_cast<volatile int*>(smem + kSmemMisc);
        misc[0] = misc[1] = misc[2] = 0;
        misc[3] = misc[4] = misc[5] = 0;
        misc[6] = -1;
        misc[13] = 0;
        if (worker == 0) atomicAdd(&P.status->pushes, static_cast<unsigned long long>(D.num_ready[0] + D.num_ready[1]));
    }
    if (P.num_calls <= kMaxCallExt) {  // grid extents of every call at this binding (masking)
        // (.z: first data-dependent tensor the call writes, -1 = none; .w: how many, consecutive)
        int4* cext = reinterpret_cast<int4*>(smem + kSmemCallExt);
        for (int c = threadIdx.x; c < P.num_calls; c += blockDim.x) {
            const int rank = __ldg(P.call_rank + c);
            const int dd = __ldg(D.call_dd + c);
            cext[c] = make_int4(rank > 0 ? static_cast<int>(eval_code(P, c, 0)) : 1,
                                rank > 1 ? static_cast<int>(eval_code(P, c, 1)) : 1, dd < 0 ? -1 : (dd & 0xffff),
                                dd < 0 ? 0 : (dd >> 16));
        }
    }
    if constexpr (kTC) tc_setup(smem);
    __syncthreads();
    if constexpr (kTC) tc_fence_after();
    const int warp = threadIdx.x >> 5;
    if (warp < kConsumerWarps) {
        dyn_consumer_loop<kMoE, kTC>(P, D, worker, smem);
        if constexpr (kTC) tc_teardown(smem);
    } else if (warp == kProducerWarp) {
        dyn_producer_loop(P, D, worker, smem);
    } else if (warp == kDmaWarp && worker == 0 && P.has_dma) {
        dyn_dma_loop(P, D, P.num_calls <= kMaxCallExt ? reinterpret_cast<const int4*>(smem + kSmemCallExt) : nullptr);
    }
}

__global__ void et_dynamic_reset_kernel(const __grid_constant__ StaticParams P, const __grid_constant__ DynParams D) {
    dyn_reset_state(P, D, D.ctl, D.rem, D.slots, D.fired, D.disp, P.cnt, blockIdx.x, gridDim.x);
}

}  // namespace etk

int et_static_smem_bytes() { return etk::kSmemTotal; }

namespace {
template <typename K>
int launch_persistent(K kernel, bool& configured, int num_workers, void* stream, void** args) {
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, etk::kSmemTotal);
        if (e != cudaSuccess) return static_cast<int>(e);
        configured = true;
    }
    // Cooperative launch: every worker must be co-resident for the spin-waits
    // on Event Tensors to make progress (SURVEY hard part (ii)).
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(num_workers);
    cfg.blockDim = dim3(etk::kThreads);
    cfg.dynamicSmemBytes = etk::kSmemTotal;
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return static_cast<int>(cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(kernel), args));
}
}  // namespace

// variant bit 0: MoE bodies; bit 1: tensor-core GEMV (TMEM) bodies.  Batches above
// 8 need the tensor-core variant (the mma.sync GEMV carries the batch in n8).
int et_launch_static(const etk::StaticParams& p, int num_workers, int max_batch, int variant, void* stream) {
    if (max_batch > ((variant & 2) ? etk::kMaxBatchTc : etk::kMaxBatch)) return static_cast<int>(cudaErrorInvalidValue);
    static bool conf[4] = {false, false, false, false};
    void* args[] = {const_cast<etk::StaticParams*>(&p)};
    switch (variant & 3) {
        case 1: return launch_persistent(etk::et_static_kernel<true, false>, conf[1], num_workers, stream, args);
        case 2: return launch_persistent(etk::et_static_kernel<false, true>, conf[2], num_workers, stream, args);
        case 3: return launch_persistent(etk::et_static_kernel<true, true>, conf[3], num_workers, stream, args);
        default: return launch_persistent(etk::et_static_kernel<false, false>, conf[0], num_workers, stream, args);
    }
}

int et_launch_dynamic(const etk::StaticParams& p, const etk::DynParams& d, int num_workers, int variant, void* stream) {
    static bool conf[4] = {false, false, false, false};
    void* args[] = {const_cast<etk::StaticParams*>(&p), const_cast<etk::DynParams*>(&d)};
    switch (variant & 3) {
        case 1: return launch_persistent(etk::et_dynamic_kernel<true, false>, conf[1], num_workers, stream, args);
        case 2: return launch_persistent(etk::et_dynamic_kernel<false, true>, conf[2], num_workers, stream, args);
        case 3: return launch_persistent(etk::et_dynamic_kernel<true, true>, conf[3], num_workers, stream, args);
        default: return launch_persistent(etk::et_dynamic_kernel<false, false>, conf[0], num_workers, stream, args);
    }
}

int et_dynamic_reset(const etk::StaticParams& p, const etk::DynParams& d, void* stream) {
    etk::et_dynamic_reset_kernel<<<64, 256, 0, static_cast<cudaStream_t>(stream)>>>(p, d);
    return static_cast<int>(cudaGetLastError());
}
