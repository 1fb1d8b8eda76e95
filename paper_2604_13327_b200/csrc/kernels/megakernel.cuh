// Device-side program layout shared by the runtime (host) and the persistent
// megakernel.  See include/et_runtime.h for the C ABI these are built from.
#pragma once

#include <stdint.h>

#include "et_runtime.h"

namespace etk {

constexpr int kConsumerWarps = 8;
constexpr int kConsumers = kConsumerWarps * 32;   // compute threads
constexpr int kProducerWarp = kConsumerWarps;     // TMA issuer
constexpr int kDmaWarp = kConsumerWarps + 1;      // DMA-queue executor (worker 0 only)
constexpr int kThreads = (kConsumerWarps + 2) * 32;
// Chunk c lives in stage c % kStages and is consumed by warp c % kConsumerWarps.
// With kStages == kConsumerWarps every stage has exactly one consumer warp that
// takes its chunks in order, so an mbarrier parity can never alias a phase two
// steps ahead even though TMA copies may complete out of order.  Chunks that
// every warp must read (attention K/V blocks) are released by their owner after
// a consumer barrier.
constexpr int kStages = kConsumerWarps;
constexpr int kStageBytes = 20480;
constexpr int kXBytes = 28 * 1024;
constexpr int kAccFloats = 2048;
constexpr int kMaxSymbols = 8;
constexpr int kMaxRuntime = 16;
constexpr int kMaxRank = 4;
constexpr int kMaxBatch = 8;   // GEMV batch rows carried in the mma M dimension

constexpr int kMaxTableSlots = 512;   // per-CTA slot table in shared memory
constexpr int kMaxTableCalls = 1024;  // per-call sample extent of dim 0

constexpr int kSmemRing = 0;
constexpr int kSmemX = kSmemRing + kStages * kStageBytes;
constexpr int kSmemAcc = kSmemX + kXBytes;
constexpr int kSmemTable = kSmemAcc + kAccFloats * 4;
constexpr int kSmemExt0 = kSmemTable + (kMaxTableSlots + 1) * 16;
constexpr int kSmemBar = kSmemExt0 + kMaxTableCalls * 4;
constexpr int kSmemMisc = kSmemBar + 2 * kStages * 8;
constexpr int kSmemTotal = kSmemMisc + 512;

// Device status word block (one per runtime).
struct DevStatus {
    int code;       // et_status; 0 while running
    int worker;
    int slot;
    int counter;
    int value;
    int pad;
    unsigned long long executed;
    unsigned long long noops;
    unsigned long long pushes;
    unsigned long long pops;
};

struct StaticParams {
    // graph
    int num_symbols;
    int num_calls;
    const int* call_rank;
    const int* call_extent_from;
    const int* grid_code_off;
    const int* code_op;
    const long long* code_arg;
    // sample
    const int* call_extents;
    int num_queues;
    int has_dma;
    const int* queue_off;
    int num_slots;
    const int* slot_call;
    const int* slot_flat;
    const int* slot_duration;
    const int* wait_off;
    const int* waits;
    const int* notify_off;
    const int* notifies;
    int num_counters;
    const int* initial_counts;
    // step state
    uint32_t* cnt;        // this step's notify counts
    uint32_t* cnt_other;  // the other parity buffer: zeroed for the next step
    int cnt_capacity;
    int* const* rt;       // runtime tensors (device pointers)
    long long rt_len[kMaxRuntime];
    int num_rt;
    const et_op* ops;
    et_trace_rec* trace;
    int record;
    DevStatus* status;        // this step's status block
    DevStatus* status_other;  // zeroed for the next step
    long long binding[kMaxSymbols];
    long long watchdog_ns;
    long long tick_ns;
    long long step_limit;  // 0 = unlimited
    int prefetch;
    int table_ok;  // every coordinate fits 16 bits (slot tables usable)
    long long l2_ahead;  // bytes the producer prefetches into L2 beyond the ring
};

}  // namespace etk

// Host-side launcher (megakernel.cu).
int et_launch_static(const etk::StaticParams& p, int num_workers, int max_batch, void* stream);
int et_static_smem_bytes();
