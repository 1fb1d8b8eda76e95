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
constexpr int kStages = 10;
constexpr int kStageBytes = 16384;
constexpr int kXBytes = 48 * 1024;
constexpr int kAccFloats = 4096;
constexpr int kMaxSymbols = 8;
constexpr int kMaxRuntime = 16;
constexpr int kMaxRank = 4;

constexpr int kSmemRing = 0;
constexpr int kSmemX = kSmemRing + kStages * kStageBytes;
constexpr int kSmemAcc = kSmemX + kXBytes;
constexpr int kSmemBar = kSmemAcc + kAccFloats * 4;
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
};

}  // namespace etk

// Host-side launcher (megakernel.cu).
int et_launch_static(const etk::StaticParams& p, int num_workers, void* stream);
int et_static_smem_bytes();
