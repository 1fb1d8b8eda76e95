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
constexpr int kXBytes = 32 * 1024;
constexpr int kAccFloats = 2048;
constexpr int kMaxSymbols = 8;
constexpr int kMaxRuntime = 512;  // runtime tensors per graph (6 per MoE layer)
constexpr int kMaxRank = 4;
// Attention partial row per (q head, split): m, l, 2 pad floats, then o[dh] -- 16-byte
// aligned rows, so a group's partials move with bulk copies.
constexpr int kPartHead = 4;
constexpr int kMaxBatch = 8;   // GEMV batch rows carried in the mma M dimension
constexpr int kMaxBatchTc = 128;  // tensor-core GEMV: batch = MMA N (Npad * kp * 2 <= 16 KB)

constexpr int kMaxTableSlots = 512;   // per-CTA slot table in shared memory
constexpr int kMaxTableCalls = 1024;  // per-call sample extent of dim 0

constexpr int kSmemRing = 0;
constexpr int kSmemX = kSmemRing + kStages * kStageBytes;
constexpr int kSmemAcc = kSmemX + kXBytes;
constexpr int kSmemTable = kSmemAcc + kAccFloats * 4;
constexpr int kSmemExt0 = kSmemTable + (kMaxTableSlots + 1) * 16;
constexpr int kSmemBar = kSmemExt0 + kMaxTableCalls * 4;
constexpr int kSmemMisc = kSmemBar + 2 * kStages * 8;
constexpr int kSmemOp = kSmemMisc + 512;      // the running task's et_op record (copied before its waits)
constexpr int kSmemPre = kSmemOp + 256;       // small constant operands staged before the waits (RoPE freqs)
constexpr int kSmemTotal = kSmemPre + 512;

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
    int rt_len[kMaxRuntime];  // elements at the binding
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
    int step_id;         // stamped into trace records (dynamic: tasks that ran this step)
    int debug;           // ET_DEBUG env bits (timing experiments only): 1 = skip Event Tensor waits,
                         // 2 = record consumer ring-stall ns of warp 0 in the trace pad field
};

constexpr int kMaxDd = 128;  // data-dependent event tensors per graph (dynamic mode; one per MoE layer)

// Per-step control block of the dynamic scheduler (double-buffered).
struct DynCtl {
    unsigned int head[2];       // pop cursor per resource class (0 = SM, 1 = DMA)
    unsigned int tail[2];       // push cursor per resource class
    int total[2];               // tasks that will ever be pushed, per class
    int writer_rem[kMaxDd];     // writer-call tasks still running, per dd tensor
    int revealed[kMaxDd];
};

struct DynParams {
    int num_tasks;
    const int* task_call;
    const int* task_flat;
    const int* task_duration;
    const int* task_wait_off;
    const int* task_waits;
    const uint8_t* task_wait_armed;
    const int* task_notify_off;
    const int* task_notifies;
    const int* task_rem_init;
    const int* task_class;       // 0 = SM, 1 = DMA
    const int* consumer_off;
    const int* consumers;
    const int* call_first_task;
    const int* call_routed_rt;
    const int* call_routed_base;
    const int* call_range_rt;
    const int* call_range_base;
    const uint8_t* call_range_armed;
    int num_dd;
    int dd_base[kMaxDd];
    int dd_count[kMaxDd];
    int dd_counts_rt[kMaxDd];
    int dd_writer_call[kMaxDd];
    int dd_range_call[kMaxDd];   // call range-triggered by this tensor, or -1
    int dd_range_uniform_el[kMaxDd];  // the one element all its tasks notify, or -1
    const int* el_dd;
    int num_ready[2];
    int class_total[2];          // tasks per resource class (before extent_from shrink)
    const int* ready;            // seeded tasks, SM class then DMA class
    int early_push;
    // state: this step and the other parity (reset for the next step)
    DynCtl* ctl;
    DynCtl* ctl_other;
    int* rem;
    int* rem_other;
    int* slots;        // [2][num_tasks] task id + 1, 0 = not yet pushed
    int* slots_other;
    unsigned int* fired;
    unsigned int* fired_other;
    unsigned int* disp;
    unsigned int* disp_other;
    unsigned long long* push_time;
    int writer_tasks[kMaxDd];    // task count of each dd tensor's writer call
    // packed per-task / per-element records (one 16-byte load each on the hot path)
    const int4* task_desc;       // (call, coord0, coord1, ext0 of the call at the sample)
    const int4* task_rng;        // (wait_off, wait_end, notify_off, notify_end)
    const int4* el_info;         // (consumer_off, consumer_end, dd tensor or -1, initial count)
    const int* call_dd;          // per call: first data-dependent tensor it writes | count << 16, or -1
    const int4* task_note;       // first notify of the task when static: (element, consumer_off,
                                 // consumer_end, initial count), else element = -1
    // consumers[] entries carry bit 31 when that consumer has exactly one pending
    // wait (it is ready the moment the element fires: no rem[] decrement needed)
};

constexpr int kSmemCallExt = kSmemTable;       // dynamic kernel: per-call grid extents at the binding and
                                               // the data-dependent tensors it writes (int4)
constexpr int kMaxCallExt = (kSmemBar - kSmemTable) / 16;

}  // namespace etk

// Host-side launcher (megakernel.cu).
// moe != 0 selects the instantiation that contains the MoE tile bodies
int et_launch_static(const etk::StaticParams& p, int num_workers, int max_batch, int variant, void* stream);
int et_static_smem_bytes();
int et_launch_dynamic(const etk::StaticParams& p, const etk::DynParams& d, int num_workers, int variant, void* stream);
int et_dynamic_reset(const etk::StaticParams& p, const etk::DynParams& d, void* stream);
