/*
 * et_runtime.h — C ABI of the B200 Event Tensor megakernel runtime.
 *
 * This is the drop-in boundary for the reference's executor:
 *   ref proj/include/etsim/simulate.hpp:23  simulate(const StaticMegakernel&, binding, realization*, SimConfig)
 *   ref proj/include/etsim/simulate.hpp:29  simulate(const DynamicMegakernel&, ...)
 *   ref proj/src/simulate.cpp:88-298        StaticEngine   (queue walk, WAIT spin, NOTIFY atomic dec)
 *   ref proj/src/simulate.cpp:303-668       DynamicEngine  (push/pop ready queue, early push, reveal)
 * The reference runs those as a CPU discrete-event simulation; here one
 * persistent sm_100a kernel launch executes a whole step on the GPU.
 * The C++ API (headers under include/etsim/) and the Python module are thin layers
 * that lower graphs on the host, flatten them into the plain arrays below and
 * call these functions.  Plain pointers and sizes only; no C++ or torch types.
 *
 * Ownership: the caller owns every host array passed in (copied during the
 * call); the runtime owns all device memory it allocates.  Device pointers
 * inside et_op (weights, activations, KV caches) belong to the caller and
 * must outlive the steps that use them.  One runtime per device and stream;
 * handles are not thread-safe.
 *
 * Status codes: 0 = OK; ET_ERR_INVALID maps to etsim::Error (Python
 * GraphError); ET_ERR_DEADLOCK / ET_ERR_UNDERFLOW / ET_ERR_STEP_LIMIT map to
 * etsim::SimError kinds (Python SimulationError), as in
 * ref proj/python/bindings.cpp:99-109.
 */
#ifndef ET_RUNTIME_H_
#define ET_RUNTIME_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ET_ABI_VERSION 1

enum et_status {
    ET_OK = 0,
    ET_ERR_INVALID = 1,
    ET_ERR_CUDA = 2,
    ET_ERR_DEADLOCK = 3,
    ET_ERR_UNDERFLOW = 4,
    ET_ERR_STEP_LIMIT = 5,
    ET_ERR_NO_DEVICE = 6
};

enum et_mode { ET_MODE_STATIC = 0, ET_MODE_DYNAMIC = 1 };

/* Tile operations a device function can be bound to (per call).  ET_OP_NONE
 * runs the synthetic body: spin for duration * tick_ns nanoseconds. */
enum et_op_kind {
    ET_OP_NONE = 0,
    ET_OP_SPLITK_PARTIAL = 1, /* int32 partial row sums (paper section 2.2)       */
    ET_OP_SPLITK_FINAL = 2,   /* int32 final row sums over the partials            */
    ET_OP_GEMV = 3,           /* row-range GEMV, fused RMSNorm prologue, epilogues */
    ET_OP_ATTN_SPLIT = 4,     /* split-K (flash-decoding) attention over KV cache  */
    ET_OP_ATTN_MERGE = 5,     /* merge splits + new token, append KV               */
    ET_OP_MOE_ROUTE = 6,      /* router GEMV + top-k + counts + indptr             */
    ET_OP_MOE_EXPERT = 7,     /* expert gate/up/down for one routed tile           */
    ET_OP_ALLREDUCE = 8,      /* NVLink peer-memory allreduce (tensor parallel)    */
    ET_OP_MOE_GROUP = 9,      /* scatter routed (token, k) slots into expert lists */
    ET_OP_MOE_COMBINE = 10,   /* weighted combine of expert outputs + residual     */
    ET_OP_ARGMAX = 11,        /* greedy token from the lm_head's argmax words      */
    ET_OP_EMBED = 12,         /* embedding rows of the step's tokens -> fp32 stream */
    ET_OP_GEMV_TC = 13,       /* large-batch GEMV on tcgen05 tensor cores (TMEM)   */
    ET_OP_NORM = 14,          /* RMSNorm of the stream -> bf16 tensor-core operand */
    ET_OP_REDUCE = 15,        /* sum of k-split partial tiles (GEMM + reduce-scatter) */
    ET_OP_COPY = 16,          /* chunk copy (all-gather + GEMM, DMA queue)         */
    ET_OP_KIND_LAST = 16      /* (highest kind with a device body; et_bind_ops rejects
                                 the rest, and ET_OP_MOE_GROUP / ET_OP_MOE_COMBINE,
                                 whose work the routed notify and the expert tiles'
                                 red.add epilogue absorb) */
};

/* One bound tile operation.  Meaning of i[], f[], p[] is per kind and is
 * documented in paper_2604_13327_b200/csrc/kernels/ops.cuh. */
typedef struct et_op {
    int32_t kind;
    int32_t flags;
    int32_t i[14];
    float f[4];
    uint64_t p[12];
} et_op;

typedef struct et_config {
    int32_t device;
    int32_t num_workers;     /* persistent CTAs == SM queues of the program        */
    int32_t record_trace;    /* write per-slot timestamps                          */
    int32_t enable_prefetch; /* producer warp stages weights ahead of the waits     */
    int64_t watchdog_ns;     /* a wait spinning longer than this reports deadlock   */
    int64_t tick_ns;         /* synthetic body length per duration unit            */
    int64_t step_limit;      /* > 0: abort after this many executed tasks (StepLimit) */
    int32_t max_batch;       /* largest batch a GEMV tile sees (<= 8)               */
    int32_t reserved;
    int64_t l2_prefetch_bytes; /* per worker: weights prefetched into L2 beyond the
                                  shared-memory ring (< 0: default)                  */
} et_config;

/* Shape-independent description of the graph (uploaded once). */
typedef struct et_graph_desc {
    int32_t num_symbols;             /* GraphFunction::symbols order            */
    int32_t num_calls;
    const int32_t* call_rank;        /* [num_calls], <= 4                        */
    const int32_t* call_extent_from; /* [num_calls] runtime tensor index or -1   */
    const int32_t* grid_code_off;    /* [num_calls*4+1] postfix code per (call,dim) */
    const int32_t* code_op;          /* etsim::ExprOp                             */
    const int64_t* code_arg;
    int32_t code_len;
    int32_t num_runtime_tensors;
    const int64_t* runtime_capacity; /* [num_runtime_tensors] int32 elements to allocate */
    const int32_t* runtime_len_off;  /* [num_runtime_tensors+1] postfix code of each tensor's length */
} et_graph_desc;

/* One sampled static schedule (ref sched_static.hpp:22-37), flattened.  Slots
 * are listed queue by queue; queue q spans [queue_off[q], queue_off[q+1]).  When
 * has_dma is set, queue num_queues is the DMA channel. */
typedef struct et_sample_desc {
    const int64_t* binding;          /* [num_symbols]                             */
    const int32_t* call_extents;     /* [num_calls*4] grid extents at the sample  */
    int32_t num_queues;
    int32_t has_dma;
    const int32_t* queue_off;        /* [num_queues + has_dma + 1]                */
    int32_t num_slots;
    const int32_t* slot_task;        /* task id in the sample's materialization   */
    const int32_t* slot_call;
    const int32_t* slot_flat;        /* row-major index in the call's sample grid  */
    const int32_t* slot_duration;    /* synthetic duration units, may be NULL     */
    const int32_t* wait_off;         /* [num_slots+1]                              */
    const int32_t* waits;
    const int32_t* notify_off;       /* [num_slots+1]                              */
    const int32_t* notifies;
    int32_t num_counters;
    const int32_t* initial_counts;   /* [num_counters]                             */
    const int32_t* counter_dd;       /* [num_counters] runtime counts tensor or -1 (dynamic) */
} et_sample_desc;

/* Dynamic-scheduler program for one sample (ref sched_dynamic.hpp and the
 * engine state of ref simulate.cpp:303-354), flattened.  Tasks are the sample
 * grids' tasks in program order (id = call_first_task[call] + flat).  Static
 * map edges are resolved on the host; data-dependent edges are resolved on the
 * device from runtime tensors written by their writer task:
 *   routed notify  (ref materialize.cpp:288-304): element = base + routing[flat]
 *   range trigger  (ref materialize.cpp:252-273): task f of the call waits on
 *                  base + g where indptr[g] <= f < indptr[g+1]; tasks at or past
 *                  indptr[last] do not exist (extent_from)
 * Data-dependent elements get their initial count from their counts tensor and
 * become visible when the writer call's tasks have all finished (ref
 * simulate.cpp:326-345, 632-649). */
typedef struct et_dynamic_desc {
    int32_t num_tasks;
    const int32_t* task_call;           /* [num_tasks]                               */
    const int32_t* task_flat;           /* row-major index in the call's sample grid */
    const int32_t* task_duration;       /* synthetic duration units, may be NULL     */
    const int32_t* task_wait_off;       /* [num_tasks+1] static-map waits            */
    const int32_t* task_waits;
    const uint8_t* task_wait_armed;     /* aligned with task_waits                   */
    const int32_t* task_notify_off;     /* [num_tasks+1] static-map notifies         */
    const int32_t* task_notifies;
    const int32_t* task_rem_init;       /* waits that must fire before the push      */
    const int32_t* consumer_off;        /* [num_counters+1] static-map consumers     */
    const int32_t* consumers;
    const int32_t* call_first_task;     /* [num_calls]                               */
    const int32_t* call_routed_rt;      /* routing tensor of a routed notify, or -1  */
    const int32_t* call_routed_base;    /* event element base of that notify         */
    const int32_t* call_range_rt;       /* indptr tensor of a range trigger, or -1   */
    const int32_t* call_range_base;
    const uint8_t* call_range_armed;
    int32_t num_dd;                     /* data-dependent event tensors              */
    const int32_t* dd_base;             /* [num_dd] first element                    */
    const int32_t* dd_count;            /* [num_dd] elements                         */
    const int32_t* dd_counts_rt;        /* [num_dd] runtime tensor holding counts    */
    const int32_t* dd_writer_call;      /* [num_dd] call whose completion reveals it */
    const int32_t* el_dd;               /* [num_counters] dd tensor index or -1      */
    int32_t num_ready;                  /* tasks ready at launch (seeded in id order)*/
    const int32_t* ready;
    int32_t early_push;
} et_dynamic_desc;

/* Per-slot (static) or per-task (dynamic) trace record, nanoseconds of
 * %globaltimer.  flags bit0 = masked no-op. */
typedef struct et_trace_rec {
    int64_t t_push;       /* dynamic: task entered the ready queue (0: seeded) */
    int64_t t_begin;      /* slot reached / task popped                 */
    int64_t t_wait_end;   /* all waits satisfied                        */
    int64_t t_prologue;   /* body prologue done (activations staged), 0 if none */
    int64_t t_exec_end;   /* body finished                              */
    int64_t t_notify_end; /* all notifies issued                        */
    int32_t worker;
    int32_t flags;
    int32_t task;         /* slot index (static) / task id (dynamic)    */
    int32_t pad;
} et_trace_rec;

/* Outcome of the last step.  On a device-detected failure `worker`, `slot`,
 * `counter` and `value` locate the first blocked or underflowing wait. */
typedef struct et_step_info {
    int32_t status;
    int32_t sample_index;
    int32_t worker;
    int32_t slot;
    int32_t counter;
    int32_t value;
    int64_t tasks_executed;
    int64_t noop_tasks;
    int64_t pushes;
    int64_t pops;
    float kernel_ms;      /* CUDA-event time of the step's launch (when synchronous) */
    int32_t step_id;      /* stamped into the trace records' pad field             */
} et_step_info;

typedef struct et_runtime et_runtime;

int et_abi_version(void);
int et_device_count(int* count);
int et_create(const et_config* cfg, et_runtime** out);
int et_destroy(et_runtime* rt);
const char* et_last_error(const et_runtime* rt);

int et_upload_graph(et_runtime* rt, const et_graph_desc* g);
/* Replaces all samples; `samples` must be sorted as the kernel selects them
 * (ascending size symbol, ref sched_static.cpp:101-104). */
int et_upload_static(et_runtime* rt, const et_sample_desc* samples, int32_t num_samples);
int et_upload_dynamic(et_runtime* rt, const et_sample_desc* samples, const et_dynamic_desc* dyn,
                      int32_t num_samples);
int et_bind_ops(et_runtime* rt, const et_op* ops, int32_t num_calls);
/* Ahead-of-time program image (replaces ref json_io.cpp:294-376 / 455-494, the
 * reference's kernel_to_json / kernel_from_json "compile once, run many" form):
 * et_save_program writes the graph and static samples exactly as uploaded (flat
 * arrays, length-prefixed) plus an opaque metadata blob (the Python Executor stores
 * the symbol / runtime-tensor / call names there); et_load_program uploads a saved
 * image into a fresh runtime -- no lowering, no flattening -- and returns the
 * metadata (*meta_len in: capacity of meta_out, out: its size; meta_out may be
 * NULL to query).  Op tables hold this process's device pointers and are bound
 * again after a load (et_bind_ops).  Dynamic programs have no image. */
int et_save_program(et_runtime* rt, const char* path, const void* meta, int64_t meta_len);
int et_load_program(et_runtime* rt, const char* path, void* meta_out, int64_t* meta_len);

/* Copies host values into a runtime tensor (a routing realization supplied by
 * the host).  Tensors not written this way are produced on the device by their
 * writer task (e.g. ET_OP_MOE_ROUTE). */
int et_set_runtime_tensor(et_runtime* rt, int32_t index, const int32_t* values, int64_t n);
int et_clear_runtime_tensors(et_runtime* rt);
int et_get_runtime_tensor(et_runtime* rt, int32_t index, int32_t* values, int64_t n);

/* Runs one step at the binding (values in graph-symbol order).  The smallest
 * sample covering the binding on every symbol is selected (ref
 * sched_static.cpp:111-139); grids, masks and extent_from are evaluated on the
 * device.  `stream` is a cudaStream_t (NULL = the runtime's stream).  With
 * synchronous != 0 the call waits and fills `info` (may be NULL); otherwise it
 * only enqueues the launch (use et_sync to collect status). */
int et_step(et_runtime* rt, const int64_t* binding, int32_t num_symbols, void* stream, int32_t synchronous,
            et_step_info* info);
int et_sync(et_runtime* rt, et_step_info* info);
/* Diagnostics only (timing experiments, scripts/diag_*.py): the megakernel's
 * debug bits (StaticParams::debug in csrc/kernels/megakernel.cuh; 0 = normal).
 * Initialised from the ET_DEBUG environment variable at et_create. */
int et_set_debug(et_runtime* rt, int32_t bits);
/* Per-worker L2 run-ahead of the weight producer in bytes (et_config.l2_prefetch_bytes;
 * negative = off), changeable between steps. */
int et_set_l2_prefetch(et_runtime* rt, int64_t bytes);

/* Event Tensor counters of the last step in the reference's representation
 * (initial count minus notifies received; all zero after a clean step). */
int et_read_counters(et_runtime* rt, int64_t* out, int64_t n);
/* Trace of the last step: fills up to *n records and sets *n to the count. */
int et_read_trace(et_runtime* rt, et_trace_rec* out, int64_t* n);

/* Peer memory for tensor parallelism (setup only; the handles are exchanged by
 * the caller, e.g. over torch.distributed).  The row-parallel allreduce task
 * (ET_OP_ALLREDUCE) then reads peers' partials and stores peers' Event Tensor
 * flags through these mappings over NVLink -- no NCCL on the data path.  The
 * reference has no counterpart (it models TP only as task graphs, ref
 * workloads.cpp:30-79; SPEC.md:8 excludes multi-GPU). */
int et_ipc_get_handle(const void* dev_ptr, void* handle /* 64 bytes */);
int et_ipc_open_handle(const void* handle /* 64 bytes */, int32_t device, void** dev_ptr);
int et_ipc_close_handle(void* dev_ptr);

#ifdef __cplusplus
}
#endif

#endif /* ET_RUNTIME_H_ */
