// C-ABI runtime (include/et_runtime.h): device memory for programs, counters,
// runtime tensors, status and traces; sample selection; one cooperative
// launch of the persistent megakernel per step.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../kernels/megakernel.cuh"
#include "../kernels/ops.cuh"
#include "et_runtime.h"

namespace {

template <typename T>
struct DevArray {
    T* ptr = nullptr;
    size_t n = 0;
    DevArray() = default;
    DevArray(const DevArray&) = delete;
    DevArray& operator=(const DevArray&) = delete;
    DevArray(DevArray&& o) noexcept : ptr(o.ptr), n(o.n) { o.ptr = nullptr, o.n = 0; }
    DevArray& operator=(DevArray&& o) noexcept {
        if (this != &o) {
            release();
            ptr = o.ptr, n = o.n;
            o.ptr = nullptr, o.n = 0;
        }
        return *this;
    }
    ~DevArray() { release(); }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        n = 0;
    }
    cudaError_t alloc(size_t count) {
        release();
        n = count;
        if (count == 0) return cudaSuccess;
        return cudaMalloc(&ptr, count * sizeof(T));
    }
    cudaError_t upload(const T* host, size_t count) {
        cudaError_t e = alloc(count);
        if (e != cudaSuccess || count == 0) return e;
        if (!host) return cudaMemset(ptr, 0, count * sizeof(T));
        return cudaMemcpy(ptr, host, count * sizeof(T), cudaMemcpyHostToDevice);
    }
};

struct Sample {
    std::vector<int64_t> binding;
    std::vector<int32_t> call_extents;
    int num_queues = 0, has_dma = 0, num_slots = 0, num_counters = 0;
    std::vector<int32_t> initial_counts;  // host copy for counter readback
    int table_ok = 1;                     // all grid extents < 65536 (16-bit slot-table coordinates)
    DevArray<int32_t> d_call_extents, d_queue_off, d_slot_call, d_slot_flat, d_slot_duration, d_wait_off, d_waits,
        d_notify_off, d_notifies, d_initial;
    // dynamic scheduler program (ET_MODE_DYNAMIC)
    int num_tasks = 0;
    etk::DynParams dyn{};  // device pointers into the arrays below + scalars
    DevArray<int32_t> d_task_call, d_task_flat, d_task_duration, d_task_wait_off, d_task_waits, d_task_notify_off,
        d_task_notifies, d_task_rem_init, d_task_class, d_consumer_off, d_consumers, d_call_first_task, d_call_routed_rt,
        d_call_routed_base, d_call_range_rt, d_call_range_base, d_el_dd, d_ready;
    DevArray<int4> d_task_desc, d_task_rng, d_el_info, d_task_note;
    DevArray<int32_t> d_call_dd;
    DevArray<uint8_t> d_task_wait_armed, d_call_range_armed;
};

int64_t eval_host(const std::vector<int32_t>& op, const std::vector<int64_t>& arg, int b, int e,
                  const int64_t* binding, bool* ok) {
    int64_t st[32];
    int sp = 0;
    for (int i = b; i < e; ++i) {
        if (op[i] == 0 || op[i] == 1) {
            if (sp >= 32) {
                *ok = false;
                return 0;
            }
            st[sp++] = op[i] == 0 ? arg[i] : binding[arg[i]];
            if (st[sp - 1] < 0) *ok = false;
            continue;
        }
        if (sp < 2) {
            *ok = false;
            return 0;
        }
        const int64_t y = st[--sp], x = st[sp - 1];
        int64_t r = 0;
        switch (op[i]) {
            case 2: r = x + y; break;
            case 3: r = x * y; break;
            case 4: if (y == 0) { *ok = false; return 0; } r = x / y; break;
            case 5: if (y == 0) { *ok = false; return 0; } r = x % y; break;
            case 6: r = std::min(x, y); break;
            default: r = std::max(x, y); break;
        }
        if (r < 0) *ok = false;
        st[sp - 1] = r;
    }
    return sp ? st[0] : 0;
}

}  // namespace

struct et_runtime {
    et_config cfg{};
    std::string err;
    cudaStream_t stream = nullptr;
    int sm_count = 0;

    // graph
    int num_symbols = 0, num_calls = 0;
    std::vector<int32_t> call_rank, call_extent_from, grid_code_off, code_op, rt_len_off;
    std::vector<int64_t> code_arg, rt_capacity;
    DevArray<int32_t> d_call_rank, d_call_extent_from, d_grid_code_off, d_code_op;
    DevArray<int64_t> d_code_arg;
    std::vector<DevArray<int32_t>> d_rt;
    DevArray<int*> d_rt_table;

    std::vector<Sample> samples;
    DevArray<et_op> d_ops;
    int has_moe = 0;  // kernel variant: bit 0 MoE bodies, bit 1 tensor-core GEMV bodies (bound ops)
    int ops_bound = 0;
    // per-step host work memoised by binding: the covering sample and the runtime tensor
    // lengths of the last binding (a serving loop repeats shapes); reset by every upload
    // and op-table bind
    std::vector<int64_t> memo_binding;
    int memo_pick = -1;
    std::vector<int> memo_rt_len;
    std::vector<et_op> h_ops;  // host copy of the bound op table (launch-time capacity checks)

    int mode = ET_MODE_STATIC;
    // dynamic scheduler state, two parities
    DevArray<etk::DynCtl> d_ctl;
    DevArray<int> d_rem, d_slots;
    DevArray<unsigned int> d_fired, d_disp;
    DevArray<unsigned long long> d_push_time;
    int max_tasks = 0;
    int prepared[2] = {-1, -1};  // sample each parity's state was initialised for
    DevArray<uint32_t> d_cnt;  // [2][cap]
    int cnt_capacity = 0;
    DevArray<etk::DevStatus> d_status;  // [2]
    DevArray<et_trace_rec> d_trace;
    int parity = 0;
    int steps = 0;
    int last_sample = -1;
    bool launched = false;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    bool timed = false;  // ev0/ev1 bracket the last launch (synchronous steps only)
    int debug = 0;       // ET_DEBUG at et_create
    // program image (et_save_program): the graph and static samples as uploaded
    std::vector<uint8_t> img_graph, img_samples;
    bool img_static = false;

    int fail(int code, const std::string& m) {
        err = m;
        return code;
    }
    int cuda_fail(cudaError_t e, const char* what) {
        err = std::string(what) + ": " + cudaGetErrorString(e);
        return ET_ERR_CUDA;
    }
};

#define ET_CUDA(call, what)                                   \
    do {                                                      \
        cudaError_t e__ = (call);                             \
        if (e__ != cudaSuccess) return rt->cuda_fail(e__, what); \
    } while (0)

namespace {
// Program image: length-prefixed little-endian arrays, in the field order of the
// descriptors (include/et_runtime.h), so a load needs no lowering.
struct ImgOut {
    std::vector<uint8_t>& b;
    void raw(const void* p, size_t n) {
        const uint8_t* c = static_cast<const uint8_t*>(p);
        b.insert(b.end(), c, c + n);
    }
    void i64(int64_t v) { raw(&v, 8); }
    template <typename T>
    void arr(const T* p, int64_t n) {
        i64(p ? n : -1);
        if (p && n > 0) raw(p, static_cast<size_t>(n) * sizeof(T));
    }
};
struct ImgIn {
    const uint8_t* p;
    const uint8_t* e;
    bool ok = true;
    int64_t i64() {
        int64_t v = 0;
        if (e - p < 8) { ok = false; return 0; }
        std::memcpy(&v, p, 8);
        p += 8;
        return v;
    }
    template <typename T>
    std::vector<T> arr(bool* present = nullptr) {
        const int64_t n = i64();
        if (present) *present = n >= 0;
        std::vector<T> v(static_cast<size_t>(n > 0 ? n : 0));
        const size_t bytes = v.size() * sizeof(T);
        if (static_cast<size_t>(e - p) < bytes) { ok = false; return {}; }
        if (bytes) std::memcpy(v.data(), p, bytes);
        p += bytes;
        return v;
    }
};
constexpr char kImgMagic[8] = {'E', 'T', 'P', 'R', 'O', 'G', '0', '1'};
}  // namespace

extern "C" {

int et_abi_version(void) { return ET_ABI_VERSION; }

int et_device_count(int* count) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) n = 0;
    if (count) *count = n;
    return n > 0 ? ET_OK : ET_ERR_NO_DEVICE;
}

int et_create(const et_config* cfg, et_runtime** out) {
    if (!cfg || !out) return ET_ERR_INVALID;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return ET_ERR_NO_DEVICE;
    if (cfg->device < 0 || cfg->device >= n) return ET_ERR_INVALID;
    et_runtime* rt = new et_runtime();
    rt->cfg = *cfg;
    if (rt->cfg.watchdog_ns <= 0) rt->cfg.watchdog_ns = 2'000'000'000LL;
    cudaError_t e = cudaSetDevice(cfg->device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&rt->sm_count, cudaDevAttrMultiProcessorCount, cfg->device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&rt->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreate(&rt->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&rt->ev1);
    if (e == cudaSuccess) e = rt->d_status.alloc(2);
    if (e == cudaSuccess) e = cudaMemset(rt->d_status.ptr, 0, 2 * sizeof(etk::DevStatus));
    if (e != cudaSuccess) {
        delete rt;
        return ET_ERR_CUDA;
    }
    if (rt->cfg.num_workers <= 0) rt->cfg.num_workers = rt->sm_count;
    {  // timing-experiment switches (megakernel.cuh StaticParams::debug), read once
        const char* dbg = getenv("ET_DEBUG");
        rt->debug = dbg ? atoi(dbg) : 0;
    }
    *out = rt;
    return ET_OK;
}

int et_destroy(et_runtime* rt) {
    if (!rt) return ET_OK;
    cudaSetDevice(rt->cfg.device);
    if (rt->stream) cudaStreamSynchronize(rt->stream);
    if (rt->ev0) cudaEventDestroy(rt->ev0);
    if (rt->ev1) cudaEventDestroy(rt->ev1);
    if (rt->stream) cudaStreamDestroy(rt->stream);
    delete rt;
    return ET_OK;
}

const char* et_last_error(const et_runtime* rt) { return rt ? rt->err.c_str() : "null runtime"; }

int et_upload_graph(et_runtime* rt, const et_graph_desc* g) {
    if (!rt || !g) return ET_ERR_INVALID;
    if (g->num_symbols > etk::kMaxSymbols) return rt->fail(ET_ERR_INVALID, "too many symbols for the device binding");
    if (g->num_runtime_tensors > etk::kMaxRuntime) return rt->fail(ET_ERR_INVALID, "too many runtime tensors");
    cudaSetDevice(rt->cfg.device);
    rt->num_symbols = g->num_symbols;
    rt->num_calls = g->num_calls;
    rt->call_rank.assign(g->call_rank, g->call_rank + g->num_calls);
    rt->call_extent_from.assign(g->call_extent_from, g->call_extent_from + g->num_calls);
    rt->grid_code_off.assign(g->grid_code_off, g->grid_code_off + g->num_calls * 4 + 1);
    rt->code_op.assign(g->code_op, g->code_op + g->code_len);
    rt->code_arg.assign(g->code_arg, g->code_arg + g->code_len);
    for (int c = 0; c < g->num_calls; ++c)
        if (rt->call_rank[c] > etk::kMaxRank) return rt->fail(ET_ERR_INVALID, "grid rank above 4 is not supported");
    ET_CUDA(rt->d_call_rank.upload(rt->call_rank.data(), rt->call_rank.size()), "upload graph");
    ET_CUDA(rt->d_call_extent_from.upload(rt->call_extent_from.data(), rt->call_extent_from.size()), "upload graph");
    ET_CUDA(rt->d_grid_code_off.upload(rt->grid_code_off.data(), rt->grid_code_off.size()), "upload graph");
    ET_CUDA(rt->d_code_op.upload(rt->code_op.data(), std::max<size_t>(1, rt->code_op.size())), "upload graph");
    ET_CUDA(rt->d_code_arg.upload(rt->code_arg.data(), std::max<size_t>(1, rt->code_arg.size())), "upload graph");
    rt->rt_capacity.assign(g->runtime_capacity, g->runtime_capacity + g->num_runtime_tensors);
    rt->rt_len_off.assign(g->runtime_len_off, g->runtime_len_off + g->num_runtime_tensors + 1);
    rt->d_rt.clear();
    rt->d_rt.resize(static_cast<size_t>(g->num_runtime_tensors));
    std::vector<int*> table(static_cast<size_t>(std::max(1, g->num_runtime_tensors)), nullptr);
    for (int i = 0; i < g->num_runtime_tensors; ++i) {
        ET_CUDA(rt->d_rt[static_cast<size_t>(i)].upload(nullptr, static_cast<size_t>(std::max<int64_t>(1, rt->rt_capacity[i]))),
                "runtime tensors");
        table[static_cast<size_t>(i)] = rt->d_rt[static_cast<size_t>(i)].ptr;
    }
    ET_CUDA(rt->d_rt_table.upload(table.data(), table.size()), "runtime tensors");
    rt->samples.clear();
    rt->memo_pick = -1;
    rt->last_sample = -1;
    rt->img_graph.clear();
    rt->img_samples.clear();
    rt->img_static = false;
    ImgOut o{rt->img_graph};
    o.i64(g->num_symbols);
    o.arr(g->call_rank, g->num_calls);
    o.arr(g->call_extent_from, g->num_calls);
    o.arr(g->grid_code_off, g->num_calls * 4 + 1);
    o.arr(g->code_op, g->code_len);
    o.arr(g->code_arg, g->code_len);
    o.arr(g->runtime_capacity, g->num_runtime_tensors);
    o.arr(g->runtime_len_off, g->num_runtime_tensors + 1);
    return ET_OK;
}

int et_upload_static(et_runtime* rt, const et_sample_desc* s, int32_t num_samples) {
    if (!rt || (!s && num_samples > 0)) return ET_ERR_INVALID;
    cudaSetDevice(rt->cfg.device);
    cudaStreamSynchronize(rt->stream);
    rt->samples.clear();
    rt->memo_pick = -1;
    rt->samples.resize(static_cast<size_t>(num_samples));
    int max_counters = 1, max_slots = 1;
    for (int i = 0; i < num_samples; ++i) {
        const et_sample_desc& d = s[i];
        Sample& S = rt->samples[static_cast<size_t>(i)];
        if (d.num_queues != rt->cfg.num_workers)
            return rt->fail(ET_ERR_INVALID, "kernel was compiled for " + std::to_string(d.num_queues) +
                                                " SMs, run asked for " + std::to_string(rt->cfg.num_workers));
        if (d.num_queues > rt->sm_count)
            return rt->fail(ET_ERR_INVALID, "program needs " + std::to_string(d.num_queues) +
                                                " co-resident workers; the device has " + std::to_string(rt->sm_count) +
                                                " SMs");
        S.binding.assign(d.binding, d.binding + rt->num_symbols);
        S.call_extents.assign(d.call_extents, d.call_extents + rt->num_calls * 4);
        S.num_queues = d.num_queues;
        S.has_dma = d.has_dma;
        S.num_slots = d.num_slots;
        S.num_counters = d.num_counters;
        S.initial_counts.assign(d.initial_counts, d.initial_counts + d.num_counters);
        for (int c = 0; c < rt->num_calls; ++c)
            for (int k = 0; k < 4; ++k)
                if (S.call_extents[static_cast<size_t>(c * 4 + k)] >= 65536) S.table_ok = 0;
        const size_t nq = static_cast<size_t>(d.num_queues + d.has_dma + 1);
        const int nw = d.wait_off[d.num_slots], nn = d.notify_off[d.num_slots];
        ET_CUDA(S.d_call_extents.upload(d.call_extents, static_cast<size_t>(rt->num_calls * 4)), "upload sample");
        ET_CUDA(S.d_queue_off.upload(d.queue_off, nq), "upload sample");
        ET_CUDA(S.d_slot_call.upload(d.slot_call, static_cast<size_t>(std::max(1, d.num_slots))), "upload sample");
        ET_CUDA(S.d_slot_flat.upload(d.slot_flat, static_cast<size_t>(std::max(1, d.num_slots))), "upload sample");
        if (d.slot_duration)
            ET_CUDA(S.d_slot_duration.upload(d.slot_duration, static_cast<size_t>(std::max(1, d.num_slots))), "upload sample");
        ET_CUDA(S.d_wait_off.upload(d.wait_off, static_cast<size_t>(d.num_slots + 1)), "upload sample");
        ET_CUDA(S.d_waits.upload(d.waits, static_cast<size_t>(std::max(1, nw))), "upload sample");
        ET_CUDA(S.d_notify_off.upload(d.notify_off, static_cast<size_t>(d.num_slots + 1)), "upload sample");
        ET_CUDA(S.d_notifies.upload(d.notifies, static_cast<size_t>(std::max(1, nn))), "upload sample");
        ET_CUDA(S.d_initial.upload(d.initial_counts, static_cast<size_t>(std::max(1, d.num_counters))), "upload sample");
        max_counters = std::max(max_counters, d.num_counters);
        max_slots = std::max(max_slots, d.num_slots);
    }
    rt->cnt_capacity = max_counters;
    ET_CUDA(rt->d_cnt.upload(nullptr, static_cast<size_t>(2 * max_counters)), "counters");
    ET_CUDA(rt->d_trace.upload(nullptr, static_cast<size_t>(max_slots)), "trace");
    ET_CUDA(cudaMemset(rt->d_status.ptr, 0, 2 * sizeof(etk::DevStatus)), "status");
    rt->parity = 0;
    rt->last_sample = -1;
    rt->launched = false;
    rt->mode = ET_MODE_STATIC;
    rt->img_samples.clear();
    ImgOut o{rt->img_samples};
    o.i64(num_samples);
    for (int i = 0; i < num_samples; ++i) {
        const et_sample_desc& d = s[i];
        const int64_t nq = d.num_queues + d.has_dma + 1;
        o.i64(d.num_queues);
        o.i64(d.has_dma);
        o.i64(d.num_slots);
        o.i64(d.num_counters);
        o.arr(d.binding, rt->num_symbols);
        o.arr(d.call_extents, rt->num_calls * 4);
        o.arr(d.queue_off, nq);
        o.arr(d.slot_task, d.num_slots);
        o.arr(d.slot_call, d.num_slots);
        o.arr(d.slot_flat, d.num_slots);
        o.arr(d.slot_duration, d.num_slots);
        o.arr(d.wait_off, d.num_slots + 1);
        o.arr(d.waits, d.wait_off[d.num_slots]);
        o.arr(d.notify_off, d.num_slots + 1);
        o.arr(d.notifies, d.notify_off[d.num_slots]);
        o.arr(d.initial_counts, d.num_counters);
    }
    rt->img_static = true;
    return ET_OK;
}

int et_save_program(et_runtime* rt, const char* path, const void* meta, int64_t meta_len) {
    if (!rt || !path || meta_len < 0 || (meta_len > 0 && !meta)) return ET_ERR_INVALID;
    if (!rt->img_static) return rt->fail(ET_ERR_INVALID, "no static program uploaded (dynamic programs have no image)");
    FILE* f = std::fopen(path, "wb");
    if (!f) return rt->fail(ET_ERR_INVALID, std::string("cannot write ") + path);
    std::vector<uint8_t> head;
    ImgOut o{head};
    o.raw(kImgMagic, 8);
    o.i64(ET_ABI_VERSION);
    o.i64(rt->cfg.num_workers);
    o.arr(static_cast<const uint8_t*>(meta), meta_len);
    o.i64(static_cast<int64_t>(rt->img_graph.size()));
    o.i64(static_cast<int64_t>(rt->img_samples.size()));
    bool ok = std::fwrite(head.data(), 1, head.size(), f) == head.size();
    ok = ok && std::fwrite(rt->img_graph.data(), 1, rt->img_graph.size(), f) == rt->img_graph.size();
    ok = ok && std::fwrite(rt->img_samples.data(), 1, rt->img_samples.size(), f) == rt->img_samples.size();
    ok = std::fclose(f) == 0 && ok;
    return ok ? ET_OK : rt->fail(ET_ERR_INVALID, std::string("short write to ") + path);
}

int et_load_program(et_runtime* rt, const char* path, void* meta_out, int64_t* meta_len) {
    if (!rt || !path) return ET_ERR_INVALID;
    FILE* f = std::fopen(path, "rb");
    if (!f) return rt->fail(ET_ERR_INVALID, std::string("cannot read ") + path);
    std::vector<uint8_t> buf;
    uint8_t tmp[1 << 16];
    size_t n;
    while ((n = std::fread(tmp, 1, sizeof(tmp), f)) > 0) buf.insert(buf.end(), tmp, tmp + n);
    std::fclose(f);
    if (buf.size() < 8 || std::memcmp(buf.data(), kImgMagic, 8) != 0)
        return rt->fail(ET_ERR_INVALID, std::string(path) + " is not a program image");
    ImgIn in{buf.data() + 8, buf.data() + buf.size()};
    if (in.i64() != ET_ABI_VERSION) return rt->fail(ET_ERR_INVALID, "program image from another ABI version");
    const int64_t workers = in.i64();
    if (workers != rt->cfg.num_workers)
        return rt->fail(ET_ERR_INVALID, "program image was lowered for " + std::to_string(workers) + " workers");
    const std::vector<uint8_t> meta = in.arr<uint8_t>();
    if (meta_len) {
        const int64_t cap = *meta_len;
        *meta_len = static_cast<int64_t>(meta.size());
        if (meta_out && cap >= static_cast<int64_t>(meta.size()) && !meta.empty())
            std::memcpy(meta_out, meta.data(), meta.size());
    }
    in.i64();
    in.i64();
    // graph
    et_graph_desc g{};
    g.num_symbols = static_cast<int32_t>(in.i64());
    const auto call_rank = in.arr<int32_t>(), call_ef = in.arr<int32_t>(), grid_off = in.arr<int32_t>(),
               code_op = in.arr<int32_t>();
    const auto code_arg = in.arr<int64_t>(), rt_cap = in.arr<int64_t>();
    const auto rt_len_off = in.arr<int32_t>();
    if (!in.ok) return rt->fail(ET_ERR_INVALID, "truncated program image (graph)");
    g.num_calls = static_cast<int32_t>(call_rank.size());
    g.call_rank = call_rank.data();
    g.call_extent_from = call_ef.data();
    g.grid_code_off = grid_off.data();
    g.code_op = code_op.data();
    g.code_arg = code_arg.data();
    g.code_len = static_cast<int32_t>(code_op.size());
    g.num_runtime_tensors = static_cast<int32_t>(rt_cap.size());
    g.runtime_capacity = rt_cap.data();
    g.runtime_len_off = rt_len_off.data();
    int rc = et_upload_graph(rt, &g);
    if (rc != ET_OK) return rc;
    // samples
    const int64_t ns = in.i64();
    if (!in.ok || ns < 0 || ns > (1 << 20)) return rt->fail(ET_ERR_INVALID, "corrupt program image (samples)");
    struct S {
        std::vector<int64_t> binding;
        std::vector<int32_t> a[11];
        bool has_dur = false;
    };
    std::vector<S> keep(static_cast<size_t>(ns));
    std::vector<et_sample_desc> descs(static_cast<size_t>(ns));
    for (int64_t i = 0; i < ns; ++i) {
        S& k = keep[static_cast<size_t>(i)];
        et_sample_desc& d = descs[static_cast<size_t>(i)];
        d.num_queues = static_cast<int32_t>(in.i64());
        d.has_dma = static_cast<int32_t>(in.i64());
        d.num_slots = static_cast<int32_t>(in.i64());
        d.num_counters = static_cast<int32_t>(in.i64());
        k.binding = in.arr<int64_t>();
        for (int j = 0; j < 11; ++j) k.a[j] = in.arr<int32_t>(j == 5 ? &k.has_dur : nullptr);
        if (!in.ok) return rt->fail(ET_ERR_INVALID, "truncated program image (sample)");
        d.binding = k.binding.data();
        d.call_extents = k.a[0].data();
        d.queue_off = k.a[1].data();
        d.slot_task = k.a[2].data();
        d.slot_call = k.a[3].data();
        d.slot_flat = k.a[4].data();
        d.slot_duration = k.has_dur ? k.a[5].data() : nullptr;
        d.wait_off = k.a[6].data();
        d.waits = k.a[7].data();
        d.notify_off = k.a[8].data();
        d.notifies = k.a[9].data();
        d.initial_counts = k.a[10].data();
        d.counter_dd = nullptr;
    }
    return et_upload_static(rt, descs.data(), static_cast<int32_t>(ns));
}

int et_upload_dynamic(et_runtime* rt, const et_sample_desc* s, const et_dynamic_desc* dyn, int32_t num_samples) {
    if (!rt || !s || !dyn || num_samples <= 0) return ET_ERR_INVALID;
    int rc = et_upload_static(rt, s, num_samples);  // sample bindings, extents, counters, status
    if (rc != ET_OK) return rc;
    rt->mode = ET_MODE_DYNAMIC;
    rt->img_static = false;  // program images hold static schedules only
    for (int c = 0; c < rt->num_calls; ++c)
        if (rt->call_rank[static_cast<size_t>(c)] > 2)
            return rt->fail(ET_ERR_INVALID, "the dynamic scheduler supports grids of rank <= 2");
    int max_tasks = 1;
    for (int i = 0; i < num_samples; ++i) {
        const et_dynamic_desc& d = dyn[i];
        Sample& S = rt->samples[static_cast<size_t>(i)];
        if (d.num_dd > etk::kMaxDd) return rt->fail(ET_ERR_INVALID, "too many data-dependent event tensors");
        if (d.num_tasks >= (1 << 21) - 1)  // ready-queue slot words carry task + 1 in 21 bits
            return rt->fail(ET_ERR_INVALID, "the dynamic scheduler supports fewer than 2^21 - 1 tasks per sample");
        const size_t nt = static_cast<size_t>(std::max(1, d.num_tasks));
        const size_t nw = static_cast<size_t>(std::max(1, d.task_wait_off[d.num_tasks]));
        const size_t nn = static_cast<size_t>(std::max(1, d.task_notify_off[d.num_tasks]));
        const size_t nc = static_cast<size_t>(std::max(1, d.consumer_off[S.num_counters]));
        const size_t ncall = static_cast<size_t>(std::max(1, rt->num_calls));
        std::vector<int32_t> cls(nt, 0);
        int totals[2] = {0, 0};
        for (int t = 0; t < d.num_tasks; ++t) {
            // resource class from the queue layout: DMA-class tasks are flagged by slot_call's
            // queue in the static descriptor; here by the sample's has_dma + call list
            cls[static_cast<size_t>(t)] = 0;
        }
        if (S.has_dma && s[i].slot_task) {
            const int q0 = s[i].queue_off[S.num_queues], q1 = s[i].queue_off[S.num_queues + 1];
            for (int k = q0; k < q1; ++k) cls[static_cast<size_t>(s[i].slot_task[k])] = 1;
        }
        for (int t = 0; t < d.num_tasks; ++t) ++totals[cls[static_cast<size_t>(t)]];
        std::vector<int32_t> ready0, ready1;
        for (int k = 0; k < d.num_ready; ++k) (cls[static_cast<size_t>(d.ready[k])] ? ready1 : ready0).push_back(d.ready[k]);
        std::vector<int32_t> ready(ready0);
        ready.insert(ready.end(), ready1.begin(), ready1.end());
        S.num_tasks = d.num_tasks;
        ET_CUDA(S.d_task_call.upload(d.task_call, nt), "upload dynamic");
        ET_CUDA(S.d_task_flat.upload(d.task_flat, nt), "upload dynamic");
        if (d.task_duration) ET_CUDA(S.d_task_duration.upload(d.task_duration, nt), "upload dynamic");
        ET_CUDA(S.d_task_wait_off.upload(d.task_wait_off, nt + 1), "upload dynamic");
        ET_CUDA(S.d_task_waits.upload(d.task_waits, nw), "upload dynamic");
        ET_CUDA(S.d_task_wait_armed.upload(d.task_wait_armed, nw), "upload dynamic");
        ET_CUDA(S.d_task_notify_off.upload(d.task_notify_off, nt + 1), "upload dynamic");
        ET_CUDA(S.d_task_notifies.upload(d.task_notifies, nn), "upload dynamic");
        ET_CUDA(S.d_task_rem_init.upload(d.task_rem_init, nt), "upload dynamic");
        ET_CUDA(S.d_task_class.upload(cls.data(), nt), "upload dynamic");
        ET_CUDA(S.d_consumer_off.upload(d.consumer_off, static_cast<size_t>(S.num_counters) + 1), "upload dynamic");
        ET_CUDA(S.d_consumers.upload(d.consumers, nc), "upload dynamic");
        ET_CUDA(S.d_call_first_task.upload(d.call_first_task, ncall), "upload dynamic");
        ET_CUDA(S.d_call_routed_rt.upload(d.call_routed_rt, ncall), "upload dynamic");
        ET_CUDA(S.d_call_routed_base.upload(d.call_routed_base, ncall), "upload dynamic");
        ET_CUDA(S.d_call_range_rt.upload(d.call_range_rt, ncall), "upload dynamic");
        ET_CUDA(S.d_call_range_base.upload(d.call_range_base, ncall), "upload dynamic");
        ET_CUDA(S.d_call_range_armed.upload(d.call_range_armed, ncall), "upload dynamic");
        ET_CUDA(S.d_el_dd.upload(d.el_dd, static_cast<size_t>(std::max(1, S.num_counters))), "upload dynamic");
        {  // packed records for the device hot path
            std::vector<int4> desc(nt), rng(nt), info(static_cast<size_t>(std::max(1, S.num_counters)));
            for (int t = 0; t < d.num_tasks; ++t) {
                const int c = d.task_call[t];
                const int rank = rt->call_rank[static_cast<size_t>(c)];
                int flat = d.task_flat[t];
                int coord[4] = {0, 0, 0, 0};
                for (int k = rank - 1; k >= 0; --k) {
                    const int e = S.call_extents[static_cast<size_t>(c * 4 + k)];
                    coord[k] = e > 0 ? flat % e : 0;
                    flat = e > 0 ? flat / e : 0;
                }
                desc[static_cast<size_t>(t)] = make_int4(c, coord[0], coord[1], S.call_extents[static_cast<size_t>(c * 4)]);
                rng[static_cast<size_t>(t)] = make_int4(d.task_wait_off[t], d.task_wait_off[t + 1], d.task_notify_off[t],
                                                        d.task_notify_off[t + 1]);
            }
            for (int el = 0; el < S.num_counters; ++el)
                info[static_cast<size_t>(el)] = make_int4(d.consumer_off[el], d.consumer_off[el + 1], d.el_dd[el],
                                                          s[i].initial_counts[el]);
            std::vector<int4> note(nt, make_int4(-1, 0, 0, 0));
            for (int t = 0; t < d.num_tasks; ++t) {
                if (d.task_notify_off[t + 1] <= d.task_notify_off[t]) continue;
                const int el = d.task_notifies[d.task_notify_off[t]];
                if (d.el_dd[el] < 0) note[static_cast<size_t>(t)] = info[static_cast<size_t>(el)], note[static_cast<size_t>(t)].x = el,
                                     note[static_cast<size_t>(t)].y = d.consumer_off[el],
                                     note[static_cast<size_t>(t)].z = d.consumer_off[el + 1];
            }
            ET_CUDA(S.d_task_note.upload(note.data(), nt), "upload dynamic");
            // per call: the data-dependent tensors it writes (consecutive indices), first | count << 16
            std::vector<int32_t> cdd(static_cast<size_t>(std::max(1, rt->num_calls)), -1);
            for (int t = 0; t < d.num_dd; ++t) {
                const int c = d.dd_writer_call[t];
                if (c < 0 || c >= rt->num_calls) continue;
                int32_t& e = cdd[static_cast<size_t>(c)];
                if (e < 0) e = t | (1 << 16);
                else if ((e & 0xffff) + (e >> 16) == t) e += 1 << 16;
                else return rt->fail(ET_ERR_INVALID, "a call's data-dependent tensors must be consecutive");
            }
            ET_CUDA(S.d_call_dd.upload(cdd.data(), cdd.size()), "upload dynamic");
            std::vector<int32_t> cons(d.consumers, d.consumers + d.consumer_off[S.num_counters]);
            // task (bits 0..20), its call (21..29; 511 = more calls than fit), bit 30: DMA class,
            // bit 31: single pending wait (ready when this fires) -- megakernel.cu cons_task
            for (auto& c : cons) {
                const int t = c;
                const int call = d.task_call[t] < 511 ? d.task_call[t] : 511;
                c = t | (call << 21);
                if (cls[static_cast<size_t>(t)] == 1) c |= 0x40000000;
                if (d.task_rem_init[t] == 1 && d.call_range_rt[d.task_call[t]] < 0) c |= static_cast<int32_t>(0x80000000u);
            }
            ET_CUDA(S.d_consumers.upload(cons.empty() ? nullptr : cons.data(), nc), "upload dynamic");
            ET_CUDA(S.d_task_desc.upload(desc.data(), nt), "upload dynamic");
            ET_CUDA(S.d_task_rng.upload(rng.data(), nt), "upload dynamic");
            ET_CUDA(S.d_el_info.upload(info.data(), info.size()), "upload dynamic");
        }
        ET_CUDA(S.d_ready.upload(ready.empty() ? nullptr : ready.data(), std::max<size_t>(1, ready.size())),
                "upload dynamic");
        etk::DynParams& P = S.dyn;
        P = etk::DynParams{};
        P.num_tasks = d.num_tasks;
        P.task_call = S.d_task_call.ptr;
        P.task_flat = S.d_task_flat.ptr;
        P.task_duration = d.task_duration ? S.d_task_duration.ptr : nullptr;
        P.task_wait_off = S.d_task_wait_off.ptr;
        P.task_waits = S.d_task_waits.ptr;
        P.task_wait_armed = S.d_task_wait_armed.ptr;
        P.task_notify_off = S.d_task_notify_off.ptr;
        P.task_notifies = S.d_task_notifies.ptr;
        P.task_rem_init = S.d_task_rem_init.ptr;
        P.task_class = S.d_task_class.ptr;
        P.consumer_off = S.d_consumer_off.ptr;
        P.consumers = S.d_consumers.ptr;
        P.call_first_task = S.d_call_first_task.ptr;
        P.call_routed_rt = S.d_call_routed_rt.ptr;
        P.call_routed_base = S.d_call_routed_base.ptr;
        P.call_range_rt = S.d_call_range_rt.ptr;
        P.call_range_base = S.d_call_range_base.ptr;
        P.call_range_armed = S.d_call_range_armed.ptr;
        P.num_dd = d.num_dd;
        for (int t = 0; t < d.num_dd; ++t) {
            P.dd_base[t] = d.dd_base[t];
            P.dd_count[t] = d.dd_count[t];
            P.dd_counts_rt[t] = d.dd_counts_rt[t];
            P.dd_writer_call[t] = d.dd_writer_call[t];
            P.dd_range_call[t] = -1;
            for (int c = 0; c < rt->num_calls; ++c)
                if (d.call_range_rt[c] >= 0 && d.call_range_base[c] == d.dd_base[t]) P.dd_range_call[t] = c;
            // the element every task of the range call notifies, when there is exactly one (one
            // notify per task, the same element): the never-instantiated tail tasks are then
            // credited with a single add at reveal time instead of one atomic per task
            P.dd_range_uniform_el[t] = -1;
            if (P.dd_range_call[t] >= 0) {
                int el = -2;
                for (int task = 0; task < d.num_tasks && el != -1; ++task) {
                    if (d.task_call[task] != P.dd_range_call[t]) continue;
                    const int n0 = d.task_notify_off[task], n1 = d.task_notify_off[task + 1];
                    if (n1 - n0 != 1 || (el >= 0 && d.task_notifies[n0] != el)) el = -1;
                    else el = d.task_notifies[n0];
                }
                P.dd_range_uniform_el[t] = el >= 0 ? el : -1;
            }
            int wt = 1;
            for (int k = 0; k < rt->call_rank[static_cast<size_t>(d.dd_writer_call[t])]; ++k)
                wt *= S.call_extents[static_cast<size_t>(d.dd_writer_call[t] * 4 + k)];
            P.writer_tasks[t] = wt;
        }
        P.el_dd = S.d_el_dd.ptr;
        P.task_desc = S.d_task_desc.ptr;
        P.task_rng = S.d_task_rng.ptr;
        P.el_info = S.d_el_info.ptr;
        P.task_note = S.d_task_note.ptr;
        P.call_dd = S.d_call_dd.ptr;
        P.num_ready[0] = static_cast<int>(ready0.size());
        P.num_ready[1] = static_cast<int>(ready1.size());
        P.class_total[0] = totals[0];
        P.class_total[1] = totals[1];
        P.ready = S.d_ready.ptr;
        P.early_push = d.early_push;
        max_tasks = std::max(max_tasks, d.num_tasks);
    }
    rt->max_tasks = max_tasks;
    ET_CUDA(rt->d_ctl.upload(nullptr, 2), "dynamic state");
    ET_CUDA(rt->d_rem.upload(nullptr, static_cast<size_t>(2 * max_tasks)), "dynamic state");
    ET_CUDA(rt->d_slots.upload(nullptr, static_cast<size_t>(4 * max_tasks)), "dynamic state");
    ET_CUDA(rt->d_fired.upload(nullptr, static_cast<size_t>(2 * rt->cnt_capacity)), "dynamic state");
    ET_CUDA(rt->d_disp.upload(nullptr, static_cast<size_t>(2 * rt->cnt_capacity)), "dynamic state");
    ET_CUDA(rt->d_push_time.upload(nullptr, static_cast<size_t>(max_tasks)), "dynamic state");
    ET_CUDA(rt->d_trace.upload(nullptr, static_cast<size_t>(max_tasks)), "trace");
    rt->prepared[0] = rt->prepared[1] = -1;
    return ET_OK;
}

namespace {
// A GEMV task accumulates nseg x rows x b fp32 values in shared memory (kAccFloats);
// bound the rows of the widest task from the span arithmetic of ops.cuh gemv_span.
bool gemv_acc_fits(const et_op& op, int64_t grid0, const int64_t* binding) {
    if (op.kind == ET_OP_GEMV_TC) {  // TMEM columns, operand shapes and piece buffers
        const bool tiled = etk::tc_tiled(op);  // f4 GEMM tiles: i12 tasks per token block, batch i10
        const int64_t nb = tiled ? op.i[10] : op.i[5] >= 0 ? binding[op.i[5]] : 1;
        const int npad = etk::tc_npad(static_cast<int>(nb));
        const int kp = op.i[6], splits = op.i[3] > 0 ? op.i[3] : 1;
        const int64_t tasks = tiled ? op.i[12] : grid0;
        if (nb > etk::kMaxBatchTc || kp <= 0 || kp % 64 || op.i[1] % kp || op.i[0] % 128) return false;
        if (static_cast<int64_t>(npad) * kp * 2 > etk::kTcXBuf || tasks % splits) return false;
        if (splits > 1 && op.i[4] != etk::EPI_ADD && !(tiled && op.i[4] == etk::EPI_F32 && op.i[11] > 0)) return false;
        if (tiled && (nb % 16 || op.i[4] != etk::EPI_F32)) return false;
        const int64_t G = tasks / splits, nblk = op.i[0] / 128;
        return op.i[2] * ((nblk + G - 1) / G) * npad <= etk::kTmemCols;
    }
    if (op.kind != ET_OP_GEMV) return true;
    const bool grouped = (op.flags & 16) != 0;
    const int64_t T = grouped ? op.i[13] : grid0;
    if (T <= 0) return true;
    const int64_t nb = op.i[5] >= 0 ? binding[op.i[5]] : 1;
    const int64_t kst = op.i[1] / 16;
    int64_t rows;
    if (op.i[13] && !grouped) {  // split-K: an even span of k-step pairs may straddle row tiles
        const int64_t pairs = static_cast<int64_t>(op.i[0] / 16) * kst / 2;
        rows = ((2 * ((pairs + T - 1) / T) + kst - 1) / kst + 1) * 16;
    } else {
        const int64_t align = op.i[7] > 16 ? op.i[7] : 16;
        rows = ((op.i[0] / align + T - 1) / T) * align;
    }
    return op.i[2] * rows * nb <= etk::kAccFloats;
}
}  // namespace

int et_bind_ops(et_runtime* rt, const et_op* ops, int32_t num_calls) {
    if (!rt || (!ops && num_calls > 0)) return ET_ERR_INVALID;
    // A rejected table leaves the runtime unbound (et_step refuses to launch) rather
    // than running whatever table was bound before.
    rt->ops_bound = 0;
    if (num_calls != rt->num_calls) return rt->fail(ET_ERR_INVALID, "op table must have one entry per call");
    // validate everything before touching the device copy
    int variant = 0;
    for (int32_t c = 0; c < num_calls; ++c) {
        const int k = ops[c].kind;
        if (k == ET_OP_MOE_GROUP || k == ET_OP_MOE_COMBINE || k < ET_OP_NONE || k > ET_OP_KIND_LAST)
            return rt->fail(ET_ERR_INVALID, "call " + std::to_string(c) + ": op kind " + std::to_string(k) +
                                                " has no device body (the routed notify / red.add epilogues "
                                                "replace MOE_GROUP and MOE_COMBINE)");
        if (k == ET_OP_MOE_ROUTE || k == ET_OP_MOE_EXPERT) variant |= 1;
        // attention groups wider than 512 (head, dim) outputs (e.g. Llama-3-70B: 8 q heads per kv
        // head) need the wide split / merge bodies, compiled into the kMoE instantiations
        if ((k == ET_OP_ATTN_SPLIT || k == ET_OP_ATTN_MERGE) && ops[c].i[0] * ops[c].i[1] > 2 * etk::kConsumers)
            variant |= 1;
        else if (k == ET_OP_GEMV_TC || k == ET_OP_NORM) variant |= 2;
        if (k == ET_OP_COPY && (rt->mode != ET_MODE_STATIC || ops[c].i[0] <= 0 || ops[c].i[0] % 16))
            return rt->fail(ET_ERR_INVALID, "call " + std::to_string(c) + ": copies run on the static scheduler's "
                                            "DMA queue, in 16-byte multiples");
        if (k == ET_OP_REDUCE && (ops[c].i[4] % 4 || ops[c].i[0] % 4 || ops[c].i[2] < 1))
            return rt->fail(ET_ERR_INVALID, "call " + std::to_string(c) + ": reduce tiles need rows % 4 == 0");
    }
    for (int32_t c = 0; c < num_calls; ++c) {
        const et_op& o = ops[c];
        if (o.kind == ET_OP_GEMV && o.i[3] == 2) {  // attention-merge prologue (megakernel.cu body_gemv)
            if (o.i[5] >= 0 || o.i[8] <= 0 || o.i[1] % o.i[8] || o.i[11] <= 0 || o.i[12] <= 0 || o.i[1] > 4 * etk::kConsumers ||
                3LL * (o.i[1] / o.i[8]) * o.i[12] > etk::kAccFloats || !o.p[2] || (o.p[5] && (o.i[9] <= 0 || o.i[13] <= 0)))
                return rt->fail(ET_ERR_INVALID, "call " + std::to_string(c) + ": GEMV x mode 2 (attention merge) "
                                "needs b = 1, K a multiple of head_dim up to 1024, and 3 * heads * split cap <= " +
                                std::to_string(etk::kAccFloats));
        }
        if (o.kind == ET_OP_MOE_EXPERT) {
            // body_moe_expert keeps gate / up accumulators for up to 8 tokens [2][IR][8] fp32, the
            // activations [8][IR] bf16 and 16 words of tile state in the accumulator area
            const int rs = o.i[2], ir = rs > 0 ? o.i[0] / rs : 0;
            if (rs <= 0 || o.i[0] % rs || ir % 32 || 2LL * ir * 8 + ir * 4 + 16 > etk::kAccFloats)
                return rt->fail(ET_ERR_INVALID, "call " + std::to_string(c) + ": MoE expert row splits need "
                                "(expert_inter / row_splits) a multiple of 32 with 20 * rows + 16 <= " +
                                std::to_string(etk::kAccFloats) + " (at most 96 rows)");
        }
        if (o.kind == ET_OP_ATTN_SPLIT && (o.flags & 1024) && (variant & 2))
            return rt->fail(ET_ERR_INVALID, "call " + std::to_string(c) + ": attention flags bit 10 (new token "
                            "folded by the last split) is implemented by the mma.sync instantiations only");
    }
    for (int32_t c = 0; c < num_calls; ++c) {
        if (ops[c].kind != ET_OP_ATTN_SPLIT && ops[c].kind != ET_OP_ATTN_MERGE) continue;
        const int dh = ops[c].i[0], G = ops[c].i[1], CH = ops[c].i[2];
        if (dh > etk::kConsumers)  // the split prologue loads one dimension per consumer thread
            return rt->fail(ET_ERR_INVALID, "attention head_dim must not exceed 256");
        if (G * dh > 4 * etk::kConsumers)  // the wide bodies hold 4 (head, dim) outputs per thread
            return rt->fail(ET_ERR_INVALID, "attention groups need q heads per kv head x head_dim <= 1024");
        if ((ops[c].flags & 256) && dh % 64 != 0)  // chunk j ^ (pos % 8) must stay inside the row
            return rt->fail(ET_ERR_INVALID, "chunk-swizzled KV rows (attention flags bit 8) need head_dim % 64 == 0");
        if ((variant & 2) && ops[c].kind == ET_OP_ATTN_SPLIT && (G > 8 || dh % 16 != 0 || dh > 128 || CH != 64))
            // the tensor-core instantiation runs attention on mma.sync tiles (attn_split_mma)
            return rt->fail(ET_ERR_INVALID, "tensor-core attention needs <= 8 q heads per kv head, head_dim "
                                            "a multiple of 16 up to 128 and 64-position blocks");
    }
    cudaSetDevice(rt->cfg.device);
    cudaStreamSynchronize(rt->stream);
    ET_CUDA(rt->d_ops.upload(ops, static_cast<size_t>(std::max(1, num_calls))), "bind ops");
    rt->has_moe = variant;
    rt->h_ops.assign(ops, ops + num_calls);
    rt->ops_bound = 1;
    rt->memo_pick = -1;
    return ET_OK;
}

int et_set_runtime_tensor(et_runtime* rt, int32_t index, const int32_t* values, int64_t n) {
    if (!rt || index < 0 || index >= static_cast<int>(rt->d_rt.size())) return ET_ERR_INVALID;
    if (n > rt->rt_capacity[static_cast<size_t>(index)])
        return rt->fail(ET_ERR_INVALID, "runtime tensor larger than its capacity");
    cudaSetDevice(rt->cfg.device);
    ET_CUDA(cudaMemcpyAsync(rt->d_rt[static_cast<size_t>(index)].ptr, values, static_cast<size_t>(n) * 4,
                            cudaMemcpyHostToDevice, rt->stream),
            "runtime tensor");
    ET_CUDA(cudaStreamSynchronize(rt->stream), "runtime tensor");
    return ET_OK;
}

int et_clear_runtime_tensors(et_runtime* rt) {
    if (!rt) return ET_ERR_INVALID;
    cudaSetDevice(rt->cfg.device);
    for (auto& d : rt->d_rt)
        if (d.ptr) ET_CUDA(cudaMemsetAsync(d.ptr, 0, d.n * 4, rt->stream), "runtime tensor");
    return ET_OK;
}

int et_get_runtime_tensor(et_runtime* rt, int32_t index, int32_t* values, int64_t n) {
    if (!rt || index < 0 || index >= static_cast<int>(rt->d_rt.size())) return ET_ERR_INVALID;
    cudaSetDevice(rt->cfg.device);
    const int64_t m = std::min<int64_t>(n, static_cast<int64_t>(rt->d_rt[static_cast<size_t>(index)].n));
    ET_CUDA(cudaStreamSynchronize(rt->stream), "runtime tensor");
    ET_CUDA(cudaMemcpy(values, rt->d_rt[static_cast<size_t>(index)].ptr, static_cast<size_t>(m) * 4, cudaMemcpyDeviceToHost),
            "runtime tensor");
    return ET_OK;
}

// After a failed step the op-side state that the kernels normally leave clean for
// the next step (split-arrival counters of the fused attention merge and the MoE
// route, raw split-K q/k/v and router accumulators zeroed by their consumers) may
// be half-updated: zero it, sized by the runtime's max_batch.
static void reset_op_state(et_runtime* rt) {
    const size_t B = static_cast<size_t>(std::max(1, rt->cfg.max_batch));
    for (const et_op& op : rt->h_ops) {
        if (op.kind == ET_OP_ATTN_SPLIT && (op.flags & 2) && op.p[5])
            cudaMemset(reinterpret_cast<void*>(op.p[5]), 0, B * static_cast<size_t>(std::max(1, op.i[6])) * 4);
        if (op.kind == ET_OP_ATTN_SPLIT && (op.flags & 32) && op.p[0] && op.i[7] > 0)
            cudaMemset(reinterpret_cast<void*>(op.p[0]), 0, B * static_cast<size_t>(op.i[7]) * 4);
        if (op.kind == ET_OP_MOE_ROUTE) {
            if (op.p[7]) cudaMemset(reinterpret_cast<void*>(op.p[7]), 0, 4);
            if ((op.flags & 2) && op.p[1]) cudaMemset(reinterpret_cast<void*>(op.p[1]), 0, B * static_cast<size_t>(op.i[0]) * 4);
        }
    }
}

static int collect(et_runtime* rt, et_step_info* info) {
    ET_CUDA(cudaStreamSynchronize(rt->stream), "step");
    etk::DevStatus st{}, prev{};
    const int cur = rt->parity ^ 1;  // parity already advanced past the last launch
    ET_CUDA(cudaMemcpy(&st, rt->d_status.ptr + cur, sizeof(st), cudaMemcpyDeviceToHost), "status");
    // An earlier asynchronous step's error is sticky: a launch never zeroes a status
    // block that holds an error (megakernel.cu), and launches that find their own
    // block failed exit at once, so the first error survives until it is collected here.
    ET_CUDA(cudaMemcpy(&prev, rt->d_status.ptr + (cur ^ 1), sizeof(prev), cudaMemcpyDeviceToHost), "status");
    if (st.code == 0 && prev.code != 0) st = prev;
    if (info) {
        std::memset(info, 0, sizeof(*info));
        info->status = st.code;
        info->sample_index = rt->last_sample;
        info->worker = st.worker;
        info->slot = st.slot;
        info->counter = st.counter;
        info->value = st.value;
        info->tasks_executed = static_cast<int64_t>(st.executed);
        info->noop_tasks = static_cast<int64_t>(st.noops);
        info->pushes = static_cast<int64_t>(st.pushes);
        info->pops = static_cast<int64_t>(st.pops);
        float ms = 0.f;
        if (rt->timed) {
            if (cudaEventElapsedTime(&ms, rt->ev0, rt->ev1) == cudaSuccess) info->kernel_ms = ms;
            else (void)cudaGetLastError();  // never leave a stale error for the next launch check
        }
        info->step_id = rt->steps;
    }
    if (st.code != 0) {
        // leave the runtime reusable: clear every counter and status block
        cudaMemset(rt->d_cnt.ptr, 0, rt->d_cnt.n * sizeof(uint32_t));
        cudaMemset(rt->d_status.ptr, 0, 2 * sizeof(etk::DevStatus));
        reset_op_state(rt);
        cudaDeviceSynchronize();
        rt->prepared[0] = rt->prepared[1] = -1;
        rt->err = st.code == ET_ERR_DEADLOCK     ? "deadlock"
                  : st.code == ET_ERR_UNDERFLOW  ? "counter underflow"
                  : st.code == ET_ERR_STEP_LIMIT ? "step limit exceeded"
                                                 : "invalid tile operation (a GEMV's activations exceed shared "
                                                   "memory: batch * K * 2 > 32 KB, or batch > 8)";
        return st.code;
    }
    return ET_OK;
}

int et_step(et_runtime* rt, const int64_t* binding, int32_t num_symbols, void* stream, int32_t synchronous,
            et_step_info* info) {
    if (!rt) return ET_ERR_INVALID;
    if (num_symbols != rt->num_symbols) return rt->fail(ET_ERR_INVALID, "binding has the wrong number of symbols");
    if (rt->samples.empty()) return rt->fail(ET_ERR_INVALID, "no program uploaded");
    if (!rt->ops_bound) return rt->fail(ET_ERR_INVALID, "ops not bound");
    cudaSetDevice(rt->cfg.device);
    const bool memo = rt->memo_pick >= 0 && rt->memo_binding.size() == static_cast<size_t>(num_symbols) &&
                      std::equal(rt->memo_binding.begin(), rt->memo_binding.end(), binding);
    int pick = memo ? rt->memo_pick : -1;
    if (!memo) {
        // next-larger covering sample (samples are uploaded in selection order)
        // actual grid extents at this binding
        std::vector<int64_t> ext(static_cast<size_t>(rt->num_calls) * 4, 0);
        for (int c = 0; c < rt->num_calls; ++c)
            for (int d = 0; d < rt->call_rank[static_cast<size_t>(c)]; ++d) {
                bool ok = true;
                const int64_t a = eval_host(rt->code_op, rt->code_arg, rt->grid_code_off[static_cast<size_t>(c * 4 + d)],
                                            rt->grid_code_off[static_cast<size_t>(c * 4 + d + 1)], binding, &ok);
                if (!ok) return rt->fail(ET_ERR_INVALID, "grid of call " + std::to_string(c) + " is invalid at the binding");
                ext[static_cast<size_t>(c * 4 + d)] = a;
                if (d == 0 && !gemv_acc_fits(rt->h_ops[static_cast<size_t>(c)], a, binding))
                    return rt->fail(ET_ERR_INVALID, "GEMV call " + std::to_string(c) +
                                                        ": rows per task x batch exceed the accumulators (shared memory / "
                                                        "tensor memory) or the operand shape is invalid");
            }
        // next-larger sample covering the binding (ref sched_static.cpp:111-175) whose grids
        // also cover the actual ones (ref sched_static.cpp:153-156); a grid that is not
        // monotone in the symbols (e.g. splits shrinking with the batch) falls through to
        // the next covering sample instead of failing
        int first = -1;
        for (size_t i = 0; i < rt->samples.size() && pick < 0; ++i) {
            bool covers = true;
            for (int k = 0; k < num_symbols; ++k) covers &= rt->samples[i].binding[static_cast<size_t>(k)] >= binding[k];
            if (!covers) continue;
            if (first < 0) first = static_cast<int>(i);
            bool grids = true;
            for (int c = 0; c < rt->num_calls && grids; ++c)
                for (int d = 0; d < rt->call_rank[static_cast<size_t>(c)]; ++d)
                    grids &= ext[static_cast<size_t>(c * 4 + d)] <= rt->samples[i].call_extents[static_cast<size_t>(c * 4 + d)];
            if (grids) pick = static_cast<int>(i);
        }
        if (first < 0) return rt->fail(ET_ERR_INVALID, "binding exceeds every sampled shape");
        if (pick < 0) return rt->fail(ET_ERR_INVALID, "sampled shape does not cover the actual grid of a call");
    }
    const Sample& S = rt->samples[static_cast<size_t>(pick)];

    etk::StaticParams p{};
    p.num_symbols = rt->num_symbols;
    p.num_calls = rt->num_calls;
    p.call_rank = rt->d_call_rank.ptr;
    p.call_extent_from = rt->d_call_extent_from.ptr;
    p.grid_code_off = rt->d_grid_code_off.ptr;
    p.code_op = rt->d_code_op.ptr;
    p.code_arg = reinterpret_cast<const long long*>(rt->d_code_arg.ptr);
    p.call_extents = S.d_call_extents.ptr;
    p.num_queues = S.num_queues;
    p.has_dma = S.has_dma;
    p.queue_off = S.d_queue_off.ptr;
    p.num_slots = S.num_slots;
    p.slot_call = S.d_slot_call.ptr;
    p.slot_flat = S.d_slot_flat.ptr;
    p.slot_duration = S.d_slot_duration.ptr;
    p.wait_off = S.d_wait_off.ptr;
    p.waits = S.d_waits.ptr;
    p.notify_off = S.d_notify_off.ptr;
    p.notifies = S.d_notifies.ptr;
    p.num_counters = S.num_counters;
    p.initial_counts = S.d_initial.ptr;
    p.cnt = rt->d_cnt.ptr + static_cast<size_t>(rt->parity) * static_cast<size_t>(rt->cnt_capacity);
    p.cnt_other = rt->d_cnt.ptr + static_cast<size_t>(rt->parity ^ 1) * static_cast<size_t>(rt->cnt_capacity);
    p.cnt_capacity = rt->cnt_capacity;
    p.rt = rt->d_rt_table.ptr;
    p.num_rt = static_cast<int>(rt->d_rt.size());
    if (memo) {
        for (int i = 0; i < p.num_rt; ++i) p.rt_len[i] = rt->memo_rt_len[static_cast<size_t>(i)];
    } else {
        for (int i = 0; i < p.num_rt; ++i) {
            bool ok = true;
            p.rt_len[i] = (int)eval_host(rt->code_op, rt->code_arg, rt->rt_len_off[static_cast<size_t>(i)],
                                    rt->rt_len_off[static_cast<size_t>(i) + 1], binding, &ok);
            if (!ok || p.rt_len[i] > rt->rt_capacity[static_cast<size_t>(i)])
                return rt->fail(ET_ERR_INVALID, "runtime tensor shape invalid at the binding");
        }
        rt->memo_binding.assign(binding, binding + num_symbols);
        rt->memo_rt_len.assign(p.rt_len, p.rt_len + p.num_rt);
        rt->memo_pick = pick;
    }
    p.ops = rt->d_ops.ptr;
    p.trace = rt->d_trace.ptr;
    p.record = rt->cfg.record_trace;
    p.status = rt->d_status.ptr + rt->parity;
    p.status_other = rt->d_status.ptr + (rt->parity ^ 1);
    for (int k = 0; k < num_symbols; ++k) p.binding[k] = binding[k];
    p.watchdog_ns = rt->cfg.watchdog_ns;
    p.tick_ns = rt->cfg.tick_ns;
    p.step_limit = rt->cfg.step_limit > 0 ? rt->cfg.step_limit : 0;
    p.prefetch = rt->cfg.enable_prefetch;
    p.table_ok = S.table_ok;
    p.step_id = ++rt->steps;
    p.l2_ahead = rt->cfg.l2_prefetch_bytes < 0 ? 0 : rt->cfg.l2_prefetch_bytes;
    p.debug = rt->debug;

    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : rt->stream;
    int e = 0;
    etk::DynParams dp{};
    if (rt->mode == ET_MODE_DYNAMIC) {
        dp = S.dyn;
        const int cur = rt->parity, oth = rt->parity ^ 1;
        const size_t mt = static_cast<size_t>(rt->max_tasks), cc = static_cast<size_t>(rt->cnt_capacity);
        dp.ctl = rt->d_ctl.ptr + cur;
        dp.ctl_other = rt->d_ctl.ptr + oth;
        dp.rem = rt->d_rem.ptr + cur * mt;
        dp.rem_other = rt->d_rem.ptr + oth * mt;
        dp.slots = rt->d_slots.ptr + cur * 2 * mt;
        dp.slots_other = rt->d_slots.ptr + oth * 2 * mt;
        dp.fired = rt->d_fired.ptr + cur * cc;
        dp.fired_other = rt->d_fired.ptr + oth * cc;
        dp.disp = rt->d_disp.ptr + cur * cc;
        dp.disp_other = rt->d_disp.ptr + oth * cc;
        dp.push_time = rt->d_push_time.ptr;
        if (rt->prepared[cur] != pick) {
            e = et_dynamic_reset(p, dp, st);
            if (e != 0) return rt->cuda_fail(static_cast<cudaError_t>(e), "dynamic reset");
        }
        rt->prepared[oth] = pick;  // the launch rebuilds the other parity for this sample
        rt->prepared[cur] = -1;
    }
    rt->timed = synchronous;
    if (synchronous) cudaEventRecord(rt->ev0, st);
    if (rt->mode == ET_MODE_DYNAMIC)
        e = et_launch_dynamic(p, dp, S.num_queues, rt->has_moe, st);
    else
        e = et_launch_static(p, S.num_queues, rt->cfg.max_batch, rt->has_moe, st);
    if (e != 0) return rt->cuda_fail(static_cast<cudaError_t>(e), "launch");
    if (synchronous) cudaEventRecord(rt->ev1, st);
    rt->parity ^= 1;
    rt->last_sample = pick;
    rt->launched = true;
    if (!synchronous) return ET_OK;
    if (st != rt->stream) ET_CUDA(cudaStreamSynchronize(st), "step");
    return collect(rt, info);
}

int et_sync(et_runtime* rt, et_step_info* info) {
    if (!rt) return ET_ERR_INVALID;
    cudaSetDevice(rt->cfg.device);
    ET_CUDA(cudaDeviceSynchronize(), "sync");
    return collect(rt, info);
}

int et_set_debug(et_runtime* rt, int32_t bits) {
    if (!rt) return ET_ERR_INVALID;
    rt->debug = bits;
    return ET_OK;
}

int et_set_l2_prefetch(et_runtime* rt, int64_t bytes) {
    if (!rt) return ET_ERR_INVALID;
    rt->cfg.l2_prefetch_bytes = bytes;
    return ET_OK;
}

int et_read_counters(et_runtime* rt, int64_t* out, int64_t n) {
    if (!rt || rt->last_sample < 0) return ET_ERR_INVALID;
    cudaSetDevice(rt->cfg.device);
    const Sample& S = rt->samples[static_cast<size_t>(rt->last_sample)];
    std::vector<uint32_t> got(static_cast<size_t>(S.num_counters));
    const int cur = rt->parity ^ 1;
    ET_CUDA(cudaStreamSynchronize(rt->stream), "counters");
    if (S.num_counters > 0)
        ET_CUDA(cudaMemcpy(got.data(), rt->d_cnt.ptr + static_cast<size_t>(cur) * static_cast<size_t>(rt->cnt_capacity),
                           got.size() * 4, cudaMemcpyDeviceToHost),
                "counters");
    for (int64_t i = 0; i < std::min<int64_t>(n, S.num_counters); ++i)
        out[i] = static_cast<int64_t>(S.initial_counts[static_cast<size_t>(i)]) - static_cast<int64_t>(got[static_cast<size_t>(i)]);
    return ET_OK;
}

int et_read_trace(et_runtime* rt, et_trace_rec* out, int64_t* n) {
    if (!rt || !n || rt->last_sample < 0) return ET_ERR_INVALID;
    cudaSetDevice(rt->cfg.device);
    const Sample& S = rt->samples[static_cast<size_t>(rt->last_sample)];
    const int64_t total = rt->mode == ET_MODE_DYNAMIC ? S.num_tasks : S.num_slots;
    const int64_t m = std::min<int64_t>(*n, total);
    ET_CUDA(cudaStreamSynchronize(rt->stream), "trace");
    if (m > 0) ET_CUDA(cudaMemcpy(out, rt->d_trace.ptr, static_cast<size_t>(m) * sizeof(et_trace_rec), cudaMemcpyDeviceToHost), "trace");
    *n = total;
    return ET_OK;
}

}  // extern "C"

int et_ipc_get_handle(const void* dev_ptr, void* handle) {
    if (!dev_ptr || !handle) return ET_ERR_INVALID;
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)) != cudaSuccess) return ET_ERR_CUDA;
    std::memcpy(handle, &h, sizeof(h));
    return ET_OK;
}

int et_ipc_open_handle(const void* handle, int32_t device, void** dev_ptr) {
    if (!handle || !dev_ptr) return ET_ERR_INVALID;
    cudaSetDevice(device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    if (cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return ET_ERR_CUDA;
    return ET_OK;
}

int et_ipc_close_handle(void* dev_ptr) {
    return cudaIpcCloseMemHandle(dev_ptr) == cudaSuccess ? ET_OK : ET_ERR_CUDA;
}
