// Host side of GPU execution: flattening of lowered kernels into the C-ABI
// program arrays, the Executor, and the reference-named simulate() entry
// points (ref simulate.hpp:23-36), which here run on the device.
#include <chrono>
#include <cstdio>
#include <cstring>

#include "etsim/exec.hpp"
#include "etsim/json_io.hpp"

namespace etsim {

void raise_status(int code, const std::string& what) {
    switch (code) {
        case ET_OK: return;
        case ET_ERR_DEADLOCK: throw SimError(SimError::Kind::Deadlock, "deadlock: " + what, {what});
        case ET_ERR_UNDERFLOW: throw SimError(SimError::Kind::CounterUnderflow, "counter underflow: " + what);
        case ET_ERR_STEP_LIMIT: throw SimError(SimError::Kind::StepLimit, "step limit exceeded: " + what);
        case ET_ERR_NO_DEVICE: throw Error("no CUDA device: the executor has no CPU fallback");
        default: throw Error(what);
    }
}

bool gpu_available() {
    int n = 0;
    return et_device_count(&n) == ET_OK && n > 0;
}

namespace {

ExprPtr product_expr(const std::vector<ExprPtr>& dims) {
    ExprPtr p = SymExpr::constant(1);
    for (const auto& d : dims) p = p * d;
    return p;
}

std::vector<int64_t> binding_vector(const GraphFunction& g, const ShapeBinding& b) {
    std::vector<int64_t> v;
    for (const auto& s : g.symbols) {
        auto it = b.find(s);
        if (it == b.end()) throw Error("binding " + binding_to_string(b) + " does not bind symbol '" + s + "'");
        v.push_back(it->second);
    }
    return v;
}

struct HostSample {
    std::vector<int64_t> binding;
    std::vector<int32_t> call_extents, queue_off, slot_task, slot_call, slot_flat, slot_duration, wait_off, waits,
        notify_off, notifies, initial_counts;
    std::vector<int32_t> slot_queue;  // for trace reconstruction
    int num_queues = 0, has_dma = 0;
    // dynamic mode: data-dependent tensors (their initial counts live on the device)
    std::vector<int32_t> dd_base, dd_count, dd_counts_rt;
};

}  // namespace

struct Executor::Impl {
    StaticMegakernel k;  // dynamic mode: graph + num_sms only
    bool dyn = false;
    DynamicMegakernel dk;
    std::vector<ShapeBinding> dyn_samples;
    int last_step_id = 0;
    ExecConfig cfg;
    et_runtime* rt = nullptr;
    std::vector<HostSample> hs;
    std::vector<std::string> rt_names;
    int workers = 0;
    double upload_ms = 0;
    ShapeBinding last_binding;
    int last_sample = -1;

    ~Impl() {
        if (rt) et_destroy(rt);
    }
    void check(int code, const char* what) const {
        if (code != ET_OK) raise_status(code, std::string(what) + ": " + et_last_error(rt));
    }
};

namespace {

// Shape-independent graph description (grid / runtime-tensor length code).
struct GraphArrays {
    std::vector<int32_t> call_rank, call_ef, grid_off, code_op, rt_len_off;
    std::vector<int64_t> code_arg, rt_cap;
    et_graph_desc desc() {
        et_graph_desc gd{};
        gd.num_calls = static_cast<int32_t>(call_rank.size());
        gd.call_rank = call_rank.data();
        gd.call_extent_from = call_ef.data();
        gd.grid_code_off = grid_off.data();
        gd.code_op = code_op.data();
        gd.code_arg = code_arg.data();
        gd.code_len = static_cast<int32_t>(code_op.size());
        gd.num_runtime_tensors = static_cast<int32_t>(rt_cap.size());
        gd.runtime_capacity = rt_cap.data();
        gd.runtime_len_off = rt_len_off.data();
        return gd;
    }
};

GraphArrays graph_arrays(const GraphFunction& g, const std::vector<ShapeBinding>& samples) {
    GraphArrays a;
    auto append = [&](const ExprPtr& e) {
        const ExprCode c = compile_expr(e, g.symbols);
        for (const auto& ins : c.code) {
            a.code_op.push_back(static_cast<int32_t>(ins.op));
            a.code_arg.push_back(ins.arg);
        }
    };
    for (const auto& c : g.calls) {
        const auto& grid = g.call_grid(c);
        if (grid.size() > 4) throw Error("grid rank above 4 is not supported on the device");
        a.call_rank.push_back(static_cast<int32_t>(grid.size()));
        a.call_ef.push_back(c.extent_from.empty() ? -1 : g.runtime_index(c.extent_from));
        for (size_t d = 0; d < 4; ++d) {
            a.grid_off.push_back(static_cast<int32_t>(a.code_op.size()));
            if (d < grid.size()) append(grid[d]);
        }
    }
    a.grid_off.push_back(static_cast<int32_t>(a.code_op.size()));
    for (const auto& r : g.runtime_tensors) {
        a.rt_len_off.push_back(static_cast<int32_t>(a.code_op.size()));
        append(product_expr(r.shape));
        Int cap = 1;
        for (const auto& b : samples) cap = std::max(cap, eval_expr(product_expr(r.shape), b));
        a.rt_cap.push_back(cap);
    }
    a.rt_len_off.push_back(static_cast<int32_t>(a.code_op.size()));
    return a;
}

std::vector<int32_t> sample_extents(const GraphFunction& g, const ShapeBinding& b) {
    std::vector<int32_t> ext;
    for (const auto& c : g.calls) {
        const auto& grid = g.call_grid(c);
        for (size_t d = 0; d < 4; ++d) {
            const Int e = d < grid.size() ? eval_expr(grid[d], b) : 1;
            if (e > INT32_MAX) throw Error("grid extent exceeds int32");
            ext.push_back(static_cast<int32_t>(e));
        }
    }
    return ext;
}

// Device program of the dynamic scheduler at one sampled binding.  Static-map
// edges are resolved here (instantiate() of the graph with its data-dependent
// edges removed); routed notifies and range triggers become per-call
// descriptors resolved on the device from the runtime tensors.
struct DynProgram {
    std::vector<int32_t> task_call, task_flat, task_duration, wait_off, waits, notify_off, notifies, rem_init,
        consumer_off, consumers, call_first, routed_rt, routed_base, range_rt, range_base, el_dd, ready, dd_base,
        dd_count, dd_counts_rt, dd_writer_call, initial_counts, task_class, task_waits_total, task_notifies_total;
    std::vector<uint8_t> armed, range_armed;
    // static-descriptor view (slots = tasks; DMA-class tasks in the DMA queue)
    std::vector<int32_t> queue_off, slot_task, slot_call, slot_flat, swait_off, snotify_off;
    std::vector<int32_t> call_extents;
    std::vector<int64_t> binding;
    int num_queues = 0, has_dma = 0;
};

DynProgram build_dynamic(const DynamicMegakernel& dk, const ShapeBinding& b, int workers, const ExecConfig& cfg) {
    const GraphFunction& g = dk.graph;
    GraphFunction gs = g;
    const size_t nc = g.calls.size();
    std::vector<std::vector<size_t>> static_in(nc);
    DynProgram P;
    P.routed_rt.assign(nc, -1);
    P.routed_base.assign(nc, -1);
    P.range_rt.assign(nc, -1);
    P.range_base.assign(nc, -1);
    P.range_armed.assign(nc, 0);
    std::vector<int> routed_ev(nc, -1), range_ev(nc, -1);
    for (size_t ci = 0; ci < nc; ++ci) {
        const CallDevice& c = g.calls[ci];
        CallDevice& cs = gs.calls[ci];
        cs.in_edges.clear();
        cs.out_edges.clear();
        for (size_t e = 0; e < c.in_edges.size(); ++e) {
            const EdgeSpec& ed = c.in_edges[e];
            if (ed.kind == MapKind::StaticMap) {
                cs.in_edges.push_back(ed);
                static_in[ci].push_back(e);
            } else {
                if (range_ev[ci] >= 0) throw Error("device scheduler: at most one range trigger per call");
                range_ev[ci] = g.event_index(ed.event);
                P.range_rt[ci] = g.runtime_index(ed.indptr_tensor);
                const auto& w = dk.templates[ci].wait_edges;
                P.range_armed[ci] = e < w.size() ? w[e] : 1;
            }
        }
        for (const auto& ed : c.out_edges) {
            if (ed.kind == MapKind::StaticMap) {
                cs.out_edges.push_back(ed);
            } else {
                if (routed_ev[ci] >= 0) throw Error("device scheduler: at most one routed notify per call");
                routed_ev[ci] = g.event_index(ed.event);
                P.routed_rt[ci] = g.runtime_index(ed.routing_tensor);
            }
        }
    }
    std::vector<int> dd_of_tensor(g.event_tensors.size(), -1);
    int num_dd = 0;
    for (size_t ti = 0; ti < g.event_tensors.size(); ++ti) {
        auto& e = gs.event_tensors[ti];
        if (!e.data_dependent) continue;
        dd_of_tensor[ti] = num_dd++;  // same order as the dd_* arrays filled below
        e.data_dependent = false;
        e.counts_tensor.clear();
        e.writer.clear();
    }
    for (size_t ci = 0; ci < nc; ++ci) {
        if (routed_ev[ci] >= 0 && dd_of_tensor[static_cast<size_t>(routed_ev[ci])] < 0)
            throw Error("device scheduler: routed notifies must target a data-dependent event tensor");
        if (range_ev[ci] >= 0 && dd_of_tensor[static_cast<size_t>(range_ev[ci])] < 0)
            throw Error("device scheduler: range triggers must wait on a data-dependent event tensor");
    }
    MaterializedTaskGraph m = instantiate(gs, b, nullptr, cfg.seed);
    for (size_t ci = 0; ci < nc; ++ci) {
        if (routed_ev[ci] >= 0) P.routed_base[ci] = static_cast<int32_t>(m.tensor_offsets[static_cast<size_t>(routed_ev[ci])]);
        if (range_ev[ci] >= 0) P.range_base[ci] = static_cast<int32_t>(m.tensor_offsets[static_cast<size_t>(range_ev[ci])]);
    }
    const size_t nel = m.events.size();
    P.el_dd.assign(nel, -1);
    for (size_t ti = 0; ti < g.event_tensors.size(); ++ti) {
        if (dd_of_tensor[ti] < 0) continue;
        const auto& decl = g.event_tensors[ti];
        const Int base = m.tensor_offsets[ti];
        const Int cnt = (ti + 1 < m.tensor_offsets.size() ? m.tensor_offsets[ti + 1] : static_cast<Int>(nel)) - base;
        P.dd_base.push_back(static_cast<int32_t>(base));
        P.dd_count.push_back(static_cast<int32_t>(cnt));
        P.dd_counts_rt.push_back(g.runtime_index(decl.counts_tensor));
        int wc = -1;
        for (size_t ci = 0; ci < nc; ++ci)
            if (g.calls[ci].fn == decl.writer) wc = static_cast<int>(ci);
        if (wc < 0) throw Error("event tensor '" + decl.name + "' writer is never launched");
        P.dd_writer_call.push_back(wc);
        for (Int i = 0; i < cnt; ++i) P.el_dd[static_cast<size_t>(base + i)] = dd_of_tensor[ti];
    }
    for (const auto& e : m.events) P.initial_counts.push_back(static_cast<int32_t>(e.initial_count));
    for (size_t ci = 0; ci < nc; ++ci) P.call_first.push_back(m.call_first_task[ci]);
    P.wait_off.push_back(0);
    P.notify_off.push_back(0);
    for (const auto& t : m.tasks) {
        const auto& tmpl = dk.templates[static_cast<size_t>(t.call)].wait_edges;
        P.task_call.push_back(t.call);
        P.task_flat.push_back(static_cast<int32_t>(t.flat));
        P.task_duration.push_back(static_cast<int32_t>(t.duration));
        int rem = 0;
        const auto& ws = m.task_waits[static_cast<size_t>(t.id)];
        for (size_t k = 0; k < ws.size(); ++k) {
            const int el = ws[k];
            P.waits.push_back(el);
            const size_t orig = static_in[static_cast<size_t>(t.call)][k];
            P.armed.push_back(orig < tmpl.size() ? tmpl[orig] : 1);
            if (P.el_dd[static_cast<size_t>(el)] >= 0 || P.initial_counts[static_cast<size_t>(el)] > 0) ++rem;
        }
        if (range_ev[static_cast<size_t>(t.call)] >= 0) ++rem;
        P.rem_init.push_back(rem);
        P.wait_off.push_back(static_cast<int32_t>(P.waits.size()));
        for (int el : m.task_notifies[static_cast<size_t>(t.id)]) P.notifies.push_back(el);
        P.notify_off.push_back(static_cast<int32_t>(P.notifies.size()));
        P.task_waits_total.push_back(static_cast<int32_t>(ws.size() + (range_ev[static_cast<size_t>(t.call)] >= 0)));
        P.task_notifies_total.push_back(
            static_cast<int32_t>(m.task_notifies[static_cast<size_t>(t.id)].size() + (routed_ev[static_cast<size_t>(t.call)] >= 0)));
        if (rem == 0) P.ready.push_back(t.id);
        P.task_class.push_back(t.resource == Resource::DMA ? 1 : 0);
    }
    P.consumer_off.push_back(0);
    for (size_t el = 0; el < nel; ++el) {
        for (int c : m.event_consumers[el]) P.consumers.push_back(c);
        P.consumer_off.push_back(static_cast<int32_t>(P.consumers.size()));
    }
    // static-descriptor view
    P.binding = binding_vector(g, b);
    P.call_extents = sample_extents(g, b);
    P.num_queues = workers;
    for (size_t t = 0; t < m.tasks.size(); ++t) P.has_dma |= P.task_class[t];
    P.queue_off.assign(static_cast<size_t>(workers) + 1, 0);
    for (int cls = 0; cls < 2; ++cls)
        for (size_t t = 0; t < m.tasks.size(); ++t)
            if (P.task_class[t] == cls) {
                P.slot_task.push_back(static_cast<int32_t>(t));
                P.slot_call.push_back(P.task_call[t]);
                P.slot_flat.push_back(P.task_flat[t]);
            }
    const int32_t nsm = static_cast<int32_t>(m.tasks.size()) - static_cast<int32_t>(std::count(P.task_class.begin(), P.task_class.end(), 1));
    for (int q = 1; q <= workers; ++q) P.queue_off[static_cast<size_t>(q)] = nsm;  // all SM tasks "in queue 0"
    if (P.has_dma) P.queue_off.push_back(static_cast<int32_t>(m.tasks.size()));
    P.swait_off.assign(P.slot_task.size() + 1, 0);
    P.snotify_off.assign(P.slot_task.size() + 1, 0);
    return P;
}

}  // namespace

Executor::Executor(const DynamicMegakernel& dk, const std::vector<ShapeBinding>& samples_in, const ExecConfig& cfg)
    : impl_(new Impl) {
    Impl& I = *impl_;
    I.dyn = true;
    I.dk = dk;
    I.cfg = cfg;
    I.workers = cfg.num_workers > 0 ? cfg.num_workers : 4;
    I.k.graph = dk.graph;
    I.k.num_sms = I.workers;
    if (samples_in.empty()) throw Error("dynamic execution needs at least one sampled binding");
    const auto t0 = std::chrono::steady_clock::now();
    const GraphFunction& g = dk.graph;
    // selection order: ascending size symbol (ref sched_static.cpp:101-104)
    std::vector<ShapeBinding> samples = samples_in;
    std::stable_sort(samples.begin(), samples.end(), [&](const ShapeBinding& a, const ShapeBinding& b) {
        if (g.size_symbol.empty()) return false;
        return a.at(g.size_symbol) < b.at(g.size_symbol);
    });
    I.dyn_samples = samples;
    GraphArrays ga = graph_arrays(g, samples);
    std::vector<DynProgram> progs;
    for (const auto& b : samples) progs.push_back(build_dynamic(dk, b, I.workers, cfg));

    et_config ec{};
    ec.device = cfg.device;
    ec.num_workers = I.workers;
    ec.record_trace = cfg.record_trace ? 1 : 0;
    ec.enable_prefetch = cfg.enable_prefetch ? 1 : 0;
    ec.watchdog_ns = cfg.watchdog_ns;
    ec.tick_ns = cfg.tick_ns;
    ec.step_limit = cfg.step_limit;
    ec.max_batch = cfg.max_batch;
    ec.l2_prefetch_bytes = cfg.l2_prefetch_bytes;
    const int rc = et_create(&ec, &I.rt);
    if (rc != ET_OK) raise_status(rc, "cannot create the GPU runtime");
    et_graph_desc gd = ga.desc();
    gd.num_symbols = static_cast<int32_t>(g.symbols.size());
    I.check(et_upload_graph(I.rt, &gd), "upload graph");

    std::vector<et_sample_desc> sd(progs.size());
    std::vector<et_dynamic_desc> dd(progs.size());
    for (size_t i = 0; i < progs.size(); ++i) {
        DynProgram& P = progs[i];
        HostSample h;
        h.binding = P.binding;
        h.call_extents = P.call_extents;
        h.num_queues = P.num_queues;
        h.has_dma = P.has_dma;
        h.slot_task = P.task_call;  // trace view: per task
        h.slot_call = P.task_call;
        h.slot_flat = P.task_flat;
        h.wait_off.assign(P.task_waits_total.size() + 1, 0);
        h.notify_off.assign(P.task_notifies_total.size() + 1, 0);
        for (size_t t = 0; t < P.task_waits_total.size(); ++t) {
            h.wait_off[t + 1] = h.wait_off[t] + P.task_waits_total[t];
            h.notify_off[t + 1] = h.notify_off[t] + P.task_notifies_total[t];
        }
        h.initial_counts = P.initial_counts;
        h.slot_queue = P.task_class;
        h.dd_base = P.dd_base;
        h.dd_count = P.dd_count;
        h.dd_counts_rt = P.dd_counts_rt;
        I.hs.push_back(h);

        et_sample_desc& s = sd[i];
        s.binding = P.binding.data();
        s.call_extents = P.call_extents.data();
        s.num_queues = P.num_queues;
        s.has_dma = P.has_dma;
        s.queue_off = P.queue_off.data();
        s.num_slots = static_cast<int32_t>(P.slot_task.size());
        s.slot_task = P.slot_task.data();
        s.slot_call = P.slot_call.data();
        s.slot_flat = P.slot_flat.data();
        s.slot_duration = nullptr;
        s.wait_off = P.swait_off.data();
        s.waits = nullptr;
        s.notify_off = P.snotify_off.data();
        s.notifies = nullptr;
        s.num_counters = static_cast<int32_t>(P.initial_counts.size());
        s.initial_counts = P.initial_counts.data();
        s.counter_dd = nullptr;

        et_dynamic_desc& d = dd[i];
        d.num_tasks = static_cast<int32_t>(P.task_call.size());
        d.task_call = P.task_call.data();
        d.task_flat = P.task_flat.data();
        d.task_duration = cfg.tick_ns > 0 ? P.task_duration.data() : nullptr;
        d.task_wait_off = P.wait_off.data();
        d.task_waits = P.waits.data();
        d.task_wait_armed = P.armed.data();
        d.task_notify_off = P.notify_off.data();
        d.task_notifies = P.notifies.data();
        d.task_rem_init = P.rem_init.data();
        d.consumer_off = P.consumer_off.data();
        d.consumers = P.consumers.data();
        d.call_first_task = P.call_first.data();
        d.call_routed_rt = P.routed_rt.data();
        d.call_routed_base = P.routed_base.data();
        d.call_range_rt = P.range_rt.data();
        d.call_range_base = P.range_base.data();
        d.call_range_armed = P.range_armed.data();
        d.num_dd = static_cast<int32_t>(P.dd_base.size());
        d.dd_base = P.dd_base.data();
        d.dd_count = P.dd_count.data();
        d.dd_counts_rt = P.dd_counts_rt.data();
        d.dd_writer_call = P.dd_writer_call.data();
        d.el_dd = P.el_dd.data();
        d.num_ready = static_cast<int32_t>(P.ready.size());
        d.ready = P.ready.data();
        d.early_push = dk.early_push ? 1 : 0;
    }
    I.check(et_upload_dynamic(I.rt, sd.data(), dd.data(), static_cast<int32_t>(sd.size())), "upload dynamic program");
    std::vector<et_op> none(g.calls.size());
    std::memset(none.data(), 0, none.size() * sizeof(et_op));
    I.check(et_bind_ops(I.rt, none.data(), static_cast<int32_t>(none.size())), "bind ops");
    I.upload_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

Executor::Executor(const StaticMegakernel& k, const ExecConfig& cfg) : impl_(new Impl) {
    Impl& I = *impl_;
    I.k = k;
    I.cfg = cfg;
    I.workers = cfg.num_workers > 0 ? cfg.num_workers : k.num_sms;
    if (I.workers != k.num_sms)
        throw Error("kernel was compiled for " + std::to_string(k.num_sms) + " SMs, run asked for " +
                    std::to_string(I.workers));
    if (k.samples.empty()) throw Error("kernel has no sampled schedules");
    const auto t0 = std::chrono::steady_clock::now();
    const GraphFunction& g = k.graph;

    // ---- graph description --------------------------------------------------
    std::vector<int32_t> call_rank, call_ef, grid_off, code_op, rt_len_off;
    std::vector<int64_t> code_arg, rt_cap;
    auto append = [&](const ExprPtr& e) {
        const ExprCode c = compile_expr(e, g.symbols);
        for (const auto& ins : c.code) {
            code_op.push_back(static_cast<int32_t>(ins.op));
            code_arg.push_back(ins.arg);
        }
    };
    for (const auto& c : g.calls) {
        const auto& grid = g.call_grid(c);
        if (grid.size() > 4) throw Error("grid rank above 4 is not supported on the device");
        call_rank.push_back(static_cast<int32_t>(grid.size()));
        call_ef.push_back(c.extent_from.empty() ? -1 : g.runtime_index(c.extent_from));
        for (size_t d = 0; d < 4; ++d) {
            grid_off.push_back(static_cast<int32_t>(code_op.size()));
            if (d < grid.size()) append(grid[d]);
        }
    }
    grid_off.push_back(static_cast<int32_t>(code_op.size()));
    for (const auto& r : g.runtime_tensors) {
        I.rt_names.push_back(r.name);
        rt_len_off.push_back(static_cast<int32_t>(code_op.size()));
        append(product_expr(r.shape));
        Int cap = 1;
        for (const auto& s : k.samples) cap = std::max(cap, eval_expr(product_expr(r.shape), s.binding));
        rt_cap.push_back(cap);
    }
    rt_len_off.push_back(static_cast<int32_t>(code_op.size()));

    // ---- samples ---------------------------------------------------------------
    for (const auto& s : k.samples) {
        HostSample h;
        h.binding = binding_vector(g, s.binding);
        h.num_queues = static_cast<int>(s.sm_queues.size());
        h.has_dma = s.dma_queue.empty() ? 0 : 1;
        std::vector<std::vector<Int>> ext(g.calls.size());
        for (size_t ci = 0; ci < g.calls.size(); ++ci) {
            const auto& grid = g.call_grid(g.calls[ci]);
            for (size_t d = 0; d < 4; ++d) {
                const Int e = d < grid.size() ? eval_expr(grid[d], s.binding) : 1;
                if (e > INT32_MAX) throw Error("grid extent exceeds int32");
                if (d < grid.size()) ext[ci].push_back(e);
                h.call_extents.push_back(static_cast<int32_t>(e));
            }
        }
        auto add_queue = [&](const std::vector<QueueTask>& q, int qi) {
            for (const auto& t : q) {
                h.slot_task.push_back(t.id);
                h.slot_call.push_back(t.call);
                h.slot_flat.push_back(static_cast<int32_t>(t.flat));
                h.slot_queue.push_back(qi);
                h.wait_off.push_back(static_cast<int32_t>(h.waits.size()));
                h.waits.insert(h.waits.end(), t.waits.begin(), t.waits.end());
                h.notify_off.push_back(static_cast<int32_t>(h.notifies.size()));
                h.notifies.insert(h.notifies.end(), t.notifies.begin(), t.notifies.end());
                if (cfg.tick_ns > 0) {
                    const DeviceFunctionDecl* fn = g.find_fn(g.calls[static_cast<size_t>(t.call)].fn);
                    Int dur = 1;
                    if (fn && !fn->duration.empty())
                        dur = eval_duration(g.duration_models.at(fn->duration), cfg.seed, t.call, t.coord,
                                            ext[static_cast<size_t>(t.call)], nullptr);
                    h.slot_duration.push_back(static_cast<int32_t>(dur));
                }
            }
        };
        h.queue_off.push_back(0);
        for (size_t q = 0; q < s.sm_queues.size(); ++q) {
            add_queue(s.sm_queues[q], static_cast<int>(q));
            h.queue_off.push_back(static_cast<int32_t>(h.slot_task.size()));
        }
        if (h.has_dma) {
            add_queue(s.dma_queue, h.num_queues);
            h.queue_off.push_back(static_cast<int32_t>(h.slot_task.size()));
        }
        h.wait_off.push_back(static_cast<int32_t>(h.waits.size()));
        h.notify_off.push_back(static_cast<int32_t>(h.notifies.size()));
        for (Int c : s.initial_counts) h.initial_counts.push_back(static_cast<int32_t>(c));
        I.hs.push_back(std::move(h));
    }

    // ---- runtime ---------------------------------------------------------------
    et_config ec{};
    ec.device = cfg.device;
    ec.num_workers = I.workers;
    ec.record_trace = cfg.record_trace ? 1 : 0;
    ec.enable_prefetch = cfg.enable_prefetch ? 1 : 0;
    ec.watchdog_ns = cfg.watchdog_ns;
    ec.tick_ns = cfg.tick_ns;
    ec.step_limit = cfg.step_limit;
    ec.max_batch = cfg.max_batch;
    ec.l2_prefetch_bytes = cfg.l2_prefetch_bytes;
    const int rc = et_create(&ec, &I.rt);
    if (rc != ET_OK) raise_status(rc, "cannot create the GPU runtime");

    et_graph_desc gd{};
    gd.num_symbols = static_cast<int32_t>(g.symbols.size());
    gd.num_calls = static_cast<int32_t>(g.calls.size());
    gd.call_rank = call_rank.data();
    gd.call_extent_from = call_ef.data();
    gd.grid_code_off = grid_off.data();
    gd.code_op = code_op.data();
    gd.code_arg = code_arg.data();
    gd.code_len = static_cast<int32_t>(code_op.size());
    gd.num_runtime_tensors = static_cast<int32_t>(rt_cap.size());
    gd.runtime_capacity = rt_cap.data();
    gd.runtime_len_off = rt_len_off.data();
    I.check(et_upload_graph(I.rt, &gd), "upload graph");

    std::vector<et_sample_desc> sd(I.hs.size());
    for (size_t i = 0; i < I.hs.size(); ++i) {
        const HostSample& h = I.hs[i];
        et_sample_desc& d = sd[i];
        d.binding = h.binding.data();
        d.call_extents = h.call_extents.data();
        d.num_queues = h.num_queues;
        d.has_dma = h.has_dma;
        d.queue_off = h.queue_off.data();
        d.num_slots = static_cast<int32_t>(h.slot_task.size());
        d.slot_task = h.slot_task.data();
        d.slot_call = h.slot_call.data();
        d.slot_flat = h.slot_flat.data();
        d.slot_duration = h.slot_duration.empty() ? nullptr : h.slot_duration.data();
        d.wait_off = h.wait_off.data();
        d.waits = h.waits.data();
        d.notify_off = h.notify_off.data();
        d.notifies = h.notifies.data();
        d.num_counters = static_cast<int32_t>(h.initial_counts.size());
        d.initial_counts = h.initial_counts.data();
        d.counter_dd = nullptr;
    }
    I.check(et_upload_static(I.rt, sd.data(), static_cast<int32_t>(sd.size())), "upload program");
    std::vector<et_op> none(g.calls.size());
    std::memset(none.data(), 0, none.size() * sizeof(et_op));
    I.check(et_bind_ops(I.rt, none.data(), static_cast<int32_t>(none.size())), "bind ops");
    I.upload_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

Executor::~Executor() = default;
Executor::Executor() : impl_(new Impl) {}

void Executor::save_program(const std::string& path) const {
    const Impl& I = *impl_;
    if (I.dyn) throw Error("program images hold static schedules only");
    const std::string meta = graph_to_json(I.k.graph, -1);
    I.check(et_save_program(I.rt, path.c_str(), meta.data(), static_cast<int64_t>(meta.size())), "save program");
}

namespace {
// Reads back the flat arrays of a program image (format: runtime.cu et_save_program)
// into HostSamples (trace reconstruction and error messages need them host-side).
struct ImageReader {
    std::vector<uint8_t> buf;
    size_t pos = 0;
    int64_t i64() {
        int64_t v = 0;
        if (pos + 8 > buf.size()) throw Error("truncated program image");
        std::memcpy(&v, buf.data() + pos, 8);
        pos += 8;
        return v;
    }
    template <typename T>
    std::vector<T> arr() {
        const int64_t n = i64();
        std::vector<T> v(static_cast<size_t>(n > 0 ? n : 0));
        const size_t bytes = v.size() * sizeof(T);
        if (pos + bytes > buf.size()) throw Error("truncated program image");
        if (bytes) std::memcpy(v.data(), buf.data() + pos, bytes);
        pos += bytes;
        return v;
    }
};
}  // namespace

std::unique_ptr<Executor> Executor::load_program(const std::string& path, const ExecConfig& cfg) {
    const auto t0 = std::chrono::steady_clock::now();
    ImageReader r;
    {
        FILE* f = std::fopen(path.c_str(), "rb");
        if (!f) throw Error("cannot read " + path);
        uint8_t tmp[1 << 16];
        size_t n;
        while ((n = std::fread(tmp, 1, sizeof(tmp), f)) > 0) r.buf.insert(r.buf.end(), tmp, tmp + n);
        std::fclose(f);
    }
    r.pos = 8;  // magic (checked by et_load_program)
    r.i64();    // abi
    const int workers = static_cast<int>(r.i64());
    const auto meta = r.arr<char>();
    r.i64();
    r.i64();
    std::unique_ptr<Executor> ex(new Executor());
    Impl& I = *ex->impl_;
    I.cfg = cfg;
    I.workers = workers;
    I.k.graph = graph_from_json(std::string(meta.begin(), meta.end()));
    I.k.num_sms = workers;
    for (const auto& t : I.k.graph.runtime_tensors) I.rt_names.push_back(t.name);
    // graph section (the order of et_upload_graph): num_symbols; call_rank, call_extent_from,
    // grid_code_off, code_op (int32); code_arg, runtime_capacity (int64); runtime_len_off (int32)
    r.i64();
    for (int j = 0; j < 4; ++j) r.arr<int32_t>();
    r.arr<int64_t>();
    r.arr<int64_t>();
    r.arr<int32_t>();
    const int64_t ns = r.i64();
    for (int64_t i = 0; i < ns; ++i) {
        HostSample h;
        h.num_queues = static_cast<int>(r.i64());
        h.has_dma = static_cast<int>(r.i64());
        r.i64();  // slots
        r.i64();  // counters
        h.binding = r.arr<int64_t>();
        h.call_extents = r.arr<int32_t>();
        h.queue_off = r.arr<int32_t>();
        h.slot_task = r.arr<int32_t>();
        h.slot_call = r.arr<int32_t>();
        h.slot_flat = r.arr<int32_t>();
        h.slot_duration = r.arr<int32_t>();
        h.wait_off = r.arr<int32_t>();
        h.waits = r.arr<int32_t>();
        h.notify_off = r.arr<int32_t>();
        h.notifies = r.arr<int32_t>();
        h.initial_counts = r.arr<int32_t>();
        for (int q = 0; q + 1 < static_cast<int>(h.queue_off.size()); ++q)
            for (int s = h.queue_off[static_cast<size_t>(q)]; s < h.queue_off[static_cast<size_t>(q) + 1]; ++s)
                h.slot_queue.push_back(q);
        I.hs.push_back(std::move(h));
    }
    et_config ec{};
    ec.device = cfg.device;
    ec.num_workers = workers;
    ec.record_trace = cfg.record_trace ? 1 : 0;
    ec.enable_prefetch = cfg.enable_prefetch ? 1 : 0;
    ec.watchdog_ns = cfg.watchdog_ns;
    ec.tick_ns = cfg.tick_ns;
    ec.step_limit = cfg.step_limit;
    ec.max_batch = cfg.max_batch;
    ec.l2_prefetch_bytes = cfg.l2_prefetch_bytes;
    const int rc = et_create(&ec, &I.rt);
    if (rc != ET_OK) raise_status(rc, "cannot create the GPU runtime");
    I.check(et_load_program(I.rt, path.c_str(), nullptr, nullptr), "load program");
    std::vector<et_op> none(I.k.graph.calls.size());
    std::memset(none.data(), 0, none.size() * sizeof(et_op));
    I.check(et_bind_ops(I.rt, none.data(), static_cast<int32_t>(none.size())), "bind ops");
    I.upload_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return ex;
}

void Executor::bind_ops(const std::vector<et_op>& ops) {
    Impl& I = *impl_;
    std::vector<et_op> full(I.k.graph.calls.size());
    std::memset(full.data(), 0, full.size() * sizeof(et_op));
    for (size_t i = 0; i < ops.size() && i < full.size(); ++i) full[i] = ops[i];
    I.check(et_bind_ops(I.rt, full.data(), static_cast<int32_t>(full.size())), "bind ops");
}

void Executor::set_runtime_tensor(const std::string& name, const std::vector<Int>& values) {
    Impl& I = *impl_;
    const int idx = I.k.graph.runtime_index(name);
    if (idx < 0) throw Error("undeclared runtime tensor '" + name + "'");
    std::vector<int32_t> v(values.begin(), values.end());
    I.check(et_set_runtime_tensor(I.rt, idx, v.data(), static_cast<int64_t>(v.size())), "runtime tensor");
}

void Executor::set_realization(const RoutingRealization& r) {
    for (const auto& kv : r.tensors) set_runtime_tensor(kv.first, kv.second);
}

std::vector<Int> Executor::runtime_tensor(const std::string& name, size_t n) const {
    const Impl& I = *impl_;
    const int idx = I.k.graph.runtime_index(name);
    if (idx < 0) throw Error("undeclared runtime tensor '" + name + "'");
    std::vector<int32_t> v(n);
    I.check(et_get_runtime_tensor(I.rt, idx, v.data(), static_cast<int64_t>(n)), "runtime tensor");
    return std::vector<Int>(v.begin(), v.end());
}

void Executor::launch(const ShapeBinding& b, void* stream) {
    Impl& I = *impl_;
    const auto v = binding_vector(I.k.graph, b);
    I.check(et_step(I.rt, v.data(), static_cast<int32_t>(v.size()), stream, 0, nullptr), "launch");
    I.last_binding = b;
}

namespace {
StepStats to_stats(const et_step_info& si) {
    StepStats s;
    s.sample_index = si.sample_index;
    s.tasks_executed = si.tasks_executed;
    s.noop_tasks = si.noop_tasks;
    s.pushes = si.pushes;
    s.pops = si.pops;
    s.kernel_ms = si.kernel_ms;
    return s;
}
}  // namespace

StepStats Executor::sync() {
    Impl& I = *impl_;
    et_step_info si{};
    const int rc = et_sync(I.rt, &si);
    I.last_sample = si.sample_index;
    I.last_step_id = si.step_id;
    if (rc != ET_OK) {
        std::string where = et_last_error(I.rt);
        if (rc == ET_ERR_DEADLOCK && si.sample_index >= 0 && si.slot >= 0) {
            const HostSample& h = I.hs[static_cast<size_t>(si.sample_index)];
            const int call = h.slot_call[static_cast<size_t>(si.slot)];
            where = "SM" + std::to_string(si.worker) + " blocked in " + I.k.graph.calls[static_cast<size_t>(call)].fn +
                    " task " + std::to_string(h.slot_task[static_cast<size_t>(si.slot)]) + " waiting on counter " +
                    std::to_string(si.counter) + " (value " + std::to_string(si.value) + ")";
        }
        raise_status(rc, where);
    }
    return to_stats(si);
}

StepStats Executor::run(const ShapeBinding& b) {
    Impl& I = *impl_;
    const auto v = binding_vector(I.k.graph, b);
    et_step_info si{};
    const int rc = et_step(I.rt, v.data(), static_cast<int32_t>(v.size()), nullptr, 1, &si);
    I.last_binding = b;
    I.last_sample = si.sample_index;
    I.last_step_id = si.step_id;
    if (rc != ET_OK) {
        std::string where = std::string(et_last_error(I.rt)) + " (worker " + std::to_string(si.worker) + ", slot " +
                            std::to_string(si.slot) + ", counter " + std::to_string(si.counter) + ", value " +
                            std::to_string(si.value) + ")";
        if (si.counter == -2) where += ": a consumer ring stage never filled";
        if (si.counter == -3) where += ": the producer never got a free ring stage";
        if (rc == ET_ERR_DEADLOCK && si.sample_index >= 0 && si.slot >= 0 && si.counter >= 0) {
            const HostSample& h = I.hs[static_cast<size_t>(si.sample_index)];
            const int call = h.slot_call[static_cast<size_t>(si.slot)];
            where = (si.worker == h.num_queues ? std::string("DMA") : "SM" + std::to_string(si.worker)) +
                    " blocked in " + I.k.graph.calls[static_cast<size_t>(call)].fn + " task " +
                    std::to_string(h.slot_task[static_cast<size_t>(si.slot)]) + " waiting on counter " +
                    std::to_string(si.counter) + " (value " + std::to_string(si.value) + ")";
        }
        raise_status(rc, where);
    }
    return to_stats(si);
}

std::vector<Int> Executor::final_counters() const {
    const Impl& I = *impl_;
    if (I.last_sample < 0) throw Error("no step has run");
    const HostSample& h = I.hs[static_cast<size_t>(I.last_sample)];
    std::vector<int64_t> v(h.initial_counts.size());
    I.check(et_read_counters(I.rt, v.data(), static_cast<int64_t>(v.size())), "read counters");
    // data-dependent elements: initial value = the counts tensor written on the device
    for (size_t t = 0; t < h.dd_base.size(); ++t) {
        std::vector<int32_t> cnt(static_cast<size_t>(h.dd_count[t]));
        I.check(et_get_runtime_tensor(I.rt, h.dd_counts_rt[t], cnt.data(), h.dd_count[t]), "read counts tensor");
        for (int32_t i = 0; i < h.dd_count[t]; ++i) v[static_cast<size_t>(h.dd_base[t] + i)] += cnt[static_cast<size_t>(i)];
    }
    return std::vector<Int>(v.begin(), v.end());
}

namespace {
Trace dynamic_trace(const GraphFunction& g, const HostSample& h, const std::vector<et_trace_rec>& recs, int step_id,
                    int workers, bool has_dma, Int seed, const ShapeBinding& binding) {
    Trace t;
    t.mode = "dynamic";
    t.num_sms = workers;
    t.has_dma = has_dma;
    t.seed = seed;
    t.binding = binding;
    t.measured = true;
    t.empty_polls.assign(static_cast<size_t>(t.num_resources()), 0);
    int64_t base = INT64_MAX;
    for (const auto& r : recs)
        if (r.pad == step_id) base = std::min<int64_t>(base, r.t_push > 0 ? std::min(r.t_push, r.t_begin) : r.t_begin);
    Int last = 0;
    for (size_t task = 0; task < recs.size(); ++task) {
        const et_trace_rec& r = recs[task];
        if (r.pad != step_id) continue;  // never pushed this step (beyond a realized extent)
        TaskRecord tr;
        tr.task_id = static_cast<int>(task);
        tr.call = h.slot_call[task];
        const auto& grid = g.call_grid(g.calls[static_cast<size_t>(tr.call)]);
        std::vector<Int> ext;
        for (size_t d = 0; d < grid.size(); ++d) ext.push_back(h.call_extents[static_cast<size_t>(tr.call) * 4 + d]);
        tr.coord = unflatten_coord(h.slot_flat[task], ext);
        tr.resource = r.worker;
        tr.noop = (r.flags & 1) != 0;
        const Int tb = r.t_begin - base, tw = r.t_wait_end - base, te = r.t_exec_end - base, tn = r.t_notify_end - base;
        tr.pop = Interval{tb, tb};
        const int nw = h.wait_off[task + 1] - h.wait_off[task];
        const int nn = h.notify_off[task + 1] - h.notify_off[task];
        for (int i = 0; i < nw; ++i) tr.waits.push_back(i == 0 ? Interval{tb, tw} : Interval{tw, tw});
        tr.exec = tr.noop ? Interval{tw, tw} : Interval{tw, te};
        if (r.t_prologue > 0 && !tr.noop) tr.prefetch = Interval{tw, r.t_prologue - base};
        for (int i = 0; i < nn; ++i) tr.notifies.push_back(i == 0 ? Interval{te, tn} : Interval{tn, tn});
        last = std::max({last, tr.exec.end, nn ? tn : tr.exec.end, nw ? tw : Int(0)});
        SchedEvent push;
        push.kind = SchedEvent::Kind::Push;
        push.time = r.t_push > 0 ? r.t_push - base : 0;
        push.task_id = tr.task_id;
        push.resource = -1;
        SchedEvent pop;
        pop.kind = SchedEvent::Kind::Pop;
        pop.time = tb;
        pop.task_id = tr.task_id;
        pop.resource = r.worker;
        t.sched_events.push_back(push);
        t.sched_events.push_back(pop);
        t.tasks.push_back(std::move(tr));
    }
    std::sort(t.sched_events.begin(), t.sched_events.end(),
              [](const SchedEvent& a, const SchedEvent& b) { return a.time < b.time; });
    t.makespan = last;
    return t;
}
}  // namespace

Trace Executor::trace() const {
    const Impl& I = *impl_;
    if (I.last_sample < 0) throw Error("no step has run");
    if (I.dyn) {
        const HostSample& h = I.hs[static_cast<size_t>(I.last_sample)];
        std::vector<et_trace_rec> recs(h.slot_call.size());
        int64_t n = static_cast<int64_t>(recs.size());
        I.check(et_read_trace(I.rt, recs.data(), &n), "read trace");
        Trace t = dynamic_trace(I.k.graph, h, recs, I.last_step_id, I.workers, h.has_dma != 0, I.cfg.seed,
                                I.last_binding);
        t.final_counters = final_counters();
        return t;
    }
    const HostSample& h = I.hs[static_cast<size_t>(I.last_sample)];
    std::vector<et_trace_rec> recs(h.slot_task.size());
    int64_t n = static_cast<int64_t>(recs.size());
    I.check(et_read_trace(I.rt, recs.data(), &n), "read trace");
    Trace t;
    t.mode = "static";
    t.num_sms = h.num_queues;
    t.has_dma = h.has_dma != 0;
    t.seed = I.cfg.seed;
    t.binding = I.last_binding;
    t.measured = true;
    t.empty_polls.assign(static_cast<size_t>(t.num_resources()), 0);
    int64_t base = INT64_MAX;
    for (const auto& r : recs) base = std::min<int64_t>(base, r.t_begin);
    if (recs.empty()) base = 0;
    const GraphFunction& g = I.k.graph;
    Int last = 0;
    t.tasks.reserve(recs.size());
    for (size_t s = 0; s < recs.size(); ++s) {
        const et_trace_rec& r = recs[s];
        TaskRecord tr;
        tr.task_id = h.slot_task[s];
        tr.call = h.slot_call[s];
        const auto& grid = g.call_grid(g.calls[static_cast<size_t>(tr.call)]);
        std::vector<Int> ext;
        for (size_t d = 0; d < grid.size(); ++d) ext.push_back(h.call_extents[static_cast<size_t>(tr.call) * 4 + d]);
        tr.coord = unflatten_coord(h.slot_flat[s], ext);
        tr.resource = h.slot_queue[s];
        tr.noop = (r.flags & 1) != 0;
        const Int tb = r.t_begin - base, tw = r.t_wait_end - base, te = r.t_exec_end - base, tn = r.t_notify_end - base;
        const int nw = h.wait_off[s + 1] - h.wait_off[s];
        const int nn = h.notify_off[s + 1] - h.notify_off[s];
        for (int i = 0; i < nw; ++i) tr.waits.push_back(i == 0 ? Interval{tb, tw} : Interval{tw, tw});
        tr.exec = tr.noop ? Interval{tw, tw} : Interval{tw, te};
        if (r.t_prologue > 0 && !tr.noop) tr.prefetch = Interval{tw, r.t_prologue - base};  // staging of activations
        for (int i = 0; i < nn; ++i) tr.notifies.push_back(i == 0 ? Interval{te, tn} : Interval{tn, tn});
        last = std::max({last, tr.exec.end, nn ? tn : tr.exec.end, nw ? tw : Int(0)});
        t.tasks.push_back(std::move(tr));
    }
    t.makespan = last;
    t.final_counters = final_counters();
    return t;
}

std::vector<et_trace_rec> Executor::raw_trace() const {
    Impl& I = *impl_;
    if (I.last_sample < 0) throw Error("no step has run");
    const HostSample& h = I.hs[static_cast<size_t>(I.last_sample)];
    std::vector<et_trace_rec> recs(I.dyn ? h.slot_call.size() : h.slot_task.size());
    int64_t n = static_cast<int64_t>(recs.size());
    I.check(et_read_trace(I.rt, recs.data(), &n), "read trace");
    recs.resize(static_cast<size_t>(n));
    return recs;
}

const StaticMegakernel& Executor::kernel() const { return impl_->k; }
bool Executor::dynamic() const { return impl_->dyn; }
int Executor::num_workers() const { return impl_->workers; }
double Executor::upload_ms() const { return impl_->upload_ms; }
void Executor::set_debug(int bits) { et_set_debug(impl_->rt, bits); }
void Executor::set_l2_prefetch(Int bytes) { et_set_l2_prefetch(impl_->rt, bytes); }

// ---------------------------------------------------------------------------
// Reference-named entry points.

namespace {
ExecConfig from_sim(const SimConfig& cfg, Int total_slots) {
    ExecConfig e;
    e.num_workers = cfg.num_sms;
    e.seed = cfg.seed;
    e.enable_prefetch = cfg.enable_prefetch;
    // The reference counts simulator events; here the bound is on executed
    // tasks and only enforced when it can trigger.
    e.step_limit = cfg.step_limit < total_slots ? std::max<Int>(cfg.step_limit, 1) : 0;
    return e;
}
}  // namespace

Trace simulate(const StaticMegakernel& k, const ShapeBinding& binding, const RoutingRealization* realization,
               const SimConfig& cfg) {
    if (cfg.num_sms != k.num_sms)
        throw Error("kernel was compiled for " + std::to_string(k.num_sms) + " SMs, run asked for " +
                    std::to_string(cfg.num_sms));
    (void)select_queues(k, binding);  // same validation and errors as the reference
    Int slots = 0;
    for (const auto& s : k.samples) slots = std::max(slots, s.num_tasks());
    Executor ex(k, from_sim(cfg, slots));
    if (realization) ex.set_realization(*realization);
    ex.run(binding);
    return ex.trace();
}

Trace simulate(const DynamicMegakernel& k, const ShapeBinding& binding, const RoutingRealization* realization,
               const SimConfig& cfg) {
    // same validation as the reference's launch-time instantiation (ref simulate.cpp:307)
    (void)instantiate(k.graph, binding, realization, cfg.seed);
    ExecConfig e;
    e.num_workers = cfg.num_sms;
    e.seed = cfg.seed;
    e.enable_prefetch = cfg.enable_prefetch;
    Int tasks = 0;
    for (const auto& c : k.graph.calls) {
        Int n = 1;
        for (const auto& d : k.graph.call_grid(c)) n *= eval_expr(d, binding);
        tasks += n;
    }
    e.step_limit = cfg.step_limit < tasks ? std::max<Int>(cfg.step_limit, 1) : 0;
    Executor ex(k, {binding}, e);
    if (realization) ex.set_realization(*realization);
    ex.run(binding);
    return ex.trace();
}

Trace simulate_barrier_baseline(const GraphFunction& g0, const ShapeBinding& binding,
                                const RoutingRealization* realization, const SimConfig& cfg) {
    const auto diags = validate_graph(g0);
    if (!diags.empty()) throw Error("invalid graph: " + diags.front());
    GraphFunction g = worst_case_rewrite(g0);
    // one stage per call: a one-element barrier event between consecutive calls
    for (size_t ci = 0; ci + 1 < g.calls.size(); ++ci) {
        EventTensorDecl e;
        e.name = "__stage" + std::to_string(ci);
        e.shape = {SymExpr::constant(1)};
        g.event_tensors.push_back(e);
        EdgeSpec out;
        out.event = e.name;
        out.map = {SymExpr::constant(0)};
        g.calls[ci].out_edges.push_back(out);
        g.calls[ci + 1].in_edges.push_back(out);
    }
    StaticMegakernel k = lower_static(g, {binding}, cfg.num_sms);
    SimConfig c = cfg;
    c.num_sms = k.num_sms;
    Trace t = simulate(k, binding, realization, c);
    t.mode = "barrier";
    t.final_counters.clear();
    return t;
}

}  // namespace etsim
