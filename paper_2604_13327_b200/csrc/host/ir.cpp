// Graph IR helpers and structural validation.
// Rules follow ref src/ir.cpp:79-235 (validate_graph) and :237-252
// (summarize_graph); diagnostics are this implementation's own wording.
#include "etsim/ir.hpp"

#include <algorithm>
#include <cctype>
#include <unordered_map>

namespace etsim {

DurationModel DurationModel::constant(Int v) {
    DurationModel m;
    m.kind = Kind::Constant;
    m.value = v;
    return m;
}

DurationModel DurationModel::table_of(std::vector<Int> values) {
    DurationModel m;
    m.kind = Kind::Table;
    m.table = std::move(values);
    return m;
}

DurationModel DurationModel::uniform(Int lo, Int hi) {
    DurationModel m;
    m.kind = Kind::Uniform;
    m.lo = lo;
    m.hi = hi;
    return m;
}

DurationModel DurationModel::skewed(Int base, Int factor, std::string indptr, Int hot_group) {
    DurationModel m;
    m.kind = Kind::SkewedByGroup;
    m.base = base;
    m.factor = factor;
    m.group_indptr = std::move(indptr);
    m.hot_group = hot_group;
    return m;
}

const DeviceFunctionDecl* GraphFunction::find_fn(const std::string& name) const {
    auto it = std::find_if(device_functions.begin(), device_functions.end(),
                           [&](const DeviceFunctionDecl& f) { return f.name == name; });
    return it == device_functions.end() ? nullptr : &*it;
}

int GraphFunction::event_index(const std::string& name) const {
    for (int i = 0; i < static_cast<int>(event_tensors.size()); ++i)
        if (event_tensors[i].name == name) return i;
    return -1;
}

int GraphFunction::runtime_index(const std::string& name) const {
    for (int i = 0; i < static_cast<int>(runtime_tensors.size()); ++i)
        if (runtime_tensors[i].name == name) return i;
    return -1;
}

const std::vector<ExprPtr>& GraphFunction::call_grid(const CallDevice& c) const {
    static const std::vector<ExprPtr> none;
    if (!c.grid.empty()) return c.grid;
    const DeviceFunctionDecl* f = find_fn(c.fn);
    return f ? f->grid : none;
}

namespace {

// "t<k>" with k < rank names a task coordinate.
bool coord_symbol(const std::string& s, int rank) {
    if (s.size() < 2 || s[0] != 't') return false;
    if (!std::all_of(s.begin() + 1, s.end(), [](char c) { return std::isdigit(static_cast<unsigned char>(c)); }))
        return false;
    if (s.size() > 9) return false;
    return std::stoi(s.substr(1)) < rank;
}

struct Validator {
    const GraphFunction& g;
    std::vector<std::string> out;
    std::set<std::string> syms, fns, events, rts;

    void note(std::string s) { out.push_back(std::move(s)); }

    void closed(const std::vector<ExprPtr>& v, const std::string& where, int task_rank) {
        for (const auto& e : v) {
            if (!e) {
                note(where + ": null expression");
                continue;
            }
            for (const auto& s : free_symbols(e))
                if (!syms.count(s) && !(task_rank >= 0 && coord_symbol(s, task_rank)))
                    note(where + ": unbound symbol '" + s + "'");
        }
    }

    void declarations() {
        syms.insert(g.symbols.begin(), g.symbols.end());
        if (!g.size_symbol.empty() && !syms.count(g.size_symbol))
            note("size symbol '" + g.size_symbol + "' is not declared");
        for (const auto& f : g.device_functions) {
            if (!fns.insert(f.name).second) note("device function '" + f.name + "' declared twice");
            if (!f.duration.empty() && !g.duration_models.count(f.duration))
                note("device function '" + f.name + "': no duration model '" + f.duration + "'");
            if (!f.prefetch.empty() && !g.duration_models.count(f.prefetch))
                note("device function '" + f.name + "': no prefetch model '" + f.prefetch + "'");
        }
        for (const auto& e : g.event_tensors) {
            if (!events.insert(e.name).second) note("event tensor '" + e.name + "' declared twice");
            if (e.shape.empty()) note("event tensor '" + e.name + "' has rank 0");
            if (e.data_dependent && e.counts_tensor.empty())
                note("data-dependent event tensor '" + e.name + "' names no counts tensor");
            if (e.data_dependent && e.writer.empty())
                note("data-dependent event tensor '" + e.name + "' names no writer");
        }
        for (const auto& r : g.runtime_tensors) {
            if (!rts.insert(r.name).second) note("runtime tensor '" + r.name + "' declared twice");
            if (r.writer.empty() || !fns.count(r.writer))
                note("runtime tensor '" + r.name + "': writer '" + r.writer + "' is not a device function");
        }
        for (const auto& e : g.event_tensors) {
            if (!e.data_dependent) continue;
            if (!e.counts_tensor.empty() && !rts.count(e.counts_tensor))
                note("event tensor '" + e.name + "': counts tensor '" + e.counts_tensor + "' undeclared");
            if (!e.writer.empty() && !fns.count(e.writer))
                note("event tensor '" + e.name + "': writer '" + e.writer + "' undeclared");
        }
        for (const auto& f : g.device_functions) closed(f.grid, "grid of '" + f.name + "'", -1);
        for (const auto& e : g.event_tensors) closed(e.shape, "shape of event '" + e.name + "'", -1);
        for (const auto& r : g.runtime_tensors) closed(r.shape, "shape of runtime tensor '" + r.name + "'", -1);
    }

    void calls() {
        std::unordered_map<std::string, int> first_write;
        for (int ci = 0; ci < static_cast<int>(g.calls.size()); ++ci)
            for (const auto& e : g.calls[ci].out_edges) first_write.emplace(e.event, ci);

        for (int ci = 0; ci < static_cast<int>(g.calls.size()); ++ci) {
            const CallDevice& c = g.calls[ci];
            const std::string at = "call " + std::to_string(ci) + " (" + c.fn + ")";
            if (!fns.count(c.fn)) {
                note(at + ": device function is not declared");
                continue;
            }
            const auto& grid = g.call_grid(c);
            if (grid.empty()) note(at + ": grid has rank 0");
            const int rank = static_cast<int>(grid.size());
            closed(grid, at + " grid", -1);
            if (!c.extent_from.empty() && !rts.count(c.extent_from))
                note(at + ": extent tensor '" + c.extent_from + "' undeclared");

            for (int dir = 0; dir < 2; ++dir) {
                const bool incoming = dir == 0;
                for (const auto& e : incoming ? c.in_edges : c.out_edges) {
                    const std::string eat = at + (incoming ? " wait on '" : " notify of '") + e.event + "'";
                    const int ei = g.event_index(e.event);
                    if (ei < 0) {
                        note(eat + ": no such event tensor");
                        continue;
                    }
                    const auto& decl = g.event_tensors[ei];
                    if (e.kind == MapKind::StaticMap) {
                        if (e.map.size() != decl.shape.size())
                            note(eat + ": map has " + std::to_string(e.map.size()) +
                                 " coordinates, event rank is " + std::to_string(decl.shape.size()));
                        closed(e.map, eat + " map", rank);
                    } else if (e.kind == MapKind::DataDependentNotify) {
                        if (incoming) note(eat + ": routed notify used as a wait");
                        const int ri = g.runtime_index(e.routing_tensor);
                        if (ri < 0)
                            note(eat + ": routing tensor '" + e.routing_tensor + "' undeclared");
                        else if (g.runtime_tensors[ri].role != TensorRole::Routing)
                            note(eat + ": '" + e.routing_tensor + "' is not a routing tensor");
                    } else {
                        if (!incoming) note(eat + ": range trigger used as a notify");
                        const int ri = g.runtime_index(e.indptr_tensor);
                        if (ri < 0)
                            note(eat + ": indptr tensor '" + e.indptr_tensor + "' undeclared");
                        else if (g.runtime_tensors[ri].role != TensorRole::Indptr)
                            note(eat + ": '" + e.indptr_tensor + "' is not an indptr tensor");
                        if (decl.shape.size() != 1) note(eat + ": range trigger needs a rank-1 event");
                    }
                    if (incoming) {
                        auto it = first_write.find(e.event);
                        if (it != first_write.end() && it->second > ci)
                            note(eat + ": first written by later call " + std::to_string(it->second) +
                                 " (program order must be feed-forward)");
                    }
                }
            }
            const DeviceFunctionDecl* f = g.find_fn(c.fn);
            if (f && f->resource == Resource::DMA)
                for (const auto& e : c.out_edges)
                    if (e.kind != MapKind::StaticMap) note(at + ": DMA call with a data-dependent notify");
        }
    }

    void writers() {
        std::unordered_map<std::string, int> launches;
        for (const auto& c : g.calls) ++launches[c.fn];
        for (const auto& e : g.event_tensors)
            if (e.data_dependent && !e.writer.empty() && launches[e.writer] != 1)
                note("writer '" + e.writer + "' of event '" + e.name + "' must be launched exactly once");
        for (const auto& r : g.runtime_tensors)
            if (!r.writer.empty() && launches[r.writer] != 1)
                note("writer '" + r.writer + "' of runtime tensor '" + r.name + "' must be launched exactly once");
    }
};

}  // namespace

std::vector<std::string> validate_graph(const GraphFunction& g) {
    Validator v{g, {}, {}, {}, {}, {}};
    v.declarations();
    v.calls();
    v.writers();
    return std::move(v.out);
}

GraphSummary summarize_graph(const GraphFunction& g) {
    GraphSummary s;
    s.num_calls = static_cast<int>(g.calls.size());
    s.num_event_tensors = static_cast<int>(g.event_tensors.size());
    s.num_runtime_tensors = static_cast<int>(g.runtime_tensors.size());
    s.symbols.insert(g.symbols.begin(), g.symbols.end());
    for (const auto& e : g.event_tensors) s.has_data_dependent |= e.data_dependent;
    for (const auto& c : g.calls) {
        for (const auto& e : c.in_edges) s.has_data_dependent |= e.kind != MapKind::StaticMap;
        for (const auto& e : c.out_edges) s.has_data_dependent |= e.kind != MapKind::StaticMap;
    }
    return s;
}

}  // namespace etsim
