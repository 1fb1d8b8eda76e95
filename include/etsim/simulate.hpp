// Executor entry points (drop-in for proj/include/etsim/simulate.hpp:8-36).
//
// In the reference these run a CPU discrete-event simulator. Here the same
// calls execute the lowered megakernel on the GPU: one persistent sm_100a
// launch whose CTAs walk the per-SM queues (static) or pop a device work queue
// (dynamic), spinning on and decrementing real Event Tensor counters. There is
// no CPU execution path; without a CUDA device these throw etsim::Error.
//
// SimConfig keeps the reference's fields. On hardware, num_sms is the number of
// persistent workers (queues), seed drives synthetic durations, step_limit
// bounds the executed task count, enable_prefetch toggles run-ahead weight
// staging. notify_cost / pop_cost / push_cost_per_task / poll_quantum describe
// simulated overheads and have no hardware meaning; they are accepted and
// ignored.
#pragma once

#include "etsim/sched_dynamic.hpp"
#include "etsim/sched_static.hpp"

namespace etsim {

struct SimConfig {
    int num_sms = 4;
    Int notify_cost = 0;
    Int pop_cost = 0;
    Int push_cost_per_task = 0;
    Int poll_quantum = 1;
    Int seed = 0;
    Int step_limit = 50'000'000;
    bool enable_prefetch = true;
};

Trace simulate(const StaticMegakernel& k, const ShapeBinding& binding,
               const RoutingRealization* realization, const SimConfig& cfg);

Trace simulate(const DynamicMegakernel& k, const ShapeBinding& binding,
               const RoutingRealization* realization, const SimConfig& cfg);

// Unfused ablation: one stage per call with a device-wide barrier between
// stages (ref simulate.cpp:682-794, paper section 5.5).
Trace simulate_barrier_baseline(const GraphFunction& g, const ShapeBinding& binding,
                                const RoutingRealization* realization, const SimConfig& cfg);

}  // namespace etsim
