// Dynamic (push/pop) scheduling, Algorithm 2 of the paper (drop-in for
// proj/include/etsim/sched_dynamic.hpp:12-31).
#pragma once

#include "etsim/materialize.hpp"

namespace etsim {

struct DynamicCallTemplate {
    int call = 0;
    bool has_prefetch = false;
    std::vector<uint8_t> wait_edges;  // per in-edge: 1 = the WAIT is armed
};

struct DynamicMegakernel {
    GraphFunction graph;
    bool early_push = false;
    std::vector<DynamicCallTemplate> templates;
};

DynamicMegakernel lower_dynamic(const GraphFunction& g, bool early_push = false);
DynamicMegakernel enable_early_push(DynamicMegakernel k);

}  // namespace etsim
