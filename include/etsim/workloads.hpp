// Built-in graph templates (drop-in for proj/include/etsim/workloads.hpp).
#pragma once

#include "etsim/materialize.hpp"

namespace etsim {

GraphFunction splitk_rowsum();
GraphFunction gemm_reduce_scatter(const ExprPtr& mm_tiles, int fan_in);
GraphFunction gemm_reduce_scatter(const std::string& mm_tiles, int fan_in);
GraphFunction all_gather_gemm(Int chunks, Int tiles_per_chunk);

struct MoEParams {
    Int tokens = 8;
    Int experts = 4;
    Int top_k = 1;
    Int tile_size = 1;
    double hot_fraction = 0;
    Int hot_expert = 0;
};

GraphFunction moe_layer(const MoEParams& p);
RoutingRealization moe_realization(const MoEParams& p, Int seed);
GraphFunction random_dag(int nodes, int edges, Int seed);

}  // namespace etsim
