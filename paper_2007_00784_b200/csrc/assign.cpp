// assign.cpp -- Alg. 1 "Assign factors A_{0:L-1} and G_{1:L} to unique workers".
//
// Host-only, deterministic, identical on every rank: the assignment is a pure function of the
// factor dimensions and the world size, so no communication is needed to agree on it.
//   LPT_D3            greedy longest-processing-time on the d^3 eigendecomposition cost --
//                     the size-aware placement the paper proposes and the
//                     north_star's "greedy size-balanced" distribution;
//   ROUND_ROBIN_PAPER the paper's round robin in the form that reproduces its
//                     printed worker statistics: factor-granular [A0,G0,A1,G1,...]
//                     when W > L, layer-granular otherwise (R16);
//   LAYERWISE_LPT     K-FAC-lw: whole layers (cost d_A^3 + d_G^3) placed by LPT.
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <vector>

#include <string>

#include "kfac.h"

namespace kfac {
void set_error(const std::string &msg);
}

namespace {

void lpt(const std::vector<double> &cost, int world, std::vector<int> &owner) {
    std::vector<int> order(cost.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
    std::vector<double> load(world, 0.0);
    owner.assign(cost.size(), 0);
    for (int job : order) {
        int best = 0;
        for (int r = 1; r < world; ++r)
            if (load[r] < load[best]) best = r;
        load[best] += cost[job];
        owner[job] = best;
    }
}

}  // namespace

extern "C" kfac_status_t kfac_assign(const int32_t *dims, const int32_t *layer_of, int32_t nf,
                                     int32_t nl, int32_t world, int32_t policy, int32_t *owner) {
    if (!dims || !layer_of || !owner || nf <= 0 || nl <= 0 || world <= 0) {
        kfac::set_error("kfac_assign: null pointer or non-positive count");
        return KFAC_ERR_INVALID_VALUE;
    }
    for (int f = 0; f < nf; ++f) {
        if (dims[f] <= 0 || layer_of[f] < 0 || layer_of[f] >= nl) {
            kfac::set_error("kfac_assign: factor dimension <= 0 or layer index out of range");
            return KFAC_ERR_SHAPE;
        }
    }
    if (policy == KFAC_ASSIGN_ROUND_ROBIN_PAPER) {
        for (int f = 0; f < nf; ++f) owner[f] = world > nl ? f % world : layer_of[f] % world;
        return KFAC_OK;
    }
    std::vector<int> own;
    if (policy == KFAC_ASSIGN_LPT_D3) {
        std::vector<double> cost(nf);
        for (int f = 0; f < nf; ++f) cost[f] = (double)dims[f] * dims[f] * dims[f];
        lpt(cost, world, own);
        for (int f = 0; f < nf; ++f) owner[f] = own[f];
        return KFAC_OK;
    }
    if (policy == KFAC_ASSIGN_LAYERWISE_LPT) {
        std::vector<double> cost(nl, 0.0);
        for (int f = 0; f < nf; ++f) cost[layer_of[f]] += (double)dims[f] * dims[f] * dims[f];
        lpt(cost, world, own);
        for (int f = 0; f < nf; ++f) owner[f] = own[layer_of[f]];
        return KFAC_OK;
    }
    kfac::set_error("kfac_assign: unknown policy");
    return KFAC_ERR_INVALID_VALUE;
}
