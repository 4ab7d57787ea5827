// profile.cu -- per-launch CUDA-event timing of one kernel class (kfac_profile_start/stop), used
// by bench.py to report the dominant kernel's achieved rate against its roofline.
#include "common.cuh"

#include <mutex>
#include <vector>

namespace kfac {
namespace {

struct Rec {
    cudaEvent_t a, b;
    double bytes, flops;
};

std::mutex g_mu;
int g_class = 0;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;

cudaEvent_t get_event() {
    if (!g_pool.empty()) {
        cudaEvent_t e = g_pool.back();
        g_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

}  // namespace

int prof_begin(int kernel_class, cudaStream_t s) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_class == 0 || kernel_class != g_class) return -1;
    Rec r{get_event(), get_event(), 0.0, 0.0};
    cudaEventRecord(r.a, s);
    g_recs.push_back(r);
    return (int)g_recs.size() - 1;
}

void prof_end(int slot, cudaStream_t s, double bytes, double flops) {
    if (slot < 0) return;
    std::lock_guard<std::mutex> lk(g_mu);
    if (slot >= (int)g_recs.size()) return;
    cudaEventRecord(g_recs[slot].b, s);
    g_recs[slot].bytes = bytes;
    g_recs[slot].flops = flops;
}

}  // namespace kfac

extern "C" kfac_status_t kfac_profile_start(int32_t kernel_class) {
    KFAC_CHECK_ARG(kernel_class >= KFAC_PROF_TRD_PANEL && kernel_class <= KFAC_PROF_GEMM_TC,
                   KFAC_ERR_INVALID_VALUE, "kfac_profile_start: unknown kernel class %d", kernel_class);
    std::lock_guard<std::mutex> lk(kfac::g_mu);
    for (auto &r : kfac::g_recs) {
        kfac::g_pool.push_back(r.a);
        kfac::g_pool.push_back(r.b);
    }
    kfac::g_recs.clear();
    kfac::g_class = kernel_class;
    return KFAC_OK;
}

extern "C" kfac_status_t kfac_profile_stop(double *ms, int64_t *launches, double *bytes, double *flops) {
    KFAC_CHECK_ARG(ms && launches && bytes && flops, KFAC_ERR_INVALID_VALUE, "kfac_profile_stop: null output");
    std::lock_guard<std::mutex> lk(kfac::g_mu);
    double t = 0.0, by = 0.0, fl = 0.0;
    for (auto &r : kfac::g_recs) {
        KFAC_CUDA_TRY(cudaEventSynchronize(r.b));
        float e = 0.f;
        KFAC_CUDA_TRY(cudaEventElapsedTime(&e, r.a, r.b));
        t += e;
        by += r.bytes;
        fl += r.flops;
    }
    *ms = t;
    *launches = (int64_t)kfac::g_recs.size();
    *bytes = by;
    *flops = fl;
    kfac::g_class = 0;
    return KFAC_OK;
}
