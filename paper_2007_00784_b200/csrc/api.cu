// api.cu -- the C-ABI of libkfac: host-side validation, workspace sizing and dispatch.
// See include/kfac.h for the contract of every entry point.
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <tuple>
#include <vector>

#include "internal.cuh"

namespace kfac {

// ----- implemented in the stage translation units -----
size_t factors_workspace_bytes(const kfac_layer_t *layers, int nl);
kfac_status_t factors_run(const kfac_layer_t *layers, int nl, const float *const *act,
                          const float *const *gout, float *const *A, const int32_t *ldA,
                          float *const *G, const int32_t *ldG, float *const *pA, float *const *pG,
                          float xi, int first, float out_scale, void *ws, cudaStream_t s);
kfac_status_t unpack_run(const float *const *packed, const int32_t *dims, float *const *F, const int32_t *ldF,
                         int count, float scale, cudaStream_t s);
size_t eigen_workspace_bytes(const int32_t *dims, int count);
kfac_status_t eigen_run(const float *const *F, const int32_t *dims, const int32_t *ldF, int count,
                        float *const *Q, const int32_t *ldQ, float *const *evals, int32_t *info,
                        uint32_t flags, void *ws, cudaStream_t s);
size_t inverse_workspace_bytes(const int32_t *dims, int count);
kfac_status_t inverse_run(const float *const *F, const int32_t *dims, const int32_t *ldF, int count,
                          float damping, float *const *Finv, const int32_t *ldFinv, int32_t *info,
                          void *ws, cudaStream_t s);
size_t precond_workspace_bytes(const int32_t *d_g, const int32_t *d_a, int nl, int mode);
kfac_status_t precond_run(const int32_t *d_g, const int32_t *d_a, int nl, const float *const *grad,
                          const int32_t *ldW, const float *const *QG, const int32_t *ldQG,
                          const float *const *vG, const float *const *QA, const int32_t *ldQA,
                          const float *const *vA, float damping, int mode, float *const *out,
                          void *ws, cudaStream_t s);
size_t klclip_workspace_bytes(const int32_t *rows, const int32_t *cols, int nl);
kfac_status_t klclip_run(float *const *P, const float *const *W, const int32_t *rows,
                         const int32_t *cols, const int32_t *ld, int nl, float lr, float kappa,
                         float *nu_out, double *s_out, void *ws, cudaStream_t s);

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

std::atomic<uint64_t> &launch_counter() {
    static std::atomic<uint64_t> c{0};
    return c;
}

int num_sms() {
    static std::mutex mu;
    static std::map<int, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    cache[dev] = n;
    return n;
}

cudaError_t set_smem_attr(const void *kernel, int bytes) {
    // the attribute is an upper bound: keep the largest value requested per (kernel, device), so
    // a launch with less dynamic shared memory never lowers it under a later, larger one
    static std::mutex mu;
    static std::map<std::pair<const void *, int>, int> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_pair(kernel, dev);
    auto it = done.find(key);
    if (it != done.end() && it->second >= bytes) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done[key] = bytes;
    return e;
}

namespace {
struct SidePool {                          // per thread: streams and events of the current device
    int dev = -1;
    std::vector<cudaStream_t> st;
    std::vector<cudaEvent_t> ev;           // ev[0]: fork; ev[1 + g]: join of stream g
};
}  // namespace

cudaError_t SideFork::fork(cudaStream_t s, int n) {
    thread_local SidePool P;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (n > kMaxSide) return cudaErrorInvalidValue;
    if (P.dev != dev) {                    // a thread that switched devices starts a new pool
        P = SidePool{};
        P.dev = dev;
        P.st.reserve(kMaxSide);            // never reallocated: handed-out pointers stay valid
        P.ev.reserve(kMaxSide + 1);
    }
    while ((int)P.st.size() < n) {
        cudaStream_t x;
        if ((e = cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking)) != cudaSuccess) return e;
        P.st.push_back(x);
    }
    while ((int)P.ev.size() < n + 1) {
        cudaEvent_t x;
        if ((e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming)) != cudaSuccess) return e;
        P.ev.push_back(x);
    }
    st_ = P.st.data();
    ev_ = P.ev.data();
    n_ = n;
    if ((e = cudaEventRecord(ev_[0], s)) != cudaSuccess) return e;
    for (int g = 0; g < n; ++g)
        if ((e = cudaStreamWaitEvent(st_[g], ev_[0], 0)) != cudaSuccess) return e;
    return cudaSuccess;
}

cudaError_t SideFork::join(cudaStream_t s) {
    cudaError_t e;
    for (int g = 0; g < n_; ++g) {
        if ((e = cudaEventRecord(ev_[1 + g], st_[g])) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(s, ev_[1 + g], 0)) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

namespace {

kfac_status_t check_device() {
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) {
        set_error(std::string("no CUDA device: ") + cudaGetErrorString(e));
        return KFAC_ERR_CUDA;
    }
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (major != 10 || minor != 0) {
        set_error("libkfac is built for sm_100a (B200); device is sm_" + std::to_string(major) +
                  std::to_string(minor));
        return KFAC_ERR_UNSUPPORTED;
    }
    return KFAC_OK;
}

kfac_status_t check_matrix(const void *p, int rows, int cols, int ld, const char *what, int idx) {
    KFAC_CHECK_ARG(p != nullptr, KFAC_ERR_INVALID_VALUE, "%s[%d] is NULL", what, idx);
    KFAC_CHECK_ARG(rows > 0 && cols > 0, KFAC_ERR_SHAPE, "%s[%d]: empty matrix", what, idx);
    KFAC_CHECK_ARG(ld >= cols, KFAC_ERR_SHAPE, "%s[%d]: ld %d < cols %d", what, idx, ld, cols);
    KFAC_CHECK_ARG(ld % 4 == 0, KFAC_ERR_ALIGNMENT, "%s[%d]: ld %d not a multiple of 4", what, idx, ld);
    KFAC_CHECK_ARG(aligned16(p), KFAC_ERR_ALIGNMENT, "%s[%d]: base not 16-byte aligned", what, idx);
    return KFAC_OK;
}

kfac_status_t check_ws(void *ws, size_t have, size_t need, const char *fn) {
    KFAC_CHECK_ARG(have >= need, KFAC_ERR_WORKSPACE, "%s: workspace %zu < required %zu bytes", fn, have, need);
    KFAC_CHECK_ARG(need == 0 || ws != nullptr, KFAC_ERR_WORKSPACE, "%s: workspace is NULL", fn);
    return KFAC_OK;
}

#define RET_IF(x)                         \
    do {                                  \
        kfac_status_t _s = (x);           \
        if (_s != KFAC_OK) return _s;     \
    } while (0)

kfac_status_t check_layer(const kfac_layer_t &L, int idx) {
    KFAC_CHECK_ARG(L.kind == KFAC_LINEAR || L.kind == KFAC_CONV2D, KFAC_ERR_INVALID_VALUE,
                   "layer %d: kind %d is neither linear nor conv2d (P:417)", idx, L.kind);
    KFAC_CHECK_ARG(L.batch > 0 && L.c_in > 0 && L.c_out > 0, KFAC_ERR_SHAPE,
                   "layer %d: non-positive batch/channels", idx);
    KFAC_CHECK_ARG(L.bias_col == 0 || L.bias_col == 1, KFAC_ERR_INVALID_VALUE, "layer %d: bias_col", idx);
    if (L.kind == KFAC_LINEAR) {
        KFAC_CHECK_ARG(L.h_in == 1 && L.w_in == 1 && L.h_out == 1 && L.w_out == 1 && L.k_h == 1 &&
                           L.k_w == 1 && L.stride_h == 1 && L.stride_w == 1 && L.pad_h == 0 && L.pad_w == 0,
                       KFAC_ERR_SHAPE, "layer %d: linear layers need unit spatial geometry", idx);
    } else {
        KFAC_CHECK_ARG(L.k_h > 0 && L.k_w > 0 && L.stride_h > 0 && L.stride_w > 0 && L.pad_h >= 0 &&
                           L.pad_w >= 0 && L.h_in > 0 && L.w_in > 0,
                       KFAC_ERR_SHAPE, "layer %d: bad conv geometry", idx);
        KFAC_CHECK_ARG(L.h_out == (L.h_in + 2 * L.pad_h - L.k_h) / L.stride_h + 1 &&
                           L.w_out == (L.w_in + 2 * L.pad_w - L.k_w) / L.stride_w + 1 && L.h_out > 0 &&
                           L.w_out > 0,
                       KFAC_ERR_SHAPE, "layer %d: h_out/w_out inconsistent with the geometry", idx);
    }
    const long long rows = (long long)L.batch * L.h_out * L.w_out;
    KFAC_CHECK_ARG(rows < (1LL << 31), KFAC_ERR_SHAPE, "layer %d: %lld rows >= 2^31", idx, rows);
    const long long da = (long long)L.c_in * L.k_h * L.k_w + L.bias_col;
    KFAC_CHECK_ARG(da <= 16384 && L.c_out <= 16384, KFAC_ERR_SHAPE, "layer %d: factor dim > 16384", idx);
    return KFAC_OK;
}

}  // namespace
}  // namespace kfac

using namespace kfac;

extern "C" {

int32_t kfac_version(void) { return 100; }

uint64_t kfac_launch_count(void) { return launch_counter().load(); }

const char *kfac_last_error(void) { return g_last_error.c_str(); }

const char *kfac_status_string(kfac_status_t s) {
    switch (s) {
        case KFAC_OK: return "KFAC_OK";
        case KFAC_ERR_INVALID_VALUE: return "KFAC_ERR_INVALID_VALUE";
        case KFAC_ERR_SHAPE: return "KFAC_ERR_SHAPE";
        case KFAC_ERR_ALIGNMENT: return "KFAC_ERR_ALIGNMENT";
        case KFAC_ERR_WORKSPACE: return "KFAC_ERR_WORKSPACE";
        case KFAC_ERR_UNSUPPORTED: return "KFAC_ERR_UNSUPPORTED";
        case KFAC_ERR_CUDA: return "KFAC_ERR_CUDA";
    }
    return "KFAC_ERR_UNKNOWN";
}

kfac_status_t kfac_layer_dims(const kfac_layer_t *layer, int32_t *d_a, int32_t *d_g, int64_t *rows) {
    KFAC_CHECK_ARG(layer != nullptr, KFAC_ERR_INVALID_VALUE, "kfac_layer_dims: layer is NULL");
    RET_IF(check_layer(*layer, 0));
    if (d_a) *d_a = layer->c_in * layer->k_h * layer->k_w + layer->bias_col;
    if (d_g) *d_g = layer->c_out;
    if (rows) *rows = (int64_t)layer->batch * layer->h_out * layer->w_out;
    return KFAC_OK;
}

size_t kfac_update_factors_workspace_size(const kfac_layer_t *layers, int32_t num_layers) {
    if (!layers || num_layers <= 0) return 0;
    for (int l = 0; l < num_layers; ++l)
        if (check_layer(layers[l], l) != KFAC_OK) return 0;
    return factors_workspace_bytes(layers, num_layers);
}

kfac_status_t kfac_update_factors(const kfac_layer_t *layers, int32_t num_layers,
                                  const float *const *act, const float *const *gout,
                                  float *const *A, const int32_t *ld_A, float *const *G,
                                  const int32_t *ld_G, float *const *packed_A, float *const *packed_G,
                                  float xi, int32_t first, float out_scale,
                                  void *ws, size_t ws_bytes, kfac_stream_t stream) {
    kfac::NvtxRange nvtx_range("kfac_update_factors");
    KFAC_CHECK_ARG(layers && act && gout && A && ld_A && G && ld_G, KFAC_ERR_INVALID_VALUE,
                   "kfac_update_factors: NULL argument");
    KFAC_CHECK_ARG(num_layers > 0, KFAC_ERR_INVALID_VALUE, "kfac_update_factors: num_layers <= 0");
    KFAC_CHECK_ARG(xi >= 0.f && xi <= 1.f, KFAC_ERR_INVALID_VALUE, "xi %g not in [0,1]", xi);
    KFAC_CHECK_ARG(out_scale == out_scale, KFAC_ERR_INVALID_VALUE, "out_scale is NaN");
    for (int l = 0; l < num_layers; ++l) {
        const kfac_layer_t &L = layers[l];
        RET_IF(check_layer(L, l));
        KFAC_CHECK_ARG(act[l] && gout[l], KFAC_ERR_INVALID_VALUE, "layer %d: act/gout NULL", l);
        KFAC_CHECK_ARG(aligned16(act[l]) && aligned16(gout[l]), KFAC_ERR_ALIGNMENT,
                       "layer %d: act/gout not 16-byte aligned", l);
        const int da = L.c_in * L.k_h * L.k_w + L.bias_col;
        RET_IF(check_matrix(A[l], da, da, ld_A[l], "A", l));
        RET_IF(check_matrix(G[l], L.c_out, L.c_out, ld_G[l], "G", l));
        if (packed_A) KFAC_CHECK_ARG(packed_A[l] != nullptr, KFAC_ERR_INVALID_VALUE, "packed_A[%d] is NULL", l);
        if (packed_G) KFAC_CHECK_ARG(packed_G[l] != nullptr, KFAC_ERR_INVALID_VALUE, "packed_G[%d] is NULL", l);
    }
    RET_IF(check_ws(ws, ws_bytes, factors_workspace_bytes(layers, num_layers), "kfac_update_factors"));
    RET_IF(check_device());
    return factors_run(layers, num_layers, act, gout, A, ld_A, G, ld_G, packed_A, packed_G, xi,
                       first ? 1 : 0, out_scale, ws, reinterpret_cast<cudaStream_t>(stream));
}

kfac_status_t kfac_unpack_factors(const float *const *packed, const int32_t *dims, float *const *F,
                                  const int32_t *ld_F, int32_t count, float scale, kfac_stream_t stream) {
    kfac::NvtxRange nvtx_range("kfac_unpack_factors");
    KFAC_CHECK_ARG(packed && dims && F && ld_F, KFAC_ERR_INVALID_VALUE, "kfac_unpack_factors: NULL argument");
    KFAC_CHECK_ARG(count > 0, KFAC_ERR_INVALID_VALUE, "kfac_unpack_factors: count <= 0");
    for (int i = 0; i < count; ++i) {
        KFAC_CHECK_ARG(dims[i] > 0 && dims[i] <= 16384, KFAC_ERR_SHAPE, "dims[%d] = %d out of range", i, dims[i]);
        KFAC_CHECK_ARG(packed[i] != nullptr, KFAC_ERR_INVALID_VALUE, "packed[%d] is NULL", i);
        RET_IF(check_matrix(F[i], dims[i], dims[i], ld_F[i], "F", i));
    }
    RET_IF(check_device());
    KFAC_CHECK_ARG(scale == scale, KFAC_ERR_INVALID_VALUE, "kfac_unpack_factors: scale is NaN");
    return unpack_run(packed, dims, F, ld_F, count, scale, reinterpret_cast<cudaStream_t>(stream));
}

size_t kfac_compute_eigen_workspace_size(const int32_t *dims, int32_t count) {
    if (!dims || count <= 0) return 0;
    for (int i = 0; i < count; ++i)
        if (dims[i] <= 0 || dims[i] > 16384) return 0;
    return eigen_workspace_bytes(dims, count);
}

kfac_status_t kfac_compute_eigen(const float *const *F, const int32_t *dims, const int32_t *ld_F,
                                 int32_t count, float *const *Q, const int32_t *ld_Q,
                                 float *const *evals, int32_t *info, uint32_t flags, void *ws,
                                 size_t ws_bytes, kfac_stream_t stream) {
    kfac::NvtxRange nvtx_range("kfac_compute_eigen");
    KFAC_CHECK_ARG(F && dims && ld_F && Q && ld_Q && evals, KFAC_ERR_INVALID_VALUE,
                   "kfac_compute_eigen: NULL argument");
    KFAC_CHECK_ARG(count > 0, KFAC_ERR_INVALID_VALUE, "kfac_compute_eigen: count <= 0");
    KFAC_CHECK_ARG((flags & ~(KFAC_EIG_WARM_START | KFAC_EIG_JACOBI | KFAC_EIG_TRIDIAG | KFAC_EIG_TWO_STAGE |
                              KFAC_EIG_ONE_STAGE)) == 0 &&
                       (flags & (KFAC_EIG_JACOBI | KFAC_EIG_TRIDIAG)) != (KFAC_EIG_JACOBI | KFAC_EIG_TRIDIAG) &&
                       (flags & (KFAC_EIG_TWO_STAGE | KFAC_EIG_ONE_STAGE)) != (KFAC_EIG_TWO_STAGE | KFAC_EIG_ONE_STAGE),
                   KFAC_ERR_INVALID_VALUE, "unknown or conflicting flags 0x%x", flags);
    for (int i = 0; i < count; ++i) {
        KFAC_CHECK_ARG(dims[i] > 0 && dims[i] <= 16384, KFAC_ERR_SHAPE, "dims[%d] = %d out of range", i, dims[i]);
        RET_IF(check_matrix(F[i], dims[i], dims[i], ld_F[i], "F", i));
        RET_IF(check_matrix(Q[i], dims[i], dims[i], ld_Q[i], "Q", i));
        KFAC_CHECK_ARG(evals[i] != nullptr, KFAC_ERR_INVALID_VALUE, "evals[%d] is NULL", i);
    }
    RET_IF(check_ws(ws, ws_bytes, eigen_workspace_bytes(dims, count), "kfac_compute_eigen"));
    RET_IF(check_device());
    return eigen_run(F, dims, ld_F, count, Q, ld_Q, evals, info, flags, ws,
                     reinterpret_cast<cudaStream_t>(stream));
}

size_t kfac_compute_inverse_workspace_size(const int32_t *dims, int32_t count) {
    if (!dims || count <= 0) return 0;
    for (int i = 0; i < count; ++i)
        if (dims[i] <= 0 || dims[i] > 16384) return 0;
    return inverse_workspace_bytes(dims, count);
}

kfac_status_t kfac_compute_inverse(const float *const *F, const int32_t *dims, const int32_t *ld_F,
                                   int32_t count, float damping, float *const *Finv,
                                   const int32_t *ld_Finv, int32_t *info, void *ws, size_t ws_bytes,
                                   kfac_stream_t stream) {
    kfac::NvtxRange nvtx_range("kfac_compute_inverse");
    KFAC_CHECK_ARG(F && dims && ld_F && Finv && ld_Finv, KFAC_ERR_INVALID_VALUE,
                   "kfac_compute_inverse: NULL argument");
    KFAC_CHECK_ARG(count > 0, KFAC_ERR_INVALID_VALUE, "kfac_compute_inverse: count <= 0");
    KFAC_CHECK_ARG(damping >= 0.f, KFAC_ERR_INVALID_VALUE, "damping %g < 0", damping);
    for (int i = 0; i < count; ++i) {
        KFAC_CHECK_ARG(dims[i] > 0 && dims[i] <= 16384, KFAC_ERR_SHAPE, "dims[%d] = %d out of range", i, dims[i]);
        RET_IF(check_matrix(F[i], dims[i], dims[i], ld_F[i], "F", i));
        RET_IF(check_matrix(Finv[i], dims[i], dims[i], ld_Finv[i], "Finv", i));
    }
    RET_IF(check_ws(ws, ws_bytes, inverse_workspace_bytes(dims, count), "kfac_compute_inverse"));
    RET_IF(check_device());
    return inverse_run(F, dims, ld_F, count, damping, Finv, ld_Finv, info, ws,
                       reinterpret_cast<cudaStream_t>(stream));
}

size_t kfac_precondition_workspace_size(const int32_t *d_g, const int32_t *d_a, int32_t num_layers,
                                        int32_t mode) {
    if (!d_g || !d_a || num_layers <= 0) return 0;
    return precond_workspace_bytes(d_g, d_a, num_layers, mode);
}

kfac_status_t kfac_precondition(const int32_t *d_g, const int32_t *d_a, int32_t num_layers,
                                const float *const *grad, const int32_t *ld_W, const float *const *Q_G,
                                const int32_t *ld_QG, const float *const *v_G, const float *const *Q_A,
                                const int32_t *ld_QA, const float *const *v_A, float damping,
                                int32_t mode, float *const *out, void *ws, size_t ws_bytes,
                                kfac_stream_t stream) {
    kfac::NvtxRange nvtx_range("kfac_precondition");
    KFAC_CHECK_ARG(d_g && d_a && grad && ld_W && Q_G && ld_QG && Q_A && ld_QA && out,
                   KFAC_ERR_INVALID_VALUE, "kfac_precondition: NULL argument");
    KFAC_CHECK_ARG(num_layers > 0, KFAC_ERR_INVALID_VALUE, "kfac_precondition: num_layers <= 0");
    KFAC_CHECK_ARG(mode >= KFAC_PRECOND_EIGEN && mode <= KFAC_PRECOND_INVERSE, KFAC_ERR_INVALID_VALUE,
                   "kfac_precondition: unknown mode %d", mode);
    KFAC_CHECK_ARG(damping >= 0.f, KFAC_ERR_INVALID_VALUE, "damping %g < 0", damping);
    const bool eig = mode != KFAC_PRECOND_INVERSE;
    KFAC_CHECK_ARG(!eig || (v_G && v_A), KFAC_ERR_INVALID_VALUE, "kfac_precondition: v_G/v_A NULL");
    for (int l = 0; l < num_layers; ++l) {
        RET_IF(check_matrix(grad[l], d_g[l], d_a[l], ld_W[l], "grad", l));
        RET_IF(check_matrix(out[l], d_g[l], d_a[l], ld_W[l], "out", l));
        RET_IF(check_matrix(Q_G[l], d_g[l], d_g[l], ld_QG[l], "Q_G", l));
        RET_IF(check_matrix(Q_A[l], d_a[l], d_a[l], ld_QA[l], "Q_A", l));
        if (eig) KFAC_CHECK_ARG(v_G[l] && v_A[l], KFAC_ERR_INVALID_VALUE, "layer %d: v_G/v_A NULL", l);
    }
    RET_IF(check_ws(ws, ws_bytes, precond_workspace_bytes(d_g, d_a, num_layers, mode), "kfac_precondition"));
    RET_IF(check_device());
    return precond_run(d_g, d_a, num_layers, grad, ld_W, Q_G, ld_QG, v_G, Q_A, ld_QA, v_A, damping, mode,
                       out, ws, reinterpret_cast<cudaStream_t>(stream));
}

size_t kfac_kl_clip_workspace_size(const int32_t *rows, const int32_t *cols, int32_t num_layers) {
    if (!rows || !cols || num_layers <= 0) return 0;
    for (int l = 0; l < num_layers; ++l)
        if (rows[l] <= 0 || cols[l] <= 0) return 0;
    return klclip_workspace_bytes(rows, cols, num_layers);
}

kfac_status_t kfac_kl_clip(float *const *precond, const float *const *grad, const int32_t *rows,
                           const int32_t *cols, const int32_t *ld, int32_t num_layers, float lr,
                           float kappa, float *nu_out, double *s_out, void *ws, size_t ws_bytes,
                           kfac_stream_t stream) {
    kfac::NvtxRange nvtx_range("kfac_kl_clip");
    KFAC_CHECK_ARG(precond && grad && rows && cols && ld, KFAC_ERR_INVALID_VALUE, "kfac_kl_clip: NULL argument");
    KFAC_CHECK_ARG(num_layers > 0, KFAC_ERR_INVALID_VALUE, "kfac_kl_clip: num_layers <= 0");
    KFAC_CHECK_ARG(lr > 0.f && kappa > 0.f, KFAC_ERR_INVALID_VALUE, "kfac_kl_clip: lr and kappa must be > 0");
    for (int l = 0; l < num_layers; ++l) {
        RET_IF(check_matrix(precond[l], rows[l], cols[l], ld[l], "precond", l));
        RET_IF(check_matrix(grad[l], rows[l], cols[l], ld[l], "grad", l));
    }
    RET_IF(check_ws(ws, ws_bytes, klclip_workspace_bytes(rows, cols, num_layers), "kfac_kl_clip"));
    RET_IF(check_device());
    return klclip_run(precond, grad, rows, cols, ld, num_layers, lr, kappa, nu_out, s_out, ws,
                      reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
