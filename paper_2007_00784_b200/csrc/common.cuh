// common.cuh -- shared host/device helpers of libkfac (CUDA path only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <atomic>
#include <string>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: no-ops unless a tool (ncu --nvtx) attaches

#include "kfac.h"

namespace kfac {

// ---------------------------------------------------------------- errors --
void set_error(const std::string &msg);
std::atomic<uint64_t> &launch_counter();

struct Status {
    kfac_status_t code;
};

#define KFAC_CHECK_ARG(cond, code, ...)                                   \
    do {                                                                  \
        if (!(cond)) {                                                    \
            char _buf[512];                                               \
            snprintf(_buf, sizeof(_buf), __VA_ARGS__);                    \
            ::kfac::set_error(_buf);                                      \
            return code;                                                  \
        }                                                                 \
    } while (0)

#define KFAC_CUDA_TRY(expr)                                                        \
    do {                                                                           \
        cudaError_t _e = (expr);                                                   \
        if (_e != cudaSuccess) {                                                   \
            ::kfac::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e)); \
            return KFAC_ERR_CUDA;                                                  \
        }                                                                          \
    } while (0)

// Count and check one launch (call right after <<<>>>).
#define KFAC_LAUNCHED()                                                            \
    do {                                                                           \
        ::kfac::launch_counter().fetch_add(1, std::memory_order_relaxed);          \
        cudaError_t _e = cudaGetLastError();                                       \
        if (_e != cudaSuccess) {                                                   \
            ::kfac::set_error(std::string("kernel launch: ") + cudaGetErrorString(_e)); \
            return KFAC_ERR_CUDA;                                                  \
        }                                                                          \
    } while (0)

inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

// Bump allocator over the caller's workspace (256-byte aligned slices).
struct WsArena {
    char *base;
    size_t cap, off = 0;
    WsArena(void *p, size_t n) : base(static_cast<char *>(p)), cap(n) {}
    template <class T>
    T *take(size_t count) {
        off = round_up(off, 256);
        T *p = reinterpret_cast<T *>(base ? base + off : nullptr);
        off += count * sizeof(T);
        return p;
    }
    bool ok() const { return off <= cap; }
};

int num_sms();   // multiprocessor count of the current device (cached per device)

// Host-side NVTX range over the launches of one stage (ncu --nvtx --nvtx-include "kfac_compute_eigen/"
// selects a stage's kernels; names follow the C-ABI calls and the eigensolver phases).
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

// cudaFuncSetAttribute(kernel, MaxDynamicSharedMemorySize, bytes) on the current device, done once
// per (kernel, device, bytes); thread-safe.
cudaError_t set_smem_attr(const void *kernel, int bytes);

// Fork/join of independent launches onto side streams of the calling thread (current device):
// fork(s, n) records an event on s and makes n side streams wait for it; side(g) is stream g;
// join(s) makes s wait for every side stream used since the fork.  Stream-ordered for the caller
// and capturable in a CUDA graph.
class SideFork {
public:
    static constexpr int kMaxSide = 64;     // side streams per thread and device
    cudaError_t fork(cudaStream_t s, int n);
    cudaStream_t side(int g) const { return st_[g]; }
    cudaError_t join(cudaStream_t s);
private:
    cudaStream_t *st_ = nullptr;
    cudaEvent_t *ev_ = nullptr;
    int n_ = 0;
};

// Per-launch instrumentation (kfac_profile_start/stop).  prof_begin returns a slot (< 0 when the
// class is not armed); prof_end records the closing event and the launch's algorithmic work.
int prof_begin(int kernel_class, cudaStream_t s);
void prof_end(int slot, cudaStream_t s, double bytes, double flops);

}  // namespace kfac
