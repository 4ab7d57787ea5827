// tc_probe.cu -- test hook: minimal tcgen05 experiments (TMEM round trip, one 128x128x8 MMA with
// no-swizzle and 128B-swizzle K-major operands).  Used by tests/test_gpu_gemm.py to pin down
// descriptor / TMEM semantics on the device; not on the product path.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint32_t su32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
}

__device__ __forceinline__ void st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n\t"
        "tcgen05.wait::st.sync.aligned;" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
        "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
        "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)(layout & 7) << 61;
    return d;
}

// mode 0: TMEM store/load round trip.  mode 1: MMA, no-swizzle K-major.  mode 2: MMA, SW128 K-major.
// out: 128 x 128 floats (lane-major).  A, B: 128 x 8 (row-major, K contiguous) inputs.
__global__ void __launch_bounds__(128, 1) probe_kernel(int mode, const float *A, const float *B, float *out,
                                                       uint32_t idesc_override) {
    __shared__ __align__(1024) float sa[128 * 32];
    __shared__ __align__(1024) float sb[128 * 32];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    const int t = threadIdx.x, warp = t / 32, lane = t % 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // operands into smem
    for (int i = t; i < 128 * 8; i += 128) {
        const int r = i / 8, k = i % 8;
        if (mode == 1) {
            // no swizzle, K-major core matrices (8 rows x 16 B): k-chunk c = k/4 at c*2048 B,
            // m-group g = r/8 at g*128 B, row r%8 at 16 B, element k%4 at 4 B.
            const int off = (k / 4) * 512 + (r / 8) * 32 + (r % 8) * 4 + (k % 4);
            sa[off] = A[r * 8 + k];
            sb[off] = B[r * 8 + k];
        } else {
            // SW128 K-major: row r at 128 B, 16-B chunk (k/4) xor (r%8)
            const int chunk = (k / 4) ^ (r % 8);
            const int off = r * 32 + chunk * 4 + (k % 4);
            sa[off] = A[r * 8 + k];
            sb[off] = B[r * 8 + k];
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = slot;
    if (mode == 0) {
        uint32_t r[32];
        for (int j = 0; j < 32; ++j) r[j] = __float_as_uint((float)(lane + 32 * warp) * 1000.f + j);
        for (int c0 = 0; c0 < 128; c0 += 32) st32(tmem + ((uint32_t)(32 * warp) << 16) + c0, r);
    } else if (t == 0) {
        const uint32_t idesc = idesc_override ? idesc_override
                                              : (1u << 4) | (2u << 7) | (2u << 10) | (16u << 17) | (8u << 24);
        uint64_t da, db;
        if (mode == 1) {
            da = sdesc(su32(sa), 2048, 128, 0);
            db = sdesc(su32(sb), 2048, 128, 0);
        } else {
            da = sdesc(su32(sa), 16, 1024, 2);
            db = sdesc(su32(sb), 16, 1024, 2);
        }
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"(0u));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                     : "memory");
    }
    if (mode != 0) {
        uint32_t done = 0;
        while (!done)
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(done)
                : "r"(su32(&bar)), "r"(0)
                : "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t r[32];
        ld32(tmem + ((uint32_t)(32 * warp) << 16) + c0, r);
        for (int j = 0; j < 32; ++j) out[(32 * warp + lane) * 128 + c0 + j] = __uint_as_float(r[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}


// mode 3: dynamic smem (manually 1024-aligned), K = 32 in four k-steps (+32 B descriptor advance),
// MMA issued by warp 1 lane 0 (TMEM allocated by warp 2), epilogue after an mbarrier wait only.
__global__ void __launch_bounds__(256, 1) probe3_kernel(const float *A, const float *B, float *out, int bmn,
                                                        uint32_t lbo_mn, uint32_t sbo_mn) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    float *sa = reinterpret_cast<float *>(sm);
    float *sb = reinterpret_cast<float *>(sm + 16384);
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + 32768);
    uint32_t *slot = reinterpret_cast<uint32_t *>(sm + 32768 + 64);
    const int t = threadIdx.x, warp = t / 32, lane = t % 32;
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(slot)), "r"(128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = t; i < 128 * 32; i += 256) {
        const int r = i / 32, k = i % 32;
        const int chunk = (k / 4) ^ (r % 8);
        sa[r * 32 + chunk * 4 + (k % 4)] = A[r * 32 + k];
        if (!bmn) {
            sb[r * 32 + chunk * 4 + (k % 4)] = B[r * 32 + k];
        } else {   // B given as K x N (n contiguous): element (k, n=r) in the MN-major SW128 layout
            const int n = r;
            // SWIZZLE_128B_BASE32B MN-major atom: 4 k-rows x 128 B, 32-B chunks XOR (k % 4)
            const int off = (n / 32) * 1024 + k * 32 + ((((n % 32) / 8) ^ (k % 4)) * 8) + (n % 8);
            sb[off] = B[k * 128 + n];
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *slot;
    if (warp == 1 && lane == 0) {
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)bmn << 16) | (16u << 17) | (8u << 24);
        for (int ks = 0; ks < 4; ++ks) {
            const uint64_t da = sdesc(su32(sa) + 32 * ks, 16, 1024, 2);
            const uint64_t db = bmn ? sdesc(su32(sb) + 1024 * ks, lbo_mn, sbo_mn, 1) : sdesc(su32(sb) + 32 * ks, 16, 1024, 2);
            const uint32_t acc = ks > 0;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
                     : "memory");
    }
    if (warp >= 4) {
        uint32_t done = 0;
        while (!done)
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(done)
                : "r"(su32(bar)), "r"(0)
                : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int wq = warp - 4;
        for (int c0 = 0; c0 < 128; c0 += 32) {
            uint32_t r[32];
            ld32(tmem + ((uint32_t)(32 * wq) << 16) + c0, r);
            for (int j = 0; j < 32; ++j) out[(32 * wq + lane) * 128 + c0 + j] = __uint_as_float(r[j]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

}  // namespace

extern "C" int kfac_debug_tc_probe(int mode, const float *A, const float *B, float *out, unsigned idesc, void *stream) {
    if (mode >= 3) {
        // mode 3: B K-major; mode 4: B MN-major (LBO 4096 = MN-group stride, SBO 1024 = 8-row K group);
        // mode 5: B MN-major with LBO/SBO swapped.
        cudaFuncSetAttribute(probe3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        const uint32_t lbo = mode == 5 ? 512 : 4096, sbo = mode == 5 ? 4096 : 512;
        probe3_kernel<<<1, 256, 200 * 1024, reinterpret_cast<cudaStream_t>(stream)>>>(A, B, out, mode >= 4, lbo, sbo);
        return (int)cudaGetLastError();
    }
    probe_kernel<<<1, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(mode, A, B, out, idesc);
    return (int)cudaGetLastError();
}
