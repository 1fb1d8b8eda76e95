// Issue-rate probe for the tensor-core GEMV inner loop: one thread issues `iters`
// groups of four kind::f16 MMAs (M=128, N=n, K=16) from shared memory into TMEM,
// optionally with a tcgen05.commit per group; reports cycles per group.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o scripts/umma_rate scripts/umma_rate.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
    return static_cast<uint64_t>((addr >> 4) & 0x3fff) | (8ull << 16) | (16ull << 32) | (1ull << 46);
}

template <int N, bool kCommit, int kExtra = 0>
__global__ void rate(int iters, long long* out) {
    __shared__ __align__(1024) uint8_t sa[16384];
    __shared__ __align__(1024) uint8_t sb[N * 64 * 2];
    __shared__ __align__(8) uint64_t bar[8];
    __shared__ uint32_t taddr_s;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sa)[i] = 0x3c003c00u;
    for (int i = tid; i < N * 32; i += blockDim.x) reinterpret_cast<uint32_t*>(sb)[i] = 0x3c003c00u;
    if (tid == 0) {
        for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t taddr = taddr_s;
    if (tid == 0) {
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) | (8u << 24);
        const uint64_t a0 = sdesc(smem_u32(sa)), b0 = sdesc(smem_u32(sb));
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (kExtra & 1) {  // an mbarrier probe per group (phase 1 of bar[7] never completes -> parity 1 passes)
                uint32_t ok;
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                             : "=r"(ok) : "r"(smem_u32(&bar[7])), "r"(1u) : "memory");
                if (!ok) out[2] = 1;
            }
            if (kExtra & 2) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            for (int j = 0; j < 4; ++j) {
                const uint32_t acc = (it | j) != 0;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(taddr + (it & 3) * N),
                    "l"(a0 + j * 256), "l"(b0 + j * (N * 2)), "r"(idesc), "r"(acc));
            }
            if (kCommit)
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                    smem_u32(&bar[it & 3])));
        }
        long long t1 = clock64();
        if (kExtra & 4) {  // round trip: commit then wait for its arrival, per group (bar[4])
            t0 = clock64();
            for (int it = 0; it < iters; ++it) {
                if (!(kExtra & 8)) {
                    for (int j = 0; j < 4; ++j)
                        asm volatile(
                            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(taddr),
                            "l"(a0 + j * 256), "l"(b0 + j * (N * 2)), "r"(idesc), "r"(1u));
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                    smem_u32(&bar[4])));
                uint32_t ok = 0;
                while (!ok)
                    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                                 : "=r"(ok) : "r"(smem_u32(&bar[4])), "r"(static_cast<uint32_t>(it & 1)) : "memory");
            }
            t1 = clock64();
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[0])));
        // wait for everything to drain
        uint32_t ok = 0;
        int spins = 0;
        while (!ok && spins < 1000000) {
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                         : "=r"(ok) : "r"(smem_u32(&bar[0])), "r"(0u));
            ++spins;
        }
        long long t2 = clock64();
        out[0] = t1 - t0;
        out[1] = t2 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr));
}

template <int N, bool C, int X = 0>
void run(int iters) {
    long long* d;
    cudaMalloc(&d, 24);
    rate<N, C, X><<<1, 128>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[2] = {0, 0};
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("extra=%d N=%3d commit=%d iters=%d: issue %.1f cyc/group, drained %.1f cyc/group (%s)\n", X, N, C, iters,
           double(h[0]) / iters, double(h[1]) / iters, cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    run<16, false>(4096);
    run<16, true>(4096);
    run<64, false>(4096);
    run<64, true>(4096);
    run<128, true>(4096);
    run<16, true, 1>(4096);
    run<16, true, 2>(4096);
    run<16, true, 3>(4096);
    run<16, true, 4>(1024);
    run<16, true, 12>(1024);
    return 0;
}
