// Probe of the tcgen05 operand layouts used by the large-batch GEMV (body_gemv_umma):
// one CTA computes D[128][N] = W[128][64] . X[N][64]^T with 4 kind::f16 MMAs
// (K-major, no swizzle: 8x16-byte core matrices, LBO 128 B along K, SBO 256 B
// along M/N), accumulators in TMEM read back with tcgen05.ld.32x32b.x16.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o scripts/umma_probe scripts/umma_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <cuda_bf16.h>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((addr >> 4) & 0x3fff);
    d |= static_cast<uint64_t>(128 >> 4) << 16;  // LBO: next 8-element K chunk
    d |= static_cast<uint64_t>(256 >> 4) << 32;  // SBO: next 8-row group
    d |= 1ull << 46;                             // version (sm_100)
    return d;
}

template <int N>
__global__ void probe(const __nv_bfloat16* W, const __nv_bfloat16* X, float* D) {
    __shared__ __align__(1024) uint8_t sa[128 * 64 * 2];
    __shared__ __align__(1024) uint8_t sb[N * 64 * 2];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t taddr_s;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // W[r][k] -> kstep*4096 + (r/8)*256 + ((k%16)/8)*128 + (r%8)*16 + (k%8)*2
    for (int v = tid; v < 128 * 8; v += blockDim.x) {
        const int r = v / 8, k0 = (v % 8) * 8;
        const uint4 val = *reinterpret_cast<const uint4*>(W + r * 64 + k0);
        const int off = (k0 / 16) * 4096 + (r / 8) * 256 + ((k0 % 16) / 8) * 128 + (r % 8) * 16;
        *reinterpret_cast<uint4*>(sa + off) = val;
    }
    for (int v = tid; v < N * 8; v += blockDim.x) {
        const int r = v / 8, k0 = (v % 8) * 8;
        const uint4 val = *reinterpret_cast<const uint4*>(X + r * 64 + k0);
        const int off = (k0 / 16) * (N * 32) + (r / 8) * 256 + ((k0 % 16) / 8) * 128 + (r % 8) * 16;
        *reinterpret_cast<uint4*>(sb + off) = val;
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&taddr_s)),
                     "r"(N < 32 ? 32 : N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t taddr = taddr_s;
    if (tid == 0) {
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
                               (static_cast<uint32_t>(128 >> 4) << 24);
        for (int j = 0; j < 4; ++j) {
            const uint64_t ad = sdesc(smem_u32(sa) + j * 4096), bd = sdesc(smem_u32(sb) + j * N * 32);
            const uint32_t acc = j > 0;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(taddr),
                "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&bar)));
    }
    // wait phase 0
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
        "@!P1 bra WAIT;\n\t}\n" ::"r"(smem_u32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t r[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr + (static_cast<uint32_t>(warp * 32) << 16) + c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        const int row = warp * 32 + lane;
        for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = __uint_as_float(r[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(N < 32 ? 32 : N));
}

template <int N>
int run() {
    std::vector<__nv_bfloat16> w(128 * 64), x(N * 64);
    std::vector<float> wf(128 * 64), xf(N * 64);
    srand(1);
    for (int i = 0; i < 128 * 64; ++i) {
        w[i] = __float2bfloat16((rand() % 17 - 8) / 8.f);
        wf[i] = __bfloat162float(w[i]);
    }
    for (int i = 0; i < N * 64; ++i) {
        x[i] = __float2bfloat16((rand() % 13 - 6) / 4.f);
        xf[i] = __bfloat162float(x[i]);
    }
    __nv_bfloat16 *dw, *dx;
    float* dd;
    cudaMalloc(&dw, w.size() * 2);
    cudaMalloc(&dx, x.size() * 2);
    cudaMalloc(&dd, 128 * N * 4);
    cudaMemcpy(dw, w.data(), w.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dx, x.data(), x.size() * 2, cudaMemcpyHostToDevice);
    cudaMemset(dd, 0, 128 * N * 4);
    probe<N><<<1, 128>>>(dw, dx, dd);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("N=%d cuda error %s\n", N, cudaGetErrorString(e));
        return 1;
    }
    std::vector<float> d(128 * N);
    cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    int bad = 0;
    for (int r = 0; r < 128; ++r)
        for (int n = 0; n < N; ++n) {
            double ref = 0;
            for (int k = 0; k < 64; ++k) ref += static_cast<double>(wf[r * 64 + k]) * xf[n * 64 + k];
            const double err = fabs(ref - d[r * N + n]);
            if (err > 1e-3) {
                if (bad < 4) printf("  mismatch r=%d n=%d got %f want %f\n", r, n, d[r * N + n], ref);
                ++bad;
            }
            maxerr = err > maxerr ? err : maxerr;
        }
    printf("N=%d maxerr %g bad %d\n", N, maxerr, bad);
    return bad != 0;
}

int main() {
    int f = 0;
    f |= run<16>();
    f |= run<32>();
    f |= run<64>();
    f |= run<128>();
    printf(f ? "FAIL\n" : "PASS\n");
    return f;
}
