// Microbenchmark of the megakernel's weight-streaming ring in isolation:
// one TMA producer thread + 8 consumer warps per CTA, STAGES x CHUNK bytes of
// shared memory, streaming a large bf16 matrix (GEMV x . W^T per row).
//   mode 0: consumers only wait + release (TMA / HBM bound)
//   mode 1: every warp consumes every chunk (contiguous slices), FHFMA dot products
//   mode 2: warp c % 8 owns chunk c (needs STAGES % 8 == 0)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ringbench scripts/ringbench.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <vector>
#include "../paper_2604_13327_b200/csrc/kernels/ptx.cuh"

using namespace etk;

template <int STAGES, int CHUNK, int MODE>
__global__ void __launch_bounds__(288, 1) ring_kernel(const uint8_t* W, long long bytes_per_cta, const uint16_t* x,
                                                     int K, float* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* ring = smem;
    uint16_t* xs = reinterpret_cast<uint16_t*>(smem + STAGES * CHUNK);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * CHUNK + K * 2);
    uint64_t* empty = full + STAGES;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint8_t* src = W + blockIdx.x * bytes_per_cta;
    const int nchunks = static_cast<int>(bytes_per_cta / CHUNK);
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], MODE >= 2 ? 1 : 8);
        }
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < K / 8; i += blockDim.x) reinterpret_cast<uint4*>(xs)[i] = reinterpret_cast<const uint4*>(x)[i];
    __syncthreads();
    if (warp == 8) {
        if (lane != 0) return;
        const uint64_t pol = policy_evict_first();
        for (int c = 0; c < nchunks; ++c) {
            const int st = c % STAGES;
            const uint32_t ph = (c / STAGES) & 1;
            while (!mbar_try_wait(&empty[st], ph ^ 1u)) {
            }
            mbar_arrive_expect_tx(&full[st], CHUNK);
            bulk_g2s(ring + st * CHUNK, src + static_cast<long long>(c) * CHUNK, CHUNK, &full[st], pol);
        }
        return;
    }
    float acc = 0.f;
    const int gpr = K / 256;
    constexpr int G = CHUNK / 512;
    for (int c = 0; c < nchunks; ++c) {
        if (MODE >= 2 && (c & 7) != warp) continue;
        const int st = c % STAGES;
        const uint32_t ph = (c / STAGES) & 1;
        while (!mbar_try_wait(&full[st], ph)) {
        }
        const uint4* wl = reinterpret_cast<const uint4*>(ring + st * CHUNK) + lane;
        if (MODE == 1) {
            constexpr int S = (G + 7) / 8;
            const int j0 = warp * S;
            float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
            for (int j = j0; j < j0 + S && j < G; j += 2) {
                const int kg = (c * G + j) % gpr;
                dot8_bf16(a0, a1, wl[j * 32], reinterpret_cast<const uint4*>(xs)[kg * 32 + lane]);
                if (j + 1 < j0 + S && j + 1 < G) {
                    const int kg1 = (c * G + j + 1) % gpr;
                    dot8_bf16(a2, a3, wl[(j + 1) * 32], reinterpret_cast<const uint4*>(xs)[kg1 * 32 + lane]);
                }
            }
            acc += (a0 + a1) + (a2 + a3);
        } else if (MODE == 3 || MODE == 4) {
            // warp-owned chunk, U groups per iteration, loads first, 2U chains
            constexpr int U = MODE == 3 ? 4 : 8;
            float a[2 * U];
#pragma unroll
            for (int u = 0; u < 2 * U; ++u) a[u] = 0.f;
            const uint4* xl = reinterpret_cast<const uint4*>(xs) + lane;
            int kg = (c * G) % gpr;
            for (int j = 0; j < G; j += U) {
                uint4 w[U], xv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) w[u] = wl[(j + u) * 32];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    int k2 = kg + u;
                    if (k2 >= gpr) k2 -= gpr;
                    xv[u] = xl[k2 * 32];
                }
#pragma unroll
                for (int u = 0; u < U; ++u) dot8_bf16(a[2 * u], a[2 * u + 1], w[u], xv[u]);
                kg += U;
                if (kg >= gpr) kg -= gpr;
            }
#pragma unroll
            for (int u = 0; u < 2 * U; ++u) acc += a[u];
        } else if (MODE == 2) {
            float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
            for (int j = 0; j < G; j += 2) {
                const int kg = (c * G + j) % gpr;
                dot8_bf16(a0, a1, wl[j * 32], reinterpret_cast<const uint4*>(xs)[kg * 32 + lane]);
                dot8_bf16(a2, a3, wl[(j + 1) * 32], reinterpret_cast<const uint4*>(xs)[((kg + 1) % gpr) * 32 + lane]);
            }
            acc += (a0 + a1) + (a2 + a3);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    }
    acc = warp_sum(acc);
    if (lane == 0) atomicAdd(out, acc);
}

template <int STAGES, int CHUNK, int MODE>
void run(const uint8_t* W, const uint16_t* x, float* out, int ctas, long long per_cta, int K) {
    const int smem = STAGES * CHUNK + K * 2 + 2 * STAGES * 8 + 64;
    cudaFuncSetAttribute(ring_kernel<STAGES, CHUNK, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int it = 0; it < 5; ++it) {
        cudaEventRecord(a);
        ring_kernel<STAGES, CHUNK, MODE><<<ctas, 288, smem>>>(W, per_cta, x, K, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (it > 0 && ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    printf("stages=%2d chunk=%5d mode=%d ctas=%3d: %8.1f us  %7.1f GB/s total  %6.1f GB/s per CTA %s\n", STAGES, CHUNK,
           MODE, ctas, best * 1e3, ctas * per_cta / (best * 1e-3) / 1e9, per_cta / (best * 1e-3) / 1e9,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    const int K = 4096;
    const long long per_cta = 6LL * 1024 * 1024 + 0;  // ~6.3 MB per CTA, multiple of 80 KB below
    const long long total = 148 * per_cta + (1 << 20);
    uint8_t* W;
    uint16_t* x;
    float* out;
    cudaMalloc(&W, total);
    cudaMalloc(&x, K * 2);
    cudaMalloc(&out, 4);
    cudaMemset(W, 0, total);
    cudaMemset(x, 0, K * 2);
    long long pc16 = per_cta / 16384 * 16384, pc20 = per_cta / 20480 * 20480, pc8 = per_cta / 8192 * 8192;
    for (int ctas : {1, 148}) {
        run<8, 20480, 0>(W, x, out, ctas, pc20, K);
        run<8, 20480, 2>(W, x, out, ctas, pc20, K);
        run<8, 20480, 3>(W, x, out, ctas, pc20, K);
        run<8, 20480, 4>(W, x, out, ctas, pc20, K);
        run<16, 12288, 3>(W, x, out, ctas, per_cta / 12288 * 12288, K);
        run<16, 12288, 4>(W, x, out, ctas, per_cta / 12288 * 12288, K);
        run<8, 24576, 3>(W, x, out, ctas, per_cta / 24576 * 24576, K);
        run<8, 24576, 4>(W, x, out, ctas, per_cta / 24576 * 24576, K);
    }
    return 0;
}
