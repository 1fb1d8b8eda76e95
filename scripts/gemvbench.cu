// Microbenchmark of the megakernel's GEMV consumer (mma.sync on frag16 tiles)
// and its weight ring, in isolation.  One TMA producer thread + 8 consumer
// warps per CTA; 8 stages x 20 KB; warp c % 8 owns chunk c.
//   mode 0: consumers only  (data already in smem, no mbarriers)  -> compute rate
//   mode 1: ring, producer arrives without copying (no HBM)       -> ring protocol + compute
//   mode 2: ring with TMA bulk copies from HBM                     -> full path
//   mode 3: ring with TMA, consumers only wait + release           -> HBM / TMA rate
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gemvbench scripts/gemvbench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../paper_2604_13327_b200/csrc/kernels/ptx.cuh"

using namespace etk;

constexpr int STAGES = 8, CHUNK = 20480, TPC = CHUNK / 512;

template <int MODE>
__global__ void __launch_bounds__(320, 1) bench_kernel(const uint8_t* W, long long bytes_per_cta, int K, float* out,
                                                      unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* ring = smem;
    uint16_t* xs = reinterpret_cast<uint16_t*>(smem + STAGES * CHUNK);
    float* acc = reinterpret_cast<float*>(smem + STAGES * CHUNK + K * 2);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * CHUNK + K * 2 + 4096 * 4);
    uint64_t* empty = full + STAGES;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint8_t* src = W + blockIdx.x * bytes_per_cta;
    const int nchunks = static_cast<int>(bytes_per_cta / CHUNK);
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < K / 2; i += blockDim.x) reinterpret_cast<uint32_t*>(xs)[i] = 0x3f803f80u;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) acc[i] = 0.f;
    __syncthreads();
    const long long t_start = clock64();
    volatile unsigned int* pub = reinterpret_cast<volatile unsigned int*>(empty + STAGES);  // producer's cseq
    if (warp == 9) {  // MODE 8/10: prefetch.global.L2 warp running AHEAD chunks in front of the producer
        if (MODE == 8 || MODE == 10) {
            constexpr int AHEAD = 24;
            int next = 0;
            while (next < nchunks) {
                const int lim = static_cast<int>(*pub) + AHEAD;
                if (next >= lim) continue;
                const char* p = reinterpret_cast<const char*>(src + static_cast<long long>(next) * CHUNK);
                for (int off = lane * 128; off < CHUNK; off += 32 * 128)
                    asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p + off));
                ++next;
            }
        }
        return;
    }
    if (warp == 8) {
        if (lane != 0 || MODE == 0) return;
        const uint64_t pol = policy_evict_first();
        for (int c = 0; c < nchunks; ++c) {
            const int st = c % STAGES;
            const uint32_t ph = (c / STAGES) & 1;
            while (!mbar_try_wait(&empty[st], ph ^ 1u)) {
            }
            if (MODE == 6) {  // L2 run-ahead cursor: AHEAD chunks in front of the ring
                constexpr int AHEAD = 12;
                if (c == 0)
                    for (int a = 0; a < AHEAD && a < nchunks; ++a) bulk_prefetch_l2(src + static_cast<long long>(a) * CHUNK, CHUNK);
                if (c + AHEAD < nchunks) bulk_prefetch_l2(src + static_cast<long long>(c + AHEAD) * CHUNK, CHUNK);
            }
            if (lane == 0) *pub = c;
            if (MODE == 1 || MODE == 4 || MODE == 5) {
                mbar_arrive(&full[st]);
            } else {
                mbar_arrive_expect_tx(&full[st], CHUNK);
                bulk_g2s(ring + st * CHUNK, src + static_cast<long long>(c) * CHUNK, CHUNK, &full[st], pol);
            }
        }
        return;
    }
    const int kst = K / 16;
    const int g = lane >> 2, q = lane & 3;
    const bool xlane = g < 1;
    const uint16_t* xrow = xs + 8 * q;
    for (int c = warp; c < nchunks; c += 8) {
        const int st = c % STAGES;
        const uint32_t ph = (c / STAGES) & 1;
        if (MODE != 0)
            while (!mbar_try_wait(&full[st], ph)) {
            }
        const uint8_t* buf = ring + st * CHUNK;
        if ((MODE == 9 || MODE == 10) && (c % 64) < 8) {  // a dependency bubble: ~5 us
            const long long t = clock64();
            while (clock64() - t < 10000) {
            }
        }
        if (MODE == 4) {  // LDS only
            uint32_t x = 0;
            const uint4* ap = reinterpret_cast<const uint4*>(buf) + lane;
#pragma unroll 4
            for (int i = 0; i < TPC; i += 2) {
                const uint4 a0 = lds128(ap + i * 32);
                const uint4 a1 = lds128(ap + (i + 1) * 32);
                const uint4 xv = xlane ? lds128(xrow + i * 16) : make_uint4(0u, 0u, 0u, 0u);
                x ^= a0.x ^ a0.y ^ a0.z ^ a0.w ^ a1.x ^ a1.y ^ a1.z ^ a1.w ^ xv.x ^ xv.w;
            }
            if (x == 0x12345678u) acc[lane] = 1.f;
        } else if (MODE == 5) {  // MMA only (register operands)
            float d0[4] = {0.f, 0.f, 0.f, 0.f}, d1[4] = {0.f, 0.f, 0.f, 0.f};
            const uint4 a0 = make_uint4(lane, 1u, 2u, 3u), a1 = make_uint4(3u, lane, 1u, 0u);
#pragma unroll 4
            for (int i = 0; i < TPC; i += 2) {
                mma_bf16_16816(d0, a0, i, 7u);
                mma_bf16_16816(d1, a1, 5u, i);
            }
            if (d0[0] + d1[1] == 1234.5f) acc[lane] = 1.f;
        } else if (MODE != 3) {
            const int t0 = c * TPC;
            int done = 0;
            while (done < TPC) {
                const int tt = t0 + done;
                const int rtile = tt / kst, j = tt - rtile * kst;
                const int len = (kst - j < TPC - done) ? kst - j : TPC - done;
                float d0[4] = {0.f, 0.f, 0.f, 0.f}, d1[4] = {0.f, 0.f, 0.f, 0.f};
                const uint4* ap = reinterpret_cast<const uint4*>(buf + done * 512) + lane;
                const uint16_t* xp = xrow + j * 16;
#pragma unroll 4
                for (int i = 0; i < len; i += 2) {
                    const uint4 a0 = lds128(ap + i * 32);
                    const uint4 a1 = lds128(ap + (i + 1) * 32);
                    const uint4 xv = xlane ? lds128(xp + i * 16) : make_uint4(0u, 0u, 0u, 0u);
                    mma_bf16_16816(d0, a0, xv.x, xv.y);
                    mma_bf16_16816(d1, a1, xv.z, xv.w);
                }
                const int row = (rtile * 16 + g) & 4095;
                if (q == 0) {
                    atomicAdd(&acc[row], d0[0] + d1[0]);
                    atomicAdd(&acc[(row + 8) & 4095], d0[2] + d1[2]);
                }
                done += len;
            }
        }
        __syncwarp();
        if (lane == 0 && MODE != 0) mbar_arrive(&empty[st]);
    }
    asm volatile("bar.sync 1, 256;");
    if (threadIdx.x == 0) {
        float s = 0.f;
        for (int i = 0; i < 4096; ++i) s += acc[i];
        atomicAdd(out, s);
        atomicAdd(cyc, static_cast<unsigned long long>(clock64() - t_start));
    }
}

template <int MODE>
void run(const uint8_t* W, float* out, unsigned long long* cyc, int ctas, long long per_cta, int K) {
    const int smem = STAGES * CHUNK + K * 2 + 4096 * 4 + 2 * STAGES * 8 + 128;
    cudaFuncSetAttribute(bench_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int it = 0; it < 5; ++it) {
        cudaEventRecord(a);
        bench_kernel<MODE><<<ctas, 320, smem>>>(W, per_cta, K, out, cyc);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (it > 0 && ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    printf("mode=%d K=%5d ctas=%3d: %8.1f us  %7.1f GB/s total  %6.1f GB/s per CTA %s\n", MODE, K, ctas, best * 1e3,
           ctas * per_cta / (best * 1e-3) / 1e9, per_cta / (best * 1e-3) / 1e9,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    const long long per_cta = 6LL * 1024 * 1024 / CHUNK * CHUNK;
    const long long total = 148 * per_cta + (1 << 20);
    uint8_t* W;
    float* out;
    unsigned long long* cyc;
    cudaMalloc(&W, total);
    cudaMalloc(&out, 4);
    cudaMalloc(&cyc, 8);
    cudaMemset(W, 0, total);
    for (int K : {4096}) {
        for (int ctas : {1, 148}) {
            run<0>(W, out, cyc, ctas, per_cta, K);
            run<1>(W, out, cyc, ctas, per_cta, K);
            run<2>(W, out, cyc, ctas, per_cta, K);
            run<3>(W, out, cyc, ctas, per_cta, K);
            run<4>(W, out, cyc, ctas, per_cta, K);
            run<5>(W, out, cyc, ctas, per_cta, K);
            run<6>(W, out, cyc, ctas, per_cta, K);
            run<8>(W, out, cyc, ctas, per_cta, K);
            run<9>(W, out, cyc, ctas, per_cta, K);
            run<10>(W, out, cyc, ctas, per_cta, K);
        }
    }
    return 0;
}
