// Compact key stream microbenchmark (dev tool): 12! u32 keys (1.92 GB) written
// in 480-B runs, 8 runs per warp, one-shot grid (the rk_dp_keys32_kernel layout), with
// (a) constant values, (b) values = run base + 16-B loads from a 20-MB L2-resident offsets
// table (the real kernel's reads), (c) a plain fill-like grid-stride stream.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o store32 store32.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr uint64_t N = 479001600ull, DF = 120, RUNS = N / DF, NODES = 42706;
constexpr uint32_t RPW = 8, CH = 30;

template <bool LOAD>
__global__ void k_runs(uint32_t* k, const uint32_t* offs) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t base = ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5) * RPW;
    if (base >= RUNS) return;
    const uint32_t myu = (uint32_t)((base + lane) * 2654435761ull % NODES);
#pragma unroll
    for (uint32_t s = 0; s < RPW / 2; s++)
#pragma unroll
        for (int q = 0; q < 2; q++) {
            const uint32_t p = lane + 32u * q, r = 2u * s + (p < CH ? 0u : 1u);
            const uint32_t u = __shfl_sync(0xFFFFFFFFu, myu, r);
            if (p >= 2u * CH || base + r >= RUNS) continue;
            uint4 v = make_uint4(u, u, u, u);
            if (LOAD) {
                const uint4 o = __ldg(reinterpret_cast<const uint4*>(offs + (uint64_t)u * DF) + (p < CH ? p : p - CH));
                v = make_uint4(u + o.x, u + o.y, u + o.z, u + o.w);
            }
            __stcs(reinterpret_cast<uint4*>(k + (base + 2 * s) * DF) + p, v);
        }
}
__global__ void k_fill(uint32_t* k) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N / 4; i += (uint64_t)gridDim.x * blockDim.x)
        __stcs(reinterpret_cast<uint4*>(k) + i, make_uint4(i, i, i, i));
}

int main() {
    uint32_t *k, *offs;
    cudaMalloc(&k, N * 4);
    cudaMalloc(&offs, NODES * DF * 4);
    cudaMemset(offs, 1, NODES * DF * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const unsigned grid = (unsigned)((RUNS + 8 * RPW - 1) / (8 * RPW));
    auto t = [&](auto launch, const char* name) {
        launch();
        cudaDeviceSynchronize();
        float best = 1e9;
        for (int r = 0; r < 10; r++) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        printf("%-28s %.4f ms  %.2f TB/s\n", name, best, N * 4 / (best * 1e-3) / 1e12);
    };
    t([&] { k_runs<false><<<grid, 256>>>(k, offs); }, "runs, constant values");
    t([&] { k_runs<true><<<grid, 256>>>(k, offs); }, "runs, offsets from L2");
    t([&] { k_fill<<<148 * 8, 256>>>(k); }, "fill grid-stride 16B");
    t([&] { k_fill<<<(unsigned)(N / 4 / 256), 256>>>(k); }, "fill one-shot 16B");
    t([&] { cudaMemsetAsync(k, 1, N * 4); }, "cudaMemset");
    return 0;
}
