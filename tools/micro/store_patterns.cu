// Store-pattern microbenchmark for the memo key stream (dev tool):
// writes N u64 keys (3.83 GB = 12! keys) with different warp store layouts.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o store_patterns store_patterns.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr uint64_t N = 479001600ull, DF = 120, RUNS = N / DF;

// (1) fill-like: grid-stride, 16 B per lane, full warps
__global__ void k_fill(uint64_t* k) {
    const uint64_t n2 = N / 2;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n2; i += (uint64_t)gridDim.x * blockDim.x)
        __stcs(reinterpret_cast<ulonglong2*>(k) + i, make_ulonglong2(i, i + 1));
}
// (2) the key stream's layout: a warp owns 32 consecutive runs; per step two runs, a half-warp each,
// lane hl (15 of 16) stores 16 B at run offset 16*hl + 240*q, q = 0..3. CS = streaming stores.
template <bool CS>
__global__ void k_half(uint64_t* k) {
    const uint32_t lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
    const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5, nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t base = gw * 32; base < RUNS; base += nw * 32) {
        const uint32_t nr = (uint32_t)min((uint64_t)32, RUNS - base);
        for (uint32_t i0 = 0; i0 < nr; i0 += 2) {
            const uint32_t i = i0 + half;
            if (i < nr && hl < 15) {
                uint64_t* o = k + (base + i) * DF + 2 * hl;
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    ulonglong2 v = make_ulonglong2(base + i, q);
                    if (CS) __stcs(reinterpret_cast<ulonglong2*>(o + 30 * q), v);
                    else *reinterpret_cast<ulonglong2*>(o + 30 * q) = v;
                }
            }
        }
    }
}
// (3) full-warp contiguous over the step's 2 runs (1920 B): lane l stores pair p = l + 32q (p < 120)
__global__ void k_full2(uint64_t* k) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5, nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t base = gw * 32; base < RUNS; base += nw * 32) {
        const uint32_t nr = (uint32_t)min((uint64_t)32, RUNS - base);
        for (uint32_t i0 = 0; i0 < nr; i0 += 2) {
            const uint32_t pairs = (min(nr - i0, 2u)) * 60;
            uint64_t* o = k + (base + i0) * DF;
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const uint32_t p = lane + 32 * q;
                if (p < pairs) __stcs(reinterpret_cast<ulonglong2*>(o) + p, make_ulonglong2(base, p));
            }
        }
    }
}
// (4) full-warp contiguous over the warp's whole 32-run block (30 KB), 16 B per lane per instruction
__global__ void k_block(uint64_t* k) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5, nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t base = gw * 32; base < RUNS; base += nw * 32) {
        const uint32_t nr = (uint32_t)min((uint64_t)32, RUNS - base);
        const uint32_t pairs = nr * 60;
        ulonglong2* o = reinterpret_cast<ulonglong2*>(k + base * DF);
        for (uint32_t p = lane; p < pairs; p += 32) __stcs(o + p, make_ulonglong2(base, p));
    }
}

// fill variants: default (write-back) stores; 32-B stores; one-shot grid with 4 x 16 B per thread
__global__ void k_fill_wb(uint64_t* k) {
    const uint64_t n2 = N / 2;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n2; i += (uint64_t)gridDim.x * blockDim.x)
        reinterpret_cast<ulonglong2*>(k)[i] = make_ulonglong2(i, i + 1);
}
__device__ __forceinline__ void st256(uint64_t* p, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}
__global__ void k_fill256(uint64_t* k) {
    const uint64_t n4 = N / 4;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x)
        st256(k + 4 * i, i, i, i, i);
}
__global__ void k_fill_oneshot(uint64_t* k) {  // grid = N/2/(256*4)
    const uint64_t b = (blockIdx.x * (uint64_t)blockDim.x) * 4 + threadIdx.x;
#pragma unroll
    for (int j = 0; j < 4; j++) {
        const uint64_t i = b + j * blockDim.x;
        if (i < N / 2) reinterpret_cast<ulonglong2*>(k)[i] = make_ulonglong2(i, j);
    }
}
// full2 with 32-B stores: lane l stores quad p = l + 32q of the step's 60 quads
__global__ void k_full2_256(uint64_t* k) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5, nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t base = gw * 32; base < RUNS; base += nw * 32) {
        const uint32_t nr = (uint32_t)min((uint64_t)32, RUNS - base);
        for (uint32_t i0 = 0; i0 < nr; i0 += 2) {
            const uint32_t quads = (min(nr - i0, 2u)) * 30;
            uint64_t* o = k + (base + i0) * DF;
#pragma unroll
            for (int q = 0; q < 2; q++) {
                const uint32_t p = lane + 32 * q;
                if (p < quads) st256(o + 4 * p, base, p, q, 0);
            }
        }
    }
}

// one-shot grids (CTAs in index order sweep memory once): each warp owns RPW consecutive runs
template <int RPW>
__global__ void k_half_oneshot(uint64_t* k) {
    const uint32_t lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
    const uint64_t base = ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5) * RPW;
    if (base >= RUNS) return;
    const uint32_t nr = (uint32_t)min((uint64_t)RPW, RUNS - base);
    for (uint32_t i0 = 0; i0 < nr; i0 += 2) {
        const uint32_t i = i0 + half;
        if (i < nr && hl < 15) {
            uint64_t* o = k + (base + i) * DF + 2 * hl;
#pragma unroll
            for (int q = 0; q < 4; q++) __stcs(reinterpret_cast<ulonglong2*>(o + 30 * q), make_ulonglong2(base + i, q));
        }
    }
}
template <int RPW>
__global__ void k_full2_oneshot(uint64_t* k) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t base = ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5) * RPW;
    if (base >= RUNS) return;
    const uint32_t nr = (uint32_t)min((uint64_t)RPW, RUNS - base);
    for (uint32_t i0 = 0; i0 < nr; i0 += 2) {
        const uint32_t pairs = (min(nr - i0, 2u)) * 60;
        uint64_t* o = k + (base + i0) * DF;
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const uint32_t p = lane + 32 * q;
            if (p < pairs) __stcs(reinterpret_cast<ulonglong2*>(o) + p, make_ulonglong2(base, p));
        }
    }
}

template <class F>
float timeit(F f, int reps = 10) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < reps; i++) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main() {
    uint64_t* k;
    cudaMalloc(&k, N * 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int per : {2, 4, 8}) {
        const int g = sms * per;
        printf("ctas/SM %d: fill %.3f  half_cs %.3f  half_wb %.3f  full2 %.3f  block %.3f ms\n", per,
               timeit([&] { k_fill<<<g, 256>>>(k); }), timeit([&] { k_half<true><<<g, 256>>>(k); }),
               timeit([&] { k_half<false><<<g, 256>>>(k); }), timeit([&] { k_full2<<<g, 256>>>(k); }),
               timeit([&] { k_block<<<g, 256>>>(k); }));
    }
    printf("fill_wb %.3f fill256 %.3f oneshot %.3f\n", timeit([&] { k_fill_wb<<<sms * 8, 256>>>(k); }),
           timeit([&] { k_fill256<<<sms * 8, 256>>>(k); }),
           timeit([&] { k_fill_oneshot<<<(unsigned)((N / 2 + 1023) / 1024), 256>>>(k); }));
    for (int per : {2, 4, 8}) printf("full2_256 ctas/SM %d: %.3f\n", per, timeit([&] { k_full2_256<<<sms * per, 256>>>(k); }));
#define ONESHOT(R) printf("oneshot runs/warp %d: half %.3f full2 %.3f\n", R, \
        timeit([&] { k_half_oneshot<R><<<(unsigned)((RUNS + 8 * R - 1) / (8 * R)), 256>>>(k); }), \
        timeit([&] { k_full2_oneshot<R><<<(unsigned)((RUNS + 8 * R - 1) / (8 * R)), 256>>>(k); }));
    ONESHOT(2) ONESHOT(4) ONESHOT(8) ONESHOT(16) ONESHOT(32)
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
