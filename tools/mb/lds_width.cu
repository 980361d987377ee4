// tools/mb/lds_width.cu -- microbenchmarks behind DESIGN.md 11 "Why there is no
// further kernel headroom": per-lane random gathers from lane-replicated
// shared-memory tables with 32-, 64- and 128-bit loads (is the limit addresses
// per clock or bytes per clock?), and the same gather from __constant__ memory
// (the paper's table placement) and from L1-resident global memory.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
#include <cuda_runtime.h>
#include <cstdint>

constexpr int kThreads = 1024;
__constant__ uint32_t c_tab[1024];

template <int W>   // W = words per lane per load (1, 2, 4)
__global__ void __launch_bounds__(kThreads, 1) lds_gather(uint32_t* sink, int iters) {
    extern __shared__ __align__(16) uint32_t smem[];
    // 256 entries x 32 lanes x W words, bank group = lane: entry x, lane L at word (x*32 + L)*W
    for (int w = threadIdx.x; w < 256 * 32 * W; w += blockDim.x) smem[w] = w * 2654435761u;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    uint32_t a[16];
#pragma unroll
    for (int c = 0; c < 16; c++) a[c] = threadIdx.x * 7919u + c * 104729u + blockIdx.x;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int c = 0; c < 16; c++) {
            uint32_t idx = ((a[c] & 255u) * 32u + lane) * W;
            if (W == 1) a[c] ^= smem[idx];
            if (W == 2) { uint2 v = *reinterpret_cast<const uint2*>(smem + idx); a[c] ^= v.x + v.y; }
            if (W == 4) { uint4 v = *reinterpret_cast<const uint4*>(smem + idx); a[c] ^= v.x + v.y + v.z + v.w; }
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < 16; c++) acc ^= a[c];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void __launch_bounds__(kThreads, 1) const_gather(uint32_t* sink, int iters) {
    uint32_t a[8];
#pragma unroll
    for (int c = 0; c < 8; c++) a[c] = threadIdx.x * 7919u + c * 104729u + blockIdx.x;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int c = 0; c < 8; c++) a[c] ^= c_tab[a[c] & 1023u];
    }
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < 8; c++) acc ^= a[c];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void __launch_bounds__(kThreads, 1) l1_gather(const uint32_t* __restrict__ tab, uint32_t* sink, int iters) {
    uint32_t a[16];
#pragma unroll
    for (int c = 0; c < 16; c++) a[c] = threadIdx.x * 7919u + c * 104729u + blockIdx.x;
    const uint32_t lane = threadIdx.x & 31;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int c = 0; c < 16; c++) a[c] ^= __ldg(tab + (a[c] & 255u) * 32u + lane);   // 32 KiB, L1-resident
    }
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < 16; c++) acc ^= a[c];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

extern "C" int mb_run(int kind, void* sink, const void* tab, int grid, int iters, float* ms) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    size_t sm = kind == 1 ? 256 * 32 * 4 : kind == 2 ? 256 * 32 * 8 : kind == 4 ? 256 * 32 * 16 : 0;
    cudaFuncSetAttribute((const void*)lds_gather<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 256 * 32 * 4);
    cudaFuncSetAttribute((const void*)lds_gather<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 256 * 32 * 8);
    cudaFuncSetAttribute((const void*)lds_gather<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 256 * 32 * 16);
    for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(e0);
        uint32_t* s = (uint32_t*)sink;
        if (kind == 1) lds_gather<1><<<grid, kThreads, sm>>>(s, iters);
        else if (kind == 2) lds_gather<2><<<grid, kThreads, sm>>>(s, iters);
        else if (kind == 4) lds_gather<4><<<grid, kThreads, sm>>>(s, iters);
        else if (kind == 10) const_gather<<<grid, kThreads>>>(s, iters);
        else if (kind == 11) l1_gather<<<grid, kThreads>>>((const uint32_t*)tab, s, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return (int)cudaGetLastError();
}
