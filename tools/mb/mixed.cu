// tools/mb/mixed.cu -- is any other lookup path additive to the shared-memory
// gather?  Each thread runs 16 LDS chains per iteration plus E extra chains
// that look up through (kind 0) more LDS, (kind 1) L1-resident global loads,
// (kind 2) the texture path (tex1Dfetch).  If the extra chains cost no time
// on top of the 16 LDS chains, that path is independent of the LDS data path.
#include <cuda_runtime.h>
#include <cstdint>

constexpr int kThreads = 1024;

template <int KIND, int E>
__global__ void __launch_bounds__(kThreads, 1) mixed(const uint32_t* __restrict__ gtab, cudaTextureObject_t tex,
                                                      uint32_t* sink, int iters) {
    extern __shared__ __align__(16) uint32_t smem[];
    for (int w = threadIdx.x; w < 256 * 64; w += blockDim.x) smem[w] = w * 2654435761u;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    const char* sb = reinterpret_cast<const char*>(smem);
    uint32_t a[16], b[E > 0 ? E : 1];
#pragma unroll
    for (int c = 0; c < 16; c++) a[c] = threadIdx.x * 7919u + c * 104729u + blockIdx.x;
#pragma unroll
    for (int c = 0; c < E; c++) b[c] = threadIdx.x * 31u + c * 977u;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int c = 0; c < 16; c++)
            a[c] = *reinterpret_cast<const uint32_t*>(sb + __byte_perm(lane * 4, a[c], 0x1140));
#pragma unroll
        for (int c = 0; c < E; c++) {
            uint32_t idx = (b[c] & 255u) * 32u + lane;
            if (KIND == 0) b[c] ^= *reinterpret_cast<const uint32_t*>(sb + __byte_perm(lane * 4, b[c], 0x1150));
            if (KIND == 1) b[c] ^= __ldg(gtab + idx);
            if (KIND == 2) b[c] ^= tex1Dfetch<unsigned int>(tex, (int)idx);
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < 16; c++) acc ^= a[c];
#pragma unroll
    for (int c = 0; c < E; c++) acc ^= b[c];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int KIND, int E>
float run(const uint32_t* gtab, cudaTextureObject_t tex, uint32_t* sink, int grid, int iters) {
    cudaFuncSetAttribute((const void*)mixed<KIND, E>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaGetLastError();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms = 0;
    for (int r = 0; r < 2; r++) {
        cudaEventRecord(e0);
        mixed<KIND, E><<<grid, kThreads, 65536>>>(gtab, tex, sink, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
    }
    cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return err == cudaSuccess ? ms : -(float)err;
}

extern "C" int mixed_run(const uint32_t* gtab, uint32_t* sink, int grid, int iters, float* out) {
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = (void*)gtab;
    rd.res.linear.desc = cudaCreateChannelDesc<unsigned int>();
    rd.res.linear.sizeInBytes = 256 * 32 * 4;
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tex = 0;
    cudaCreateTextureObject(&tex, &rd, &td, nullptr);
    out[0] = run<0, 0>(gtab, tex, sink, grid, iters);
    out[1] = run<0, 2>(gtab, tex, sink, grid, iters);
    out[2] = run<0, 4>(gtab, tex, sink, grid, iters);
    out[3] = run<1, 2>(gtab, tex, sink, grid, iters);
    out[4] = run<1, 4>(gtab, tex, sink, grid, iters);
    out[5] = run<2, 2>(gtab, tex, sink, grid, iters);
    out[6] = run<2, 4>(gtab, tex, sink, grid, iters);
    cudaDestroyTextureObject(tex);
    return (int)cudaGetLastError();
}
