// tools/mb/alu.cu -- integer pipe throughput on this part: 3-input LOP3 (the
// bitsliced-AES gate), PRMT and IMAD, in lane-ops per clock per SM.  Grounds
// the bitsliced-AES estimate of DESIGN.md 11.
#include <cuda_runtime.h>
#include <cstdint>

template <int OP>
__global__ void __launch_bounds__(1024, 1) alu(uint32_t* sink, int iters, uint32_t k1, uint32_t k2) {
    uint32_t a[16];
#pragma unroll
    for (int c = 0; c < 16; c++) a[c] = threadIdx.x * 2654435761u + c;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int c = 0; c < 16; c++) {
            uint32_t b = a[(c + 1) & 15], d = a[(c + 5) & 15];
            if (OP == 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[c]) : "r"(b), "r"(d));
            if (OP == 1) a[c] = __byte_perm(a[c], b, 0x5140);
            if (OP == 2) a[c] = a[c] * k1 + b;
            if (OP == 3) a[c] = __umulhi(a[c], k1) + b;                    // IMAD.HI
            if (OP == 4) a[c] = __funnelshift_l(a[c], b, 7);              // SHF.L.W
            if (OP == 5) {                                                 // IMAD.WIDE.U32: lo / hi pair
                const uint64_t p = (uint64_t)a[c] * k1 + (uint64_t)k2;
                a[c] = (uint32_t)p + (uint32_t)(p >> 32) * k2;            // + one IMAD
            }
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < 16; c++) acc ^= a[c];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

extern "C" int alu_run(uint32_t* sink, int grid, int iters, float* out) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int op = 0; op < 6; op++) {
        for (int r = 0; r < 2; r++) {
            cudaEventRecord(e0);
            if (op == 0) alu<0><<<grid, 1024>>>(sink, iters, 3, 5);
            if (op == 1) alu<1><<<grid, 1024>>>(sink, iters, 3, 5);
            if (op == 2) alu<2><<<grid, 1024>>>(sink, iters, 3, 5);
            if (op == 3) alu<3><<<grid, 1024>>>(sink, iters, 3, 5);
            if (op == 4) alu<4><<<grid, 1024>>>(sink, iters, 3, 5);
            if (op == 5) alu<5><<<grid, 1024>>>(sink, iters, 3, 5);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&out[op], e0, e1);
        }
    }
    return (int)cudaGetLastError();
}
