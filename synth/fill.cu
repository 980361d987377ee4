// synth/fill.cu -- seeded synthetic-input generator, device side.
//
// Shared by tests and bench for BOTH the oracle and the CUDA AES path; it holds
// none of the method's arithmetic (no AES, no GF(2^8)): it only writes the
// splitmix64 counter-based stream defined in DESIGN.md "Input recipe"
// (SURVEY.md 8(d)).  The host twin is synth/__init__.py (numpy); the two are
// checked against each other in tests/test_synth.py.
//
// u64 word m of stream `seed`:
//   z = seed + (m+1)*0x9E3779B97F4A7C15; z = (z^(z>>30))*0xBF58476D1CE4E5B9;
//   z = (z^(z>>27))*0x94D049BB133111EB; word = z^(z>>31)
// Block i of a buffer = words 2i, 2i+1, little-endian.
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t splitmix(uint64_t seed, uint64_t m) {
    uint64_t z = seed + (m + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// kind 0: uniform random; 1: all zero; 2: one repeated 16-byte block (block 0 of
// the stream); 3: ASCII-like bytes in 0x20..0x7E (each byte = 0x20 + b % 95).
__global__ void splitmix_fill_kernel(ulonglong2* __restrict__ out, uint64_t first_block,
                                     uint64_t nblocks, uint64_t seed, int kind) {
    uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nblocks; i += stride) {
        uint64_t g = (kind == 2) ? 0 : first_block + i;
        ulonglong2 v;
        if (kind == 1) { v.x = 0; v.y = 0; }
        else { v.x = splitmix(seed, 2 * g); v.y = splitmix(seed, 2 * g + 1); }
        if (kind == 3) {
            uint64_t a = 0, b = 0;
            for (int k = 0; k < 8; k++) {
                a |= (uint64_t)(0x20 + ((v.x >> (8 * k)) & 0xFF) % 95) << (8 * k);
                b |= (uint64_t)(0x20 + ((v.y >> (8 * k)) & 0xFF) % 95) << (8 * k);
            }
            v.x = a; v.y = b;
        }
        out[i] = v;
    }
}

extern "C" int synth_fill(void* dev, uint64_t first_block, uint64_t nblocks, uint64_t seed,
                          int kind, void* stream) {
    if (nblocks == 0) return 0;
    if (!dev || ((uintptr_t)dev & 15)) return 1;
    int dev_id = 0, nsm = 148;
    cudaGetDevice(&dev_id);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev_id);
    uint64_t want = (nblocks + 255) / 256;
    unsigned grid = (unsigned)(want < (uint64_t)nsm * 16 ? want : (uint64_t)nsm * 16);
    splitmix_fill_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>((ulonglong2*)dev, first_block,
                                                                 nblocks, seed, kind);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
