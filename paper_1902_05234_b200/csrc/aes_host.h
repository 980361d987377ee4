// aes_host.h -- host-side helpers shared by the TUs of libaes_b200.so:
// kernel registry entries, per-device attribute cache, descriptor pool,
// argument validation, CUDA error capture.  Defined in aes_runtime.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "aes_b200.h"

namespace aesb200 {

struct KernelInfo {
    const void* fn;
    size_t smem;
};

constexpr int kMaxDev = 64;
constexpr int kThreads = 1024;   // every kernel runs 1024-thread CTAs (one per SM)

aes_status cuda_fail(cudaError_t e);                       // records e for aes_last_cuda_error()
aes_status resident_ctas(int dev, const KernelInfo& ki, int* occ, int* nsm);   // sets smem attr once
aes_status launch_kernel(const KernelInfo& ki, unsigned grid, void** args, cudaStream_t stream, bool pdl);
aes_status desc_pool(int dev, cudaMemPool_t* out);         // stream-ordered pool for descriptors
aes_status stage_h2d(int dev, void* dst, const void* src, size_t bytes, cudaStream_t s);   // pinned ring, async H2D
aes_status validate_keys(const aes_round_keys* rk, int nr);
aes_status validate_buffers(const void* in, const void* out, uint64_t nblocks);
aes_status check_device_ptr(const void* p, int dev);
// Hybrid / bitsliced kernels (aes_hybrid.cu): kernel args (in, out, n, RK, BSK, ModeP)
struct BSK;
KernelInfo pick_hybrid(int nr, bool dec, int variant, int mode);   // V_HYBRID (any mode) or V_BITSLICE (ECB)
void bitslice_keys(const aes_round_keys* rk, int decrypt, BSK* out);
// ECB launch used by the host pipeline (aes_ecb.cu)
aes_status launch_ecb(const aes_round_keys* rk, int nr, int decrypt, const void* in, void* out, uint64_t nblocks,
                      cudaStream_t stream, bool check_ptrs);

}  // namespace aesb200
