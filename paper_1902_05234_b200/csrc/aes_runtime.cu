// aes_runtime.cu -- host runtime of libaes_b200.so: CUDA error capture,
// the per-device launch-attribute cache, the PDL launch helper, the descriptor
// memory pool and staging ring, argument
// validation (everything decided before a launch, include/aes_b200.h "Errors"),
// status strings.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <shared_mutex>
#include <unordered_map>

#include "aes_b200.h"
#include "aes_host.h"

namespace aesb200 {

thread_local int t_last_cuda_error = 0;

aes_status cuda_fail(cudaError_t e) {
    t_last_cuda_error = (int)e;
    return AES_ECUDA;
}

// Per-(device, kernel) resident-CTA count; the dynamic-smem attribute is set
// once per (device, kernel) under the write lock, later calls take a shared lock.
std::shared_mutex g_attr_mu;
std::unordered_map<const void*, int> g_occ[kMaxDev];
int g_nsm[kMaxDev];

aes_status resident_ctas(int dev, const KernelInfo& ki, int* occ, int* nsm) {
    if (dev < 0 || dev >= kMaxDev) return AES_ERANGE;
    {
        std::shared_lock<std::shared_mutex> rd(g_attr_mu);
        auto it = g_occ[dev].find(ki.fn);
        if (it != g_occ[dev].end()) {
            *occ = it->second;
            *nsm = g_nsm[dev];
            return AES_OK;
        }
    }
    std::unique_lock<std::shared_mutex> wr(g_attr_mu);
    if (!g_nsm[dev]) {
        int v = 0;
        cudaError_t e = cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return cuda_fail(e);
        g_nsm[dev] = v;
    }
    *nsm = g_nsm[dev];
    auto it = g_occ[dev].find(ki.fn);
    if (it != g_occ[dev].end()) {
        *occ = it->second;
        return AES_OK;
    }
    cudaError_t e = cudaFuncSetAttribute(ki.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ki.smem);
    if (e != cudaSuccess) return cuda_fail(e);
    int o = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, ki.fn, kThreads, ki.smem);
    if (e != cudaSuccess) return cuda_fail(e);
    if (o < 1) o = 1;
    g_occ[dev].emplace(ki.fn, o);
    *occ = o;
    return AES_OK;
}

// One kernel launch of kThreads-thread CTAs, with the programmatic-dependent-
// launch attribute unless pdl == false (aes_device.cuh: every kernel fills its
// tables before griddepcontrol.wait).
aes_status launch_kernel(const KernelInfo& ki, unsigned grid, void** args, cudaStream_t stream, bool pdl) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(kThreads);
    lc.dynamicSmemBytes = ki.smem;
    lc.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = pdl ? 1 : 0;
    cudaError_t e = cudaLaunchKernelExC(&lc, ki.fn, args);
    return e == cudaSuccess ? AES_OK : cuda_fail(e);
}

// A library-owned stream-ordered memory pool per device for small per-call
// descriptors (aes_ecb_batch): memory stays cached between calls (a release
// threshold of 64 MiB) instead of being unmapped at every synchronisation as
// with the default pool's threshold of 0; torch's allocator is not touched.
std::mutex g_pool_mu;
cudaMemPool_t g_pool[kMaxDev];

aes_status desc_pool(int dev, cudaMemPool_t* out) {
    if (dev < 0 || dev >= kMaxDev) return AES_ERANGE;
    std::lock_guard<std::mutex> g(g_pool_mu);
    if (!g_pool[dev]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t p;
        cudaError_t e = cudaMemPoolCreate(&p, &props);
        if (e != cudaSuccess) return cuda_fail(e);
        uint64_t keep = 64ull << 20;
        cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep);
        g_pool[dev] = p;
    }
    *out = g_pool[dev];
    return AES_OK;
}

// Page-locked staging for small host->device descriptor copies (cudaMemcpyAsync
// from pageable memory is synchronous, from pinned memory a plain async DMA).
// A process-wide ring of kSlots slots per device: a call takes the next slot
// whose previous copy has completed (cudaEventQuery, no blocking), and only
// blocks -- on that slot's own event -- when all kSlots copies are still queued.
// Slots are released at process exit.
constexpr int kSlots = 16;
struct Slot {
    void* host = nullptr;
    size_t cap = 0;
    cudaEvent_t ev = nullptr;
};
struct StageRing {
    std::mutex mu;
    Slot slot[kSlots];
    unsigned next = 0;
    ~StageRing() {
        for (Slot& s : slot) {
            if (s.ev) cudaEventDestroy(s.ev);
            if (s.host) cudaFreeHost(s.host);
        }
    }
};
StageRing g_stage[kMaxDev];

aes_status stage_h2d(int dev, void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (dev < 0 || dev >= kMaxDev) return AES_ERANGE;
    StageRing& r = g_stage[dev];
    std::lock_guard<std::mutex> g(r.mu);
    cudaError_t e;
    int pick = -1;
    for (int k = 0; k < kSlots && pick < 0; k++) {
        const int c = (int)((r.next + k) % kSlots);
        if (!r.slot[c].ev) { pick = c; break; }
        e = cudaEventQuery(r.slot[c].ev);
        if (e == cudaSuccess) pick = c;
        else if (e != cudaErrorNotReady) return cuda_fail(e);
    }
    if (pick < 0) {   // every slot's copy still queued: wait for the oldest
        pick = (int)(r.next % kSlots);
        if ((e = cudaEventSynchronize(r.slot[pick].ev)) != cudaSuccess) return cuda_fail(e);
    }
    r.next = (unsigned)pick + 1;
    Slot& st = r.slot[pick];
    if (st.cap < bytes) {
        if (st.host) cudaFreeHost(st.host);
        st.host = nullptr;
        st.cap = 0;
        size_t cap = bytes < (64u << 10) ? (64u << 10) : 2 * bytes;
        if ((e = cudaHostAlloc(&st.host, cap, cudaHostAllocDefault)) != cudaSuccess) return cuda_fail(e);
        st.cap = cap;
    }
    if (!st.ev && (e = cudaEventCreateWithFlags(&st.ev, cudaEventDisableTiming)) != cudaSuccess) return cuda_fail(e);
    std::memcpy(st.host, src, bytes);
    if ((e = cudaMemcpyAsync(dst, st.host, bytes, cudaMemcpyHostToDevice, s)) != cudaSuccess) return cuda_fail(e);
    if ((e = cudaEventRecord(st.ev, s)) != cudaSuccess) return cuda_fail(e);
    return AES_OK;
}

aes_status validate_keys(const aes_round_keys* rk, int nr) {
    if (!rk) return AES_ENULL;
    if ((nr != 10 && nr != 12 && nr != 14) || rk->nr != nr || rk->keybits != 32 * (nr - 6)) return AES_ENR;
    return AES_OK;
}

aes_status validate_buffers(const void* in, const void* out, uint64_t nblocks) {
    if (!in || !out) return AES_ENULL;
    if (nblocks > (UINT64_MAX >> 4)) return AES_ERANGE;
    uint64_t bytes = nblocks << 4;
    uintptr_t a = (uintptr_t)in, b = (uintptr_t)out;
    if ((a | b) & 15) return AES_EALIGN;
    if (a > UINTPTR_MAX - bytes || b > UINTPTR_MAX - bytes) return AES_ERANGE;
    if (a != b && a < b + bytes && b < a + bytes) return AES_EOVERLAP;
    return AES_OK;
}

aes_status check_device_ptr(const void* p, int dev) {
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return cuda_fail(e);
    }
    if ((at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged) || at.device != dev)
        return AES_ENOTDEVICE;
    return AES_OK;
}

}  // namespace aesb200

extern "C" {

const char* aes_status_string(aes_status s) {
    switch (s) {
        case AES_OK: return "AES_OK";
        case AES_EKEYBITS: return "AES_EKEYBITS: keybits must be 128, 192 or 256";
        case AES_ENR: return "AES_ENR: nr must be 10/12/14 and match the round keys";
        case AES_ENULL: return "AES_ENULL: required pointer is NULL";
        case AES_EALIGN: return "AES_EALIGN: buffers must be 16-byte aligned";
        case AES_EOVERLAP: return "AES_EOVERLAP: in and out partially overlap";
        case AES_ERANGE: return "AES_ERANGE: size or configuration out of range";
        case AES_ENOTDEVICE: return "AES_ENOTDEVICE: buffer is not device memory of the current device";
        case AES_ECUDA: return "AES_ECUDA: CUDA runtime error (see aes_last_cuda_error)";
        case AES_EVARIANT: return "AES_EVARIANT: unknown kernel variant or states_per_thread";
        case AES_ECAPTURE: return "AES_ECAPTURE: aes_ecb_batch cannot be captured into a CUDA graph";
    }
    return "AES_?: unknown status";
}

int aes_last_cuda_error(void) { return aesb200::t_last_cuda_error; }
int aes_abi_version(void) { return AES_B200_ABI_VERSION; }

}  // extern "C"

