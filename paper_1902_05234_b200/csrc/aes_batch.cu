// aes_batch.cu -- batched multi-message ECB (aes_ecb_batch): many messages,
// each with its own key, in one launch (DESIGN.md section 11 "Batched small messages").
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <vector>

#include "aes_b200.h"
#include "aes_device.cuh"
#include "aes_host.h"

namespace aesb200 {

// ---------------------------------------------------------------------------
// Batched multi-message ECB (aes_ecb_batch): many messages, each with its own
// key, in ONE launch -- the paper's file-sized workloads at
// bulk rate instead of one launch per file.  Segment s covers global blocks
// [first, first + n); a warp's 32 consecutive global blocks find their
// segment with one warp-uniform binary search (broadcast loads) plus a short
// forward walk.  The key schedules travel BY VALUE in the kernel parameters
// (constant bank, up to 128 x 240 B): per round a message's round key is an
// LDC broadcast through the constant cache -- no shared-memory/L1TEX
// traffic, which is the resource the T-table rounds saturate.
// ---------------------------------------------------------------------------
struct BatchSeg {
    uint64_t in_off, out_off;   // byte offsets from in_base / out_base
    uint64_t first, n;          // global block range
    uint32_t key, pad;          // index into the key words (60 per key)
};

template <int KCAP>
struct BatchKeys {
    uint32_t w[KCAP * 60];   // ek (or dk) of key k at w[60k .. 60k + 4(NR+1))
};

constexpr int kBatchMaxKeys = 128;   // 128 x 240 B = 30 KiB of kernel parameters (limit 32,764 B)

template <int KCAP>
struct KeyParamAt {
    const BatchKeys<KCAP>& ks;
    uint32_t base;   // 60 * key + 4 * round
    __device__ __forceinline__ uint32_t operator[](int j) const { return ks.w[base + j]; }
};

// Each CTA owns one contiguous range of global blocks; its 1024 threads walk it
// 1024 consecutive blocks per trip, so the segment of a warp only moves
// forward: found once by a warp-uniform binary search, then advanced by a
// short forward walk (broadcast loads).
template <int NR, bool DEC, int KCAP>
__global__ void __launch_bounds__(kThreads, 1)
    batch_kernel(const char* __restrict__ in_base, char* __restrict__ out_base, const BatchSeg* __restrict__ segs,
                 uint32_t nsegs, uint64_t total, const __grid_constant__ BatchKeys<KCAP> keys) {
    extern __shared__ __align__(16) uint32_t smem[];
    pdl_launch_dependents();
    const Tab<V_REPL> tb = Tab<V_REPL>::template setup<DEC>(smem);   // ends with __syncthreads
    pdl_wait();
    const uint64_t per = (total + gridDim.x - 1) / gridDim.x;
    const uint64_t c0 = per * blockIdx.x, c1 = c0 + per < total ? c0 + per : total;
    const uint32_t lane = threadIdx.x & 31;
    uint64_t w0 = c0 + (threadIdx.x & ~31u);   // warp-uniform start of this warp's 32 blocks
    if (w0 >= c1) return;                       // (no barriers below)
    uint32_t seg;
    {   // last segment with first <= w0: warp-uniform binary search (broadcast loads)
        uint32_t lo = 0, hi = nsegs - 1;
        while (lo < hi) {
            uint32_t mid = (lo + hi + 1) >> 1;
            if (__ldg(&segs[mid].first) <= w0) lo = mid; else hi = mid - 1;
        }
        seg = lo;
    }
    // Software pipeline: the segment walk and the 128-bit load of the NEXT trip
    // are issued before the rounds of the current one, hiding their latency chain.
    // The warp's current segment is cached in registers (first, end, offsets,
    // key): while a message spans whole trips no descriptor is re-read.
    bool have = false;
    uint4 v = make_uint4(0, 0, 0, 0);
    uint4* op = nullptr;
    uint32_t kb = 0;
    uint64_t sf = 0, se = 0, sin = 0, sout = 0;   // cached descriptor of segment `seg`
    uint32_t skey = 0;
    auto load_seg = [&]() {
        const BatchSeg* sg = segs + seg;
        sf = __ldg(&sg->first);
        se = sf + __ldg(&sg->n);
        sin = __ldg(&sg->in_off);
        sout = __ldg(&sg->out_off);
        skey = __ldg(&sg->key);
    };
    load_seg();
    auto fetch = [&](uint64_t base) {
        if (base >= se) {   // warp-uniform advance: gallop then bisect over the sorted `first`s
            uint32_t lo = seg + 1, step = 1;                // first[seg+1] == se <= base
            while (lo + step < nsegs && __ldg(&segs[lo + step].first) <= base) {
                lo += step;
                step <<= 1;
            }
            uint32_t hi = lo + step < nsegs ? lo + step : nsegs;   // first[hi] > base (or hi == nsegs)
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (__ldg(&segs[mid].first) <= base) lo = mid; else hi = mid;
            }
            seg = lo;
            load_seg();
        }
        const uint64_t i = base + lane;
        have = i < c1;
        if (!have) return;
        uint64_t f = sf, io = sin, oo = sout;
        uint32_t key = skey;
        if (i >= se) {                                      // this lane runs past the warp's segment
            uint32_t sidx = seg;
            do {
                sidx++;
            } while (i >= __ldg(&segs[sidx].first) + __ldg(&segs[sidx].n));
            const BatchSeg* sg = segs + sidx;
            f = __ldg(&sg->first);
            io = __ldg(&sg->in_off);
            oo = __ldg(&sg->out_off);
            key = __ldg(&sg->key);
        }
        const uint64_t local = i - f;
        v = __ldcs(reinterpret_cast<const uint4*>(in_base + io) + local);
        op = reinterpret_cast<uint4*>(out_base + oo) + local;
        kb = 60u * key;
    };
    fetch(w0);
    while (w0 < c1) {
        const bool chave = have;
        const uint4 cv = v;
        uint4* const cop = op;
        const uint32_t ckb = kb;
        w0 += blockDim.x;
        if (w0 < c1) fetch(w0);
        if (chave) {
            uint32_t s0 = cv.x ^ keys.w[ckb], s1 = cv.y ^ keys.w[ckb + 1], s2 = cv.z ^ keys.w[ckb + 2],
                     s3 = cv.w ^ keys.w[ckb + 3];
#pragma unroll
            for (int r = 1; r < NR; r++) t_round<DEC>(tb, s0, s1, s2, s3, KeyParamAt<KCAP>{keys, ckb + 4u * r});
            __stcs(cop, final_round<DEC>(tb, s0, s1, s2, s3, KeyParamAt<KCAP>{keys, ckb + 4u * NR}));
        }
    }
}

}  // namespace aesb200

using namespace aesb200;

extern "C" aes_status aes_ecb_batch(const aes_round_keys* keys, int nkeys, int decrypt, const aes_segment* segs, uint32_t nsegs,
                         const void* in_base, void* out_base, void* stream) {
    if (!keys) return AES_ENULL;
    if (nkeys < 1 || nkeys > kBatchMaxKeys) return AES_ERANGE;
    const int nr = keys[0].nr;
    for (int k = 0; k < nkeys; k++) {
        aes_status st = validate_keys(&keys[k], nr);
        if (st) return st;
    }
    if (nsegs == 0) return AES_OK;
    if (!segs || !in_base || !out_base) return AES_ENULL;
    if (((uintptr_t)in_base | (uintptr_t)out_base) & 15) return AES_EALIGN;
    std::vector<BatchSeg> hs(nsegs);
    uint64_t total = 0;
    for (uint32_t i = 0; i < nsegs; i++) {
        const aes_segment& a = segs[i];
        if (a.key_index >= (uint32_t)nkeys) return AES_ERANGE;
        if ((a.in_offset | a.out_offset) & 15) return AES_EALIGN;
        if (a.nblocks > (UINT64_MAX >> 4) || total + a.nblocks < total) return AES_ERANGE;
        uint64_t bytes = a.nblocks << 4;
        uintptr_t pi = (uintptr_t)in_base + a.in_offset, po = (uintptr_t)out_base + a.out_offset;
        if (pi < (uintptr_t)in_base || po < (uintptr_t)out_base || pi > UINTPTR_MAX - bytes || po > UINTPTR_MAX - bytes)
            return AES_ERANGE;
        if (pi != po && pi < po + bytes && po < pi + bytes) return AES_EOVERLAP;
        hs[i] = BatchSeg{a.in_offset, a.out_offset, total, a.nblocks, a.key_index, 0};
        total += a.nblocks;
    }
    if (total == 0) return AES_OK;
    int dev = 0, occ = 1, nsm = 148;
    cudaStream_t cs0 = (cudaStream_t)stream;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e);
    aes_status st;
    cudaStreamCaptureStatus cap_st = cudaStreamCaptureStatusNone;
    if ((e = cudaStreamIsCapturing(cs0, &cap_st)) != cudaSuccess) return cuda_fail(e);
    if (cap_st != cudaStreamCaptureStatusNone) return AES_ECAPTURE;   // staged descriptors are not replayable
    if ((st = check_device_ptr(in_base, dev))) return st;
    if (out_base != in_base && (st = check_device_ptr(out_base, dev))) return st;
    const int kcap = nkeys <= 16 ? 16 : nkeys <= 64 ? 64 : kBatchMaxKeys;   // parameter bytes scale with the tier
    const void* f = nullptr;
#define AES_PICK_BATCH(K)                                                                                   \
    f = nr == 10 ? (decrypt ? (const void*)&batch_kernel<10, true, K> : (const void*)&batch_kernel<10, false, K>) \
      : nr == 12 ? (decrypt ? (const void*)&batch_kernel<12, true, K> : (const void*)&batch_kernel<12, false, K>) \
                 : (decrypt ? (const void*)&batch_kernel<14, true, K> : (const void*)&batch_kernel<14, false, K>)
    if (kcap == 16) AES_PICK_BATCH(16); else if (kcap == 64) AES_PICK_BATCH(64); else AES_PICK_BATCH(kBatchMaxKeys);
#undef AES_PICK_BATCH
    const size_t smem = decrypt ? kSmemReplDec : kSmemReplEnc;
    KernelInfo ki{f, smem};
    if ((st = resident_ctas(dev, ki, &occ, &nsm))) return st;
    // segment descriptors: one stream-ordered allocation freed after the kernel
    const size_t seg_bytes = sizeof(BatchSeg) * nsegs;
    cudaStream_t cs = (cudaStream_t)stream;
    cudaMemPool_t pool;
    if ((st = desc_pool(dev, &pool))) return st;
    void* d = nullptr;
    if ((e = cudaMallocFromPoolAsync(&d, seg_bytes, pool, cs)) != cudaSuccess) return cuda_fail(e);
    if ((st = stage_h2d(dev, d, hs.data(), seg_bytes, cs))) {
        cudaFreeAsync(d, cs);
        return st;
    }
    // key schedules by value (kernel parameters)
    static thread_local BatchKeys<kBatchMaxKeys> kbig;   // 30 KiB: off the stack
    static thread_local BatchKeys<64> kmid;
    BatchKeys<16> ksmall;
    uint32_t* kw = kcap == 16 ? ksmall.w : kcap == 64 ? kmid.w : kbig.w;
    for (int k = 0; k < nkeys; k++) std::memcpy(kw + 60 * k, decrypt ? keys[k].dk : keys[k].ek, 240);
    const char* pin = static_cast<const char*>(in_base);
    char* pout = static_cast<char*>(out_base);
    const BatchSeg* dsegs = static_cast<const BatchSeg*>(d);
    void* args[] = {(void*)&pin, (void*)&pout, (void*)&dsegs, (void*)&nsegs, (void*)&total,
                    kcap == 16 ? (void*)&ksmall : kcap == 64 ? (void*)&kmid : (void*)&kbig};
    uint64_t want = (total + 31) / 32, cap = (uint64_t)nsm * occ;
    // no PDL: the kernel's predecessor on the stream is the descriptor copy
    st = launch_kernel(ki, (unsigned)(want < cap ? want : cap), args, cs, false);
    cudaError_t e2 = cudaFreeAsync(d, cs);
    if (st) return st;
    return e2 == cudaSuccess ? AES_OK : cuda_fail(e2);
}
