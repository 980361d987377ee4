// aes_ecb.cu -- sm_100a AES kernels (steps A4..A10 of SURVEY.md 8(a)): ECB,
// CTR and CBC-decryption, the table-placement / staging ablation variants,
// the per-round trace and the LDS-gather microbenchmark, with their C ABI
// entry points (include/aes_b200.h).  The building blocks every kernel shares
// (tables, table policies, the Eq 26 round, the final round) are in
// aes_device.cuh.
//
// One 16-byte state per thread (sec 4.1), held in four
// 32-bit registers (column c = LE word c).  Rounds are the paper's T-table
// round, Eq 26:
//     e_j = T0[p_{0,j}] ^ T1[p_{1,j+1}] ^ T2[p_{2,j+2}] ^ T3[p_{3,j+3}] ^ k_j
// with column indices mod 4 (R8), and for decryption the
// equivalent-inverse round with Td0..Td3 and offsets j, j-1, j-2, j-3 (R12).
// The final round (no MixColumns, R1) takes S[x] from a byte of a Te word
// (R14) and Si[x] from a replicated Si word table.
//
// B200 design:
//  * T-tables are lane-replicated in shared memory: entry x of table i for
//    lane L lives at byte x*256 + (i&1)*128 + L*4 of region (i>>1), so every
//    lane always hits bank L -- conflict-free for any data.  The address is
//    ONE PRMT: __byte_perm(L*4, s, 0x1140 + 16k) = (byte k of s)<<8 | L*4;
//    the table base is the LDS immediate.  The paper put the tables in
//    __constant__ memory; that is kept as AES_VAR_CONST for the
//    ablation, together with an unreplicated shared-memory variant.
//  * Round keys are a by-value kernel parameter (constant bank, broadcast),
//    as the paper's "round keys in the constant memory" but
//    per launch, hence safe across concurrent streams.
//  * States move as coalesced 128-bit streaming loads/stores (LDG.128/STG.128
//    with evict-first hints); persistent grid-stride CTAs amortise the
//    per-CTA table fill.  No tensor cores: this is table lookup, not a
//    contraction (SURVEY.md 7 "Hard parts" 9).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "aes_b200.h"
#include "aes_bitslice.cuh"
#include "aes_device.cuh"
#include "aes_host.h"

namespace aesb200 {

// ---------------------------------------------------------------------------
// Kernels: persistent grid-stride, SPT states per thread per trip.
//   ecb_kernel          C_i = E(P_i) / P_i = D(C_i)                (Eq 1)
//   ctr_kernel          C_i = P_i ^ E(ctr0 + i), BE 128-bit counter  (Eq 5, R24)
//   cbc_decrypt_kernel  P_i = D(C_i) ^ C_{i-1}, C_{-1} = IV          (Eq 2, R25)
// ---------------------------------------------------------------------------
template <int NR, bool DEC, int V, int SPT, int MODE>
__device__ __forceinline__ void aes_body(const uint4* __restrict__ in, uint4* __restrict__ out, uint64_t n,
                                         const RK& rk, const ModeP& mp) {
    extern __shared__ __align__(16) uint32_t smem[];
    pdl_launch_dependents();
    const Tab<V> tb = Tab<V>::template setup<DEC>(smem);   // A4
    pdl_wait();
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    const Split sp = split_work(n, SPT * T);
    // one trip: SPT states at i, i + stride, ..., those with their okmask bit set
    auto trip = [&](uint64_t i, uint64_t stride, uint32_t okmask) {
        uint4 v[SPT], w[SPT];
#pragma unroll
        for (int k = 0; k < SPT; k++) {
            v[k] = w[k] = make_uint4(0, 0, 0, 0);
            const uint64_t j = i + k * stride;
            if (okmask >> k & 1) {                                         // A5
                if (MODE == M_ECB) v[k] = __ldcs(in + j);
                if (MODE == M_CTR) { v[k] = counter_block(mp, j); w[k] = __ldcs(in + j); }
                if (MODE == M_CBCD) {
                    v[k] = __ldg(in + j);
                    w[k] = j ? __ldg(in + j - 1) : make_uint4(mp.iv[0], mp.iv[1], mp.iv[2], mp.iv[3]);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < SPT; k++) v[k] = cipher_block<NR, DEC>(tb, v[k], rk);   // A6-A8
#pragma unroll
        for (int k = 0; k < SPT; k++)
            if (okmask >> k & 1) __stcs(out + i + k * stride, MODE == M_ECB ? v[k] : xor4(v[k], w[k]));   // A9
    };
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < sp.full; i += SPT * T)
        trip(i, T, (1u << SPT) - 1);
    // tail: this CTA's contiguous chunk, blockDim-strided
    uint32_t okmask = 0;
#pragma unroll
    for (int k = 0; k < SPT; k++) okmask |= (threadIdx.x + k * blockDim.x < sp.tlen ? 1u : 0u) << k;
    if (okmask) trip(sp.tbase + threadIdx.x, blockDim.x, okmask);
}

// ECB with the next trip's state load issued before the current trip's rounds
// (software prefetch across loop iterations; the compiler does not hoist it).
// Sequence of this thread's blocks: gid, gid + T, ... (< full), then its tail block.
template <int NR, bool DEC, int V>
__device__ __forceinline__ void ecb_prefetch_body(const uint4* __restrict__ in, uint4* __restrict__ out, uint64_t n,
                                                  const RK& rk) {
    extern __shared__ __align__(16) uint32_t smem[];
    pdl_launch_dependents();
    const Tab<V> tb = Tab<V>::template setup<DEC>(smem);
    pdl_wait();
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    const Split sp = split_work(n, T);
    const uint64_t tail = sp.tbase + threadIdx.x;
    const bool has_tail = threadIdx.x < sp.tlen;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool valid = true;
    if (i >= sp.full) { i = tail; valid = has_tail; }
    uint4 v = make_uint4(0, 0, 0, 0);
    if (valid) v = __ldcs(in + i);
    while (valid) {
        const uint4 cur = v;
        const uint64_t ci = i;
        if (i < sp.full) {
            i += T;
            if (i >= sp.full) { i = tail; valid = has_tail; }
        } else {
            valid = false;
        }
        if (valid) v = __ldcs(in + i);
        __stcs(out + ci, cipher_block<NR, DEC>(tb, cur, rk));
    }
}

template <int NR, bool DEC, int V, int SPT>
__global__ void __launch_bounds__(kThreads, 1)
    ecb_kernel(const uint4* __restrict__ in, uint4* __restrict__ out, uint64_t n, const __grid_constant__ RK rk) {
    if (SPT == 1 && V == V_REPL) ecb_prefetch_body<NR, DEC, V>(in, out, n, rk);
    else aes_body<NR, DEC, V, SPT, M_ECB>(in, out, n, rk, ModeP{});
}

template <int NR>
__global__ void __launch_bounds__(kThreads, 1)
    ctr_kernel(const uint4* __restrict__ in, uint4* __restrict__ out, uint64_t n, const __grid_constant__ RK rk,
               const __grid_constant__ ModeP mp) {
    aes_body<NR, false, V_REPL, 1, M_CTR>(in, out, n, rk, mp);
}

template <int NR>
__global__ void __launch_bounds__(kThreads, 1)
    ctr_cached_kernel(const uint4* __restrict__ in, uint4* __restrict__ out, uint64_t n,
                      const __grid_constant__ RK rk, const __grid_constant__ ModeP mp) {
    extern __shared__ __align__(16) uint32_t smem[];
    pdl_launch_dependents();
    const Tab<V_REPL> tb = Tab<V_REPL>::template setup<false>(smem);
    pdl_wait();
    // Warp-private table of group constants for the warp's next 16 trips x
    // (the <= 2 groups its 32 consecutive blocks touch): 32 entries x 8 words,
    // filled by the 32 lanes in parallel -- 27 LDS instructions per 16 trips
    // and no block-wide barrier (warps drift freely, as in the ECB kernel).
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t* wt = smem + kSmemReplEnc / 4 + warp * 256;
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t first = (uint64_t)blockIdx.x * blockDim.x + warp * 32;   // this warp's first block
    for (uint64_t t = 0;; t++) {
        const uint64_t cb = first + t * T;   // warp-uniform
        if (cb >= n) break;
        if ((t & 15) == 0) {
            __syncwarp();                    // previous 16 trips' entries fully read
            const uint64_t tcb = cb + (uint64_t)(lane >> 1) * T;
            if (tcb < n) ctr_fill_group(tb, rk, mp, tcb, lane, wt);
            __syncwarp();
        }
        const uint64_t i = cb + lane;
        if (i < n) __stcs(out + i, ctr_cached_block<NR>(tb, rk, mp, wt, (uint32_t)(t & 15), cb, lane, __ldcs(in + i)));
    }
}

template <int NR>
__global__ void __launch_bounds__(kThreads, 1)
    cbc_decrypt_kernel(const uint4* __restrict__ in, uint4* __restrict__ out, uint64_t n,
                       const __grid_constant__ RK rk, const __grid_constant__ ModeP mp) {
    aes_body<NR, true, V_REPL, 1, M_CBCD>(in, out, n, rk, mp);
}

// Debug/pin kernel (aes_ecb_trace): the state after ARK(0) and `rounds` rounds
// of the SAME t_round / final_round code the production kernels inline, one
// state per thread.  rounds = NR gives the full cipher.
template <int NR, bool DEC>
__global__ void __launch_bounds__(kThreads, 1)
    trace_kernel(const uint4* __restrict__ in, uint4* __restrict__ out, uint64_t n, const __grid_constant__ RK rk,
                 int rounds) {
    extern __shared__ __align__(16) uint32_t smem[];
    pdl_launch_dependents();
    const Tab<V_REPL> tb = Tab<V_REPL>::template setup<DEC>(smem);
    pdl_wait();
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += T) {
        uint4 v = in[i];
        uint32_t s0 = v.x ^ rk.w[0], s1 = v.y ^ rk.w[1], s2 = v.z ^ rk.w[2], s3 = v.w ^ rk.w[3];
        for (int r = 1; r <= rounds && r < NR; r++) t_round<DEC>(tb, s0, s1, s2, s3, KeyAt{rk, r});
        out[i] = rounds >= NR ? final_round<DEC>(tb, s0, s1, s2, s3, KeyAt{rk, NR}) : make_uint4(s0, s1, s2, s3);
    }
}

// ---------------------------------------------------------------------------
// LDS gather microbenchmark (the binding roofline)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 1) lds_gather_kernel(uint32_t* sink, int iters) {
    extern __shared__ __align__(16) uint32_t smem[];
    uint4* s4 = reinterpret_cast<uint4*>(smem);
    for (int q = threadIdx.x; q < 8192; q += blockDim.x) {
        int w = 4 * q;
        uint32_t v = g_tab.te[(w >> 5) & 1][(w >> 6) & 255];
        s4[q] = make_uint4(v, v, v, v);
    }
    __syncthreads();
    const char* sb = reinterpret_cast<const char*>(smem);
    const uint32_t lo = (threadIdx.x & 31) * 4;
    uint32_t a[16];
#pragma unroll
    for (int c = 0; c < 16; c++) a[c] = (threadIdx.x * 2654435761u) ^ (c * 0x9E3779B9u) ^ blockIdx.x;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int c = 0; c < 16; c++)
            a[c] = *reinterpret_cast<const uint32_t*>(sb + 128 * (c & 1) + __byte_perm(lo, a[c], 0x1140 + 16 * (c & 3)));
    }
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < 16; c++) acc ^= a[c];
    sink[(uint64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// ---------------------------------------------------------------------------
// AES_VAR_SMEM_REPL_TMA: the same rounds, with the states staged into shared
// memory by the bulk-copy engine (cp.async.bulk + mbarrier, SASS UBLKCP) --
// the north star's "TMA or cp.async staging of input tiles" (SURVEY.md 7 step
// 5(e)).  Each warp owns a 2-stage ring of 512-byte tiles (32 states): lane 0
// issues the copy of the tile two trips ahead, all lanes wait on the tile's
// mbarrier, read their state with one LDS.128, cipher it, store with STG.128.
// Kept as a measured variant: the tile still has to reach registers through
// the shared-memory data path the rounds saturate.
// ---------------------------------------------------------------------------
constexpr int kTmaStages = 2;
constexpr size_t kTmaTileBytes = 512;
constexpr size_t kTmaRing = (kThreads / 32) * kTmaStages * kTmaTileBytes;   // 32 KiB
constexpr size_t kTmaBars = (kThreads / 32) * kTmaStages * 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int NR, bool DEC>
__global__ void __launch_bounds__(kThreads, 1)
    ecb_tma_kernel(const uint4* __restrict__ in, uint4* __restrict__ out, uint64_t n, const __grid_constant__ RK rk) {
    extern __shared__ __align__(16) uint32_t smem[];
    pdl_launch_dependents();
    const Tab<V_REPL> tb = Tab<V_REPL>::template setup<DEC>(smem);
    pdl_wait();
    const size_t tab_bytes = DEC ? kSmemReplDec : kSmemReplEnc;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    char* ring = reinterpret_cast<char*>(smem) + tab_bytes + warp * kTmaStages * kTmaTileBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(smem) + tab_bytes + kTmaRing) +
                     warp * kTmaStages;
    if (lane == 0) {
        for (int st = 0; st < kTmaStages; st++)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + st)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const uint64_t total_warps = (uint64_t)gridDim.x * (kThreads / 32);
    const uint64_t chunks = (n + 31) / 32;
    const uint64_t q0 = (uint64_t)blockIdx.x * (kThreads / 32) + warp;
    auto issue = [&](uint64_t k) {            // lane 0: tile of this warp's k-th chunk -> stage k % S
        const uint64_t q = q0 + k * total_warps;
        if (q >= chunks) return;
        const uint64_t b0 = q * 32;
        const uint32_t bytes = (uint32_t)((n - b0 < 32 ? n - b0 : 32) * 16);
        const int st = (int)(k % kTmaStages);
        const uint32_t bar = smem_u32(bars + st), dst = smem_u32(ring + st * kTmaTileBytes);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
            "l"(in + b0), "r"(bytes), "r"(bar)
            : "memory");
    };
    if (lane == 0)
        for (int k = 0; k < kTmaStages; k++) issue(k);
    for (uint64_t k = 0;; k++) {
        const uint64_t q = q0 + k * total_warps;
        if (q >= chunks) break;
        const int st = (int)(k % kTmaStages);
        const uint32_t parity = (uint32_t)((k / kTmaStages) & 1);
        const uint32_t bar = smem_u32(bars + st);
        uint32_t done = 0;
        while (!done)
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(bar), "r"(parity)
                : "memory");
        const uint64_t i = q * 32 + lane;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (i < n) v = reinterpret_cast<const uint4*>(ring + st * kTmaTileBytes)[lane];
        uint32_t s0 = v.x ^ rk.w[0], s1 = v.y ^ rk.w[1], s2 = v.z ^ rk.w[2], s3 = v.w ^ rk.w[3];
        // every lane has consumed the tile (the XOR used the loaded registers): recycle the stage
        asm volatile("" ::"r"(s0), "r"(s1), "r"(s2), "r"(s3) : "memory");
        __syncwarp();
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(k + kTmaStages);
        }
#pragma unroll
        for (int r = 1; r < NR; r++) t_round<DEC>(tb, s0, s1, s2, s3, KeyAt{rk, r});
        if (i < n) __stcs(out + i, final_round<DEC>(tb, s0, s1, s2, s3, KeyAt{rk, NR}));
    }
}

// ---------------------------------------------------------------------------
// Host side: kernel registry and launch
// ---------------------------------------------------------------------------

template <int NR, bool DEC, int V, int SPT>
KernelInfo kinfo() {
    size_t sm = V == V_REPL ? (DEC ? kSmemReplDec : kSmemReplEnc) : V == V_PLAIN ? kSmemPlain : V == V_ROT ? kSmemRot : 0;   // CONST, GLOBAL: none
    return {reinterpret_cast<const void*>(&ecb_kernel<NR, DEC, V, SPT>), sm};
}

template <int NR, bool DEC>
KernelInfo pick_spt(int v, int spt) {
    if (v == V_REPL) {
        switch (spt) {
            case 1: return kinfo<NR, DEC, V_REPL, 1>();
            case 2: return kinfo<NR, DEC, V_REPL, 2>();
            case 4: return kinfo<NR, DEC, V_REPL, 4>();
        }
    } else if (spt == 1) {
        if (v == V_REPL_TMA)
            return {reinterpret_cast<const void*>(&ecb_tma_kernel<NR, DEC>),
                    (DEC ? kSmemReplDec : kSmemReplEnc) + kTmaRing + kTmaBars};
        if (v == V_PLAIN) return kinfo<NR, DEC, V_PLAIN, 1>();
        if (v == V_ROT) return kinfo<NR, DEC, V_ROT, 1>();
        if (v == V_CONST) return kinfo<NR, DEC, V_CONST, 1>();
        if (v == V_GLOBAL) return kinfo<NR, DEC, V_GLOBAL, 1>();
    }
    return {nullptr, 0};
}

KernelInfo pick(int nr, bool dec, int v, int spt) {
    switch (nr) {
        case 10: return dec ? pick_spt<10, true>(v, spt) : pick_spt<10, false>(v, spt);
        case 12: return dec ? pick_spt<12, true>(v, spt) : pick_spt<12, false>(v, spt);
        case 14: return dec ? pick_spt<14, true>(v, spt) : pick_spt<14, false>(v, spt);
    }
    return {nullptr, 0};
}

// AES_B200_CTR_KERNEL=plain selects the uncached T-table CTR kernel (A/B measurement only)
bool ctr_plain_requested() {
    static const bool plain = [] {
        const char* e = std::getenv("AES_B200_CTR_KERNEL");
        return e && std::strcmp(e, "plain") == 0;
    }();
    return plain;
}

KernelInfo pick_mode(int nr, int mode) {
    const void* f = nullptr;
    if (mode == M_CTR) {
        if (ctr_plain_requested()) {
            f = nr == 10 ? (const void*)&ctr_kernel<10> : nr == 12 ? (const void*)&ctr_kernel<12>
                                                                   : (const void*)&ctr_kernel<14>;
            return {f, kSmemReplEnc};
        }
        f = nr == 10 ? (const void*)&ctr_cached_kernel<10> : nr == 12 ? (const void*)&ctr_cached_kernel<12>
                                                                      : (const void*)&ctr_cached_kernel<14>;
        return {f, kSmemReplEnc + kCtrTableBytes};
    }
    f = nr == 10 ? (const void*)&cbc_decrypt_kernel<10> : nr == 12 ? (const void*)&cbc_decrypt_kernel<12>
                                                                   : (const void*)&cbc_decrypt_kernel<14>;
    return {f, kSmemReplDec};
}

constexpr uint64_t kHybridMinBlocks = 1ull << 23;

// AES_B200_HYBRID_MIN_BLOCKS=<n> moves the default-kernel crossover (tests use
// it to put the hybrid CTR / CBC kernels under small oracle-checked inputs).
uint64_t hybrid_min_blocks() {
    const char* e = std::getenv("AES_B200_HYBRID_MIN_BLOCKS");
    return e ? std::strtoull(e, nullptr, 10) : kHybridMinBlocks;
}

aes_status launch(const aes_round_keys* rk, int nr, int decrypt, const void* in, void* out, uint64_t nblocks,
                  cudaStream_t stream, const aes_launch_config* cfg, bool check_ptrs, int mode = M_ECB,
                  const ModeP* mp = nullptr) {
    aes_status st = validate_keys(rk, nr);
    if (st) return st;
    int variant = cfg ? cfg->variant : AES_VAR_DEFAULT;
    int spt = cfg ? cfg->states_per_thread : 0;
    int grid_req = cfg ? cfg->grid : 0;
    const int flags = cfg ? cfg->flags : 0;
    // Default: the hybrid kernel (T-table + bitsliced warps) from 2^23 blocks
    // (128 MiB) up, where its bitsliced warps get enough work to pay for
    // running 28 instead of 32 T-table warps; the replicated T-table kernel
    // below that (measured crossover 64-128 MiB).
    if (variant == AES_VAR_DEFAULT)
        variant = (spt <= 1 && nblocks >= hybrid_min_blocks() && !(mode == M_CTR && ctr_plain_requested()))
                      ? V_HYBRID
                      : V_REPL;
    if (spt == 0) spt = 1;                              // S = 1, 2, 4 measure within 1 %
    if (grid_req < 0 || (flags & ~(AES_LAUNCH_TRUSTED_PTRS | AES_LAUNCH_NO_PDL))) return AES_ERANGE;
    if (flags & AES_LAUNCH_TRUSTED_PTRS) check_ptrs = false;
    if (mode != M_ECB && variant != V_HYBRID) variant = V_REPL;   // the modes: hybrid or their own kernels
    bool bsk = variant == V_HYBRID || variant == V_BITSLICE;
    KernelInfo ki = bsk           ? (spt == 1 ? pick_hybrid(nr, decrypt != 0, variant, mode) : KernelInfo{nullptr, 0})
                    : mode != M_ECB ? pick_mode(nr, mode)
                                  : pick(nr, decrypt != 0, variant, spt);
    if (mode != M_ECB) spt = 1;
    if (!ki.fn) return AES_EVARIANT;
    if (nblocks == 0) return AES_OK;
    if ((st = validate_buffers(in, out, nblocks))) return st;
    if (mode == M_CBCD && in == out) return AES_EOVERLAP;   // C_{i-1} must survive block i-1's write
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e);
    if (check_ptrs) {
        if ((st = check_device_ptr(in, dev))) return st;
        if (out != in && (st = check_device_ptr(out, dev))) return st;
    }
    int occ = 1, nsm = 148;
    if ((st = resident_ctas(dev, ki, &occ, &nsm))) return st;
    // Persistent grid (SMs x resident CTAs), or fewer CTAs when the message is
    // small: every CTA gets >= 32 blocks (one full warp), because each one
    // pays a 128-192 KiB table fill.  The kernels split the remainder of whole
    // trips into one contiguous chunk per CTA (split_work), so all of them work.
    uint64_t per_cta = 32ull * spt;
    uint64_t want = (nblocks + per_cta - 1) / per_cta;
    uint64_t cap = grid_req ? (uint64_t)grid_req : (uint64_t)nsm * occ;
    unsigned grid = (unsigned)(want < cap ? want : cap);
    if (bsk && variant == V_HYBRID && (nblocks / 32) / grid >= (1ull << 31) - 64) {
        // beyond the hybrid kernel's 32-bit per-CTA unit counter (2^36 blocks per
        // CTA = 1 TiB): the T-table kernels compute the identical result
        bsk = false;
        ki = mode != M_ECB ? pick_mode(nr, mode) : pick(nr, decrypt != 0, V_REPL, 1);
        if ((st = resident_ctas(dev, ki, &occ, &nsm))) return st;
    }
    RK k;
    std::memcpy(k.w, decrypt ? rk->dk : rk->ek, sizeof k.w);
    const uint4* pin = static_cast<const uint4*>(in);
    uint4* pout = static_cast<uint4*>(out);
    ModeP m = mp ? *mp : ModeP{};
    void* args[] = {(void*)&pin, (void*)&pout, (void*)&nblocks, (void*)&k, (void*)&m, nullptr};
    if (bsk) {   // hybrid / bitsliced kernels: (in, out, n, RK, BSK, ModeP)
        static thread_local BSK bs;
        bitslice_keys(rk, decrypt, &bs);
        args[4] = (void*)&bs;
        args[5] = (void*)&m;
    }
    return launch_kernel(ki, grid, args, stream, !(flags & AES_LAUNCH_NO_PDL));
}

aes_status launch_ecb(const aes_round_keys* rk, int nr, int decrypt, const void* in, void* out, uint64_t nblocks,
                      cudaStream_t stream, bool check_ptrs) {
    return launch(rk, nr, decrypt, in, out, nblocks, stream, nullptr, check_ptrs);
}

}  // namespace aesb200

using namespace aesb200;

extern "C" {

aes_status aes_ecb_encrypt(const aes_round_keys* rk, int nr, const void* in, void* out, uint64_t nblocks,
                           void* stream) {
    return launch(rk, nr, 0, in, out, nblocks, (cudaStream_t)stream, nullptr, true);
}

aes_status aes_ecb_decrypt(const aes_round_keys* rk, int nr, const void* in, void* out, uint64_t nblocks,
                           void* stream) {
    return launch(rk, nr, 1, in, out, nblocks, (cudaStream_t)stream, nullptr, true);
}

aes_status aes_ecb_launch(const aes_round_keys* rk, int nr, int decrypt, const void* in, void* out,
                          uint64_t nblocks, void* stream, const aes_launch_config* cfg) {
    return launch(rk, nr, decrypt, in, out, nblocks, (cudaStream_t)stream, cfg, true);
}

aes_status aes_ctr_xcrypt(const aes_round_keys* rk, int nr, const uint8_t* iv, uint64_t block_offset,
                          const void* in, void* out, uint64_t nblocks, void* stream) {
    aes_status st = validate_keys(rk, nr);
    if (st) return st;
    if (!iv) return AES_ENULL;
    ModeP m{};
    uint64_t hi = 0, lo = 0;
    for (int b = 0; b < 8; b++) hi = (hi << 8) | iv[b];
    for (int b = 8; b < 16; b++) lo = (lo << 8) | iv[b];
    uint64_t lo2 = lo + block_offset;
    m.ctr_hi = hi + (lo2 < lo ? 1 : 0);
    m.ctr_lo = lo2;
    return launch(rk, nr, 0, in, out, nblocks, (cudaStream_t)stream, nullptr, true, M_CTR, &m);
}

aes_status aes_cbc_decrypt(const aes_round_keys* rk, int nr, const uint8_t* iv, const void* in, void* out,
                           uint64_t nblocks, void* stream) {
    aes_status st = validate_keys(rk, nr);
    if (st) return st;
    if (!iv) return AES_ENULL;
    ModeP m{};
    for (int j = 0; j < 4; j++)
        m.iv[j] = (uint32_t)iv[4 * j] | ((uint32_t)iv[4 * j + 1] << 8) | ((uint32_t)iv[4 * j + 2] << 16) |
                  ((uint32_t)iv[4 * j + 3] << 24);
    return launch(rk, nr, 1, in, out, nblocks, (cudaStream_t)stream, nullptr, true, M_CBCD, &m);
}

aes_status aes_ecb_trace(const aes_round_keys* rk, int nr, int decrypt, int rounds, const void* in, void* out,
                         uint64_t nblocks, void* stream) {
    aes_status st = validate_keys(rk, nr);
    if (st) return st;
    if (rounds < 0 || rounds > nr) return AES_ERANGE;
    if (nblocks == 0) return AES_OK;
    if ((st = validate_buffers(in, out, nblocks))) return st;
    int dev = 0, occ = 1, nsm = 148;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e);
    if ((st = check_device_ptr(in, dev))) return st;
    if (out != in && (st = check_device_ptr(out, dev))) return st;
    const void* f;
    if (nr == 10) f = decrypt ? (const void*)&trace_kernel<10, true> : (const void*)&trace_kernel<10, false>;
    else if (nr == 12) f = decrypt ? (const void*)&trace_kernel<12, true> : (const void*)&trace_kernel<12, false>;
    else f = decrypt ? (const void*)&trace_kernel<14, true> : (const void*)&trace_kernel<14, false>;
    KernelInfo ki{f, decrypt ? kSmemReplDec : kSmemReplEnc};
    if ((st = resident_ctas(dev, ki, &occ, &nsm))) return st;
    uint64_t want = (nblocks + 31) / 32, cap = (uint64_t)nsm * occ;
    RK k;
    std::memcpy(k.w, decrypt ? rk->dk : rk->ek, sizeof k.w);
    const uint4* pin = static_cast<const uint4*>(in);
    uint4* pout = static_cast<uint4*>(out);
    void* args[] = {(void*)&pin, (void*)&pout, (void*)&nblocks, (void*)&k, (void*)&rounds};
    return launch_kernel(ki, (unsigned)(want < cap ? want : cap), args, (cudaStream_t)stream, true);
}

aes_status aes_mb_lds_gather(void* sink, int grid, int iters, void* stream) {
    if (!sink) return AES_ENULL;
    if (grid <= 0 || iters < 0) return AES_ERANGE;
    int dev = 0, occ = 1, nsm = 148;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e);
    KernelInfo ki{reinterpret_cast<const void*>(&lds_gather_kernel), kSmemReplEnc};
    aes_status st = resident_ctas(dev, ki, &occ, &nsm);   // sets the smem attribute once per device
    if (st) return st;
    lds_gather_kernel<<<grid, kThreads, kSmemReplEnc, (cudaStream_t)stream>>>(static_cast<uint32_t*>(sink), iters);
    e = cudaGetLastError();
    return e == cudaSuccess ? AES_OK : cuda_fail(e);
}

}  // extern "C"
