// aes_hybrid.cu -- kernels that add bitsliced (lookup-free) warps to the
// T-table rounds (VERDICT r01 "next" 7; SURVEY.md 7 hard part 1, R26).
//
//   hybrid_kernel<NR,DEC,MODE>  AES_VAR_HYBRID (the default from 2^23 blocks):
//                           per 1024-thread CTA, kHybT warps run
//                           the T-table rounds (Eq 26, the
//                           production t_round/final_round, lane-replicated
//                           tables) and kHybB warps run the bitsliced cipher of
//                           aes_bitslice.cuh on the ALU pipe the T-table warps
//                           leave idle.  Both pull 32-block units from one
//                           CTA-local queue (a shared-memory counter), so the
//                           split adapts to whatever rate each side reaches.
//   bs_kernel<NR,DEC>       AES_VAR_BITSLICE: every warp bitsliced (the ALU-only
//                           reference point of the ablation).
// The hybrid kernel also serves the NEXT modes (MODE = M_CTR: the T-table
// warps keep ctr_cached_kernel's counter-mode caching, claiming 16 units at a
// time; M_CBCD: P_i = D(C_i) ^ C_{i-1} on both sides).
//
// Work order.  CTA c walks its "virtual" unit sequence u = 0, 1, 2, ...;
// unit u is the 32-block run starting at block
//   ((c + (u / kSuper) * grid) * kSuper + u % kSuper) * 32,
// i.e. super-chunks of kSuper units are dealt round-robin to the CTAs (all
// CTAs sweep HBM together, as the grid-stride loop of ecb_kernel does) and
// inside its super-chunk a CTA's warps take units in claim order.  The map is
// increasing in u, so the first unit at or past n ends a warp's loop.
// A T-table warp claims 2 units (two blocks per lane; 16 in CTR mode, one
// counter-group table fill per claim); a bitsliced warp claims 8
// (eight blocks per lane, unit j -> block slot j) and stops claiming once
// fewer than kTailUnits units of its CTA remain, so the slow bitsliced claims
// never form the kernel's tail.
//
// Registers: the kernel is compiled for 1024 threads x 64 registers; the
// T-table warpgroups give registers back (setmaxnreg.dec to kRegT) and the
// bitsliced warpgroup takes them (setmaxnreg.inc to kRegB):
// 28 x 56 + 4 x 120 = 32 x 64.
#include <cuda_runtime.h>

#include <cstdint>

#include "aes_b200.h"
#include "aes_bitslice.cuh"
#include "aes_device.cuh"
#include "aes_host.h"

#ifndef AES_HYB_STEP
#define AES_HYB_STEP 2
#endif

namespace aesb200 {

constexpr int kHybT = 28;                  // T-table warps per CTA (7 warpgroups)
constexpr int kHybB = kThreads / 32 - kHybT;   // bitsliced warps per CTA (1 warpgroup)
constexpr int kRegT = 56, kRegB = 120;
static_assert(kHybT * kRegT + kHybB * kRegB <= (kThreads / 32) * 64, "register budget");
static_assert(kHybT % 4 == 0 && kHybB % 4 == 0, "setmaxnreg acts on whole warpgroups");
constexpr uint64_t kUnit = 32;             // blocks per unit
constexpr uint64_t kSuper = 64;            // units per super-chunk (2048 blocks = 32 KiB)
constexpr uint64_t kTailUnits = 384;       // bitsliced warps stop claiming this close to the end
constexpr int kStep = AES_HYB_STEP;        // units per T-table claim (ECB / CBC); 4 measured 1 % slower
// The unit counter is 32-bit (a native shared-memory ATOMS.ADD; the 64-bit
// one is a CAS loop): launch() falls back to the T-table kernel when a CTA
// would need 2^31 units or more (2^36 blocks = 1 TiB per CTA).

__device__ __forceinline__ uint64_t unit_block(uint32_t u) {
    const uint64_t sc = (uint64_t)(u / (uint32_t)kSuper) * gridDim.x + blockIdx.x;   // IMAD.WIDE.U32
    return sc * (kSuper * kUnit) + (u % (uint32_t)kSuper) * kUnit;
}

// One bitsliced pass over 8 x 32 blocks: lane L handles blocks base(j) + L.
// Every load/store instruction of the warp moves 512 contiguous bytes.
//   ECB : out = E/D(in)
//   CTR : out = in ^ E(counter(i))          (counters computed, Eq 5 / R24)
//   CBCD: out = D(in) ^ in[i-1] (IV at 0)   (Eq 2 decryption / R25)
template <int NR, bool DEC, int MODE, class BaseOf>
__device__ __forceinline__ void bs_pass(const uint4* __restrict__ in, uint4* __restrict__ out, uint64_t n,
                                        const BSK& bk, const ModeP& mp, BaseOf base) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t v[8][4];
#pragma unroll
    for (int j = 0; j < 8; j++) {
        const uint64_t i = base(j) + lane;
        uint4 x = make_uint4(0, 0, 0, 0);
        if (MODE == M_CTR) x = counter_block(mp, i);
        else if (i < n) x = MODE == M_CBCD ? __ldg(in + i) : __ldcs(in + i);
        v[j][0] = x.x; v[j][1] = x.y; v[j][2] = x.z; v[j][3] = x.w;
    }
    uint32_t R[4][8];
    bs_pack(v, R, bk);
    if (DEC) bs_decrypt<NR>(R, bk);
    else bs_encrypt<NR>(R, bk);
    bs_unpack(R, v, bk);
#pragma unroll
    for (int j = 0; j < 8; j++) {
        const uint64_t i = base(j) + lane;
        if (i < n) {
            uint4 y = make_uint4(v[j][0], v[j][1], v[j][2], v[j][3]);
            if (MODE == M_CTR) y = xor4(y, __ldcs(in + i));
            if (MODE == M_CBCD) y = xor4(y, i ? __ldg(in + i - 1) : make_uint4(mp.iv[0], mp.iv[1], mp.iv[2], mp.iv[3]));
            __stcs(out + i, y);
        }
    }
}

template <int NR, bool DEC, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    hybrid_kernel(const uint4* __restrict__ in, uint4* __restrict__ out, uint64_t n, const __grid_constant__ RK rk,
                  const __grid_constant__ BSK bk, const __grid_constant__ ModeP mp) {
    extern __shared__ __align__(16) uint32_t smem[];
    __shared__ uint32_t q_next;   // next unclaimed unit of this CTA (32-bit: native ATOMS.ADD)
    pdl_launch_dependents();
    if (threadIdx.x == 0) q_next = 0;
    const Tab<V_REPL> tb = Tab<V_REPL>::template setup<DEC>(smem);   // ends with __syncthreads
    pdl_wait();
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp < kHybT) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegT));
        if (MODE == M_CTR) {
            // Counter-mode caching as in ctr_cached_kernel: a warp claims 16
            // units, its 32 lanes fill the group constants of their (<= 2)
            // counter groups into the warp's table, then it walks the units.
            uint32_t* wt = smem + kSmemReplEnc / 4 + warp * 256;
            for (;;) {
                uint32_t a = 0;
                if (lane == 0) a = atomicAdd(&q_next, 16u);
                const uint32_t u0 = __shfl_sync(0xffffffffu, a, 0);
                if (unit_block(u0) >= n) break;
                __syncwarp();                               // previous claim's entries fully read
                const uint64_t tcb = unit_block(u0 + (lane >> 1));
                if (tcb < n) ctr_fill_group(tb, rk, mp, tcb, lane, wt);
                __syncwarp();
#pragma unroll 1
                for (uint32_t t = 0; t < 16; t++) {
                    const uint64_t cb = unit_block(u0 + t);
                    if (cb >= n) break;
                    const uint64_t i = cb + lane;
                    if (i < n) __stcs(out + i, ctr_cached_block<NR>(tb, rk, mp, wt, t, cb, lane, __ldcs(in + i)));
                }
            }
            return;
        }
        // ECB / CBC decryption: one state per lane and unit
        auto t_in = [&](uint64_t i) { return MODE == M_CBCD ? __ldg(in + i) : __ldcs(in + i); };
        auto t_out = [&](uint64_t i, uint4 v) {
            uint4 y = cipher_block<NR, DEC>(tb, v, rk);
            if (MODE == M_CBCD) y = xor4(y, i ? __ldg(in + i - 1) : make_uint4(mp.iv[0], mp.iv[1], mp.iv[2], mp.iv[3]));
            return y;
        };
        // kStep units (blocks b .. b + 32*kStep - 1: every claim is a multiple of
        // kStep and kSuper is too, so they are contiguous) per claim, claimed one
        // step ahead: the atomic for step t+2 is issued before step t's rounds
        // and its result is read (shfl) only after them, so its latency hides.
        constexpr uint64_t W = kStep * kUnit;
        uint32_t a = 0;
        if (lane == 0) a = atomicAdd(&q_next, (uint32_t)kStep);
        const uint32_t ucur = __shfl_sync(0xffffffffu, a, 0);
        if (lane == 0) a = atomicAdd(&q_next, (uint32_t)kStep);
        uint32_t unxt = __shfl_sync(0xffffffffu, a, 0);
        uint64_t b = unit_block(ucur);
        if (b >= n) return;
        if (b + W <= n) {
            // whole steps: no per-lane bounds checks (the unit sequence is
            // increasing, so once a step is not whole every later one is past n)
            uint4 v[kStep];
#pragma unroll
            for (int k = 0; k < kStep; k++) v[k] = t_in(b + k * kUnit + lane);
            for (;;) {                      // the next step's states load during this step's rounds
                const uint64_t nb = unit_block(unxt);
                if (nb + W > n) {
#pragma unroll
                    for (int k = 0; k < kStep; k++) __stcs(out + b + k * kUnit + lane, t_out(b + k * kUnit + lane, v[k]));
                    b = nb;
                    break;
                }
                uint4 nv[kStep];
#pragma unroll
                for (int k = 0; k < kStep; k++) nv[k] = t_in(nb + k * kUnit + lane);
                if (lane == 0) a = atomicAdd(&q_next, (uint32_t)kStep);
#pragma unroll
                for (int k = 0; k < kStep; k++) __stcs(out + b + k * kUnit + lane, t_out(b + k * kUnit + lane, v[k]));
                unxt = __shfl_sync(0xffffffffu, a, 0);
                b = nb;
#pragma unroll
                for (int k = 0; k < kStep; k++) v[k] = nv[k];
            }
        }
        if (b < n) {                        // the one partial step (ragged end of the message)
#pragma unroll
            for (int k = 0; k < kStep; k++) {
                const uint64_t i = b + k * kUnit + lane;
                if (i < n) __stcs(out + i, t_out(i, t_in(i)));
            }
        }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegB));
        for (;;) {
            uint32_t u0 = ~0u;
            if (lane == 0) {
                const uint32_t seen = *reinterpret_cast<volatile uint32_t*>(&q_next);
                if (unit_block(seen + (uint32_t)kTailUnits) < n) u0 = atomicAdd(&q_next, 8u);
            }
            u0 = __shfl_sync(0xffffffffu, u0, 0);
            if (u0 == ~0u || unit_block(u0) >= n) break;
            bs_pass<NR, DEC, MODE>(in, out, n, bk, mp, [&](int j) { return unit_block(u0 + j); });
        }
    }
}

constexpr int kBsWarps = 16;

template <int NR, bool DEC>
__global__ void __launch_bounds__(kThreads, 1)
    bs_kernel(const uint4* __restrict__ in, uint4* __restrict__ out, uint64_t n, const __grid_constant__ RK,
              const __grid_constant__ BSK bk, const __grid_constant__ ModeP mp) {
    pdl_launch_dependents();
    pdl_wait();
    // half the warps of the CTA take all registers (16 x 104 + 16 x 24 = 32 x 64)
    if ((threadIdx.x >> 5) >= kBsWarps) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 24;");
        return;
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 104;");
    // warp-granular grid stride over groups of 256 blocks (8 units)
    const uint64_t warps = (uint64_t)gridDim.x * kBsWarps;
    for (uint64_t g = (uint64_t)blockIdx.x * kBsWarps + (threadIdx.x >> 5); g * 256 < n; g += warps)
        bs_pass<NR, DEC, M_ECB>(in, out, n, bk, mp, [&](int j) { return g * 256 + (uint64_t)j * 32; });
}

template <int NR, bool DEC>
KernelInfo hk(int v, int mode) {
    if (v == V_BITSLICE) return {reinterpret_cast<const void*>(&bs_kernel<NR, DEC>), 0};
    if (mode == M_CTR) return {reinterpret_cast<const void*>(&hybrid_kernel<NR, false, M_CTR>), kSmemReplEnc + kCtrTableBytes};
    if (mode == M_CBCD) return {reinterpret_cast<const void*>(&hybrid_kernel<NR, true, M_CBCD>), kSmemReplDec};
    return {reinterpret_cast<const void*>(&hybrid_kernel<NR, DEC, M_ECB>), DEC ? kSmemReplDec : kSmemReplEnc};
}

KernelInfo pick_hybrid(int nr, bool dec, int v, int mode) {
    switch (nr) {
        case 10: return dec ? hk<10, true>(v, mode) : hk<10, false>(v, mode);
        case 12: return dec ? hk<12, true>(v, mode) : hk<12, false>(v, mode);
        case 14: return dec ? hk<14, true>(v, mode) : hk<14, false>(v, mode);
    }
    return {nullptr, 0};
}

void bitslice_keys(const aes_round_keys* rk, int decrypt, BSK* out) {
    bs_expand_round_keys(decrypt ? rk->dk : rk->ek, rk->nr, *out);
}

}  // namespace aesb200
