// aes_ecb.cu -- sm_100a AES-ECB kernels (steps A4..A10 of SURVEY.md 8(a)) and
// the device entry points of the C ABI (include/aes_b200.h).
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
#include <cstring>
#include <mutex>
#include <vector>

#include "aes_b200.h"
#include "aes_tables.h"

namespace aesb200 {

// ---------------------------------------------------------------------------
// Table images (compile time) in global and constant memory
// ---------------------------------------------------------------------------
struct Tables4 {
    uint32_t te[4][256];   // Te0..Te3 (Eqs 22-25)
    uint32_t td[4][256];   // Td0..Td3
    uint32_t si4[256];     // Si[x] replicated in all four bytes
};

constexpr uint32_t rotl32(uint32_t v, int n) { return n ? (v << n) | (v >> (32 - n)) : v; }

constexpr Tables4 build_tables4() {
    Tables4 t{};
    for (int i = 0; i < 4; i++)
        for (int x = 0; x < 256; x++) {
            t.te[i][x] = rotl32(kTables.te0[x], 8 * i);
            t.td[i][x] = rotl32(kTables.td0[x], 8 * i);
        }
    for (int x = 0; x < 256; x++) t.si4[x] = 0x01010101u * kTables.si[x];
    return t;
}

constexpr Tables4 kTables4 = build_tables4();
static_assert(kTables4.te[1][0] == 0x6363C6A5u, "Te1 = rotl(Te0, 8)");

__device__ const Tables4 g_tab = kTables4;     // L2-resident source of the smem fill
__constant__ Tables4 c_tab = kTables4;         // AES_VAR_CONST (the paper's placement)

struct RK {
    uint32_t w[60];
};

constexpr int kThreads = 1024;

// Replicated layout (bytes).  Region C (Si4) is only used by decryption.
constexpr uint32_t kRegion = 65536;
__host__ __device__ constexpr uint32_t off_t(int i) { return (uint32_t)(i >> 1) * kRegion + (uint32_t)(i & 1) * 128u; }
constexpr uint32_t kOffSi = 2 * kRegion;
constexpr size_t kSmemReplEnc = 2 * kRegion;
constexpr size_t kSmemReplDec = 2 * kRegion + 255 * 256 + 128;
constexpr size_t kSmemPlain = (4 * 256 + 256) * 4;

enum { V_REPL = 1, V_PLAIN = 2, V_CONST = 3 };

// ---------------------------------------------------------------------------
// Table access policies: t(i, s, k) = T_i[byte k of s];  si(s, k) = Si4[byte k of s]
// ---------------------------------------------------------------------------
template <int V>
struct Tab;

template <>
struct Tab<V_REPL> {
    const char* sb;
    uint32_t lo;  // lane*4 in byte 0
    __device__ __forceinline__ uint32_t t(int i, uint32_t s, int k) const {
        return *reinterpret_cast<const uint32_t*>(sb + off_t(i) + __byte_perm(lo, s, 0x1140 + 16 * k));
    }
    __device__ __forceinline__ uint32_t si(uint32_t s, int k) const {
        return *reinterpret_cast<const uint32_t*>(sb + kOffSi + __byte_perm(lo, s, 0x1140 + 16 * k));
    }
    template <bool DEC>
    __device__ __forceinline__ static Tab setup(uint32_t* smem) {
        const uint32_t* src = DEC ? &g_tab.td[0][0] : &g_tab.te[0][0];
        uint4* s4 = reinterpret_cast<uint4*>(smem);
        // regions A,B: 32768 words; word w -> x = (w>>6)&255, table i = 2*(w>>14) + ((w>>5)&1)
        // blockDim.x == kThreads: fixed trip counts, fully unrolled so every
        // (L2-resident) table load of a thread is in flight at once
        uint32_t v[8192 / kThreads];
#pragma unroll
        for (int it = 0; it < 8192 / kThreads; it++) {
            int w = 4 * (threadIdx.x + it * kThreads);
            int x = (w >> 6) & 255, i = 2 * (w >> 14) + ((w >> 5) & 1);
            v[it] = __ldg(src + i * 256 + x);
        }
#pragma unroll
        for (int it = 0; it < 8192 / kThreads; it++)
            s4[threadIdx.x + it * kThreads] = make_uint4(v[it], v[it], v[it], v[it]);
        if (DEC) {
#pragma unroll
            for (int it = 0; it < 2048 / kThreads; it++) {
                int q = threadIdx.x + it * kThreads;
                int x = q >> 3, part = q & 7;
                uint32_t u = __ldg(g_tab.si4 + x);
                s4[(kOffSi + x * 256) / 16 + part] = make_uint4(u, u, u, u);
            }
        }
        __syncthreads();
        Tab tb;
        tb.sb = reinterpret_cast<const char*>(smem);
        tb.lo = (threadIdx.x & 31) * 4;
        return tb;
    }
};

template <>
struct Tab<V_PLAIN> {
    const uint32_t* sm;
    __device__ __forceinline__ uint32_t t(int i, uint32_t s, int k) const {
        return sm[i * 256 + ((s >> (8 * k)) & 255)];
    }
    __device__ __forceinline__ uint32_t si(uint32_t s, int k) const {
        return sm[1024 + ((s >> (8 * k)) & 255)];
    }
    template <bool DEC>
    __device__ __forceinline__ static Tab setup(uint32_t* smem) {
        const uint32_t* src = DEC ? &g_tab.td[0][0] : &g_tab.te[0][0];
        for (int w = threadIdx.x; w < 1024; w += blockDim.x) smem[w] = src[w];
        for (int w = threadIdx.x; w < 256; w += blockDim.x) smem[1024 + w] = g_tab.si4[w];
        __syncthreads();
        Tab tb;
        tb.sm = smem;
        return tb;
    }
};

template <bool DEC>
struct ConstSel;
template <>
struct ConstSel<false> {
    __device__ __forceinline__ static uint32_t get(int i, uint32_t x) { return c_tab.te[i][x]; }
};
template <>
struct ConstSel<true> {
    __device__ __forceinline__ static uint32_t get(int i, uint32_t x) { return c_tab.td[i][x]; }
};

template <>
struct Tab<V_CONST> {
    bool dec;
    __device__ __forceinline__ uint32_t t(int i, uint32_t s, int k) const {
        uint32_t x = (s >> (8 * k)) & 255;
        return dec ? ConstSel<true>::get(i, x) : ConstSel<false>::get(i, x);
    }
    __device__ __forceinline__ uint32_t si(uint32_t s, int k) const { return c_tab.si4[(s >> (8 * k)) & 255]; }
    template <bool DEC>
    __device__ __forceinline__ static Tab setup(uint32_t*) {
        Tab tb;
        tb.dec = DEC;
        return tb;
    }
};

// ---------------------------------------------------------------------------
// One block: Algorithm 1 (corrected, R1) with the Eq 26 round
// ---------------------------------------------------------------------------
// A7: one Eq 26 round on the state (s0..s3) with round key k[0..3].
// Encryption: e_j = T0[b0(s_j)] ^ T1[b1(s_{j+1})] ^ T2[b2(s_{j+2})] ^ T3[b3(s_{j+3})] ^ k_j.
// Decryption (equivalent inverse, R12): Td tables with s_j, s_{j-1}, s_{j-2}, s_{j-3}.
template <bool DEC, class TB, class K>
__device__ __forceinline__ void t_round(const TB& tb, uint32_t& s0, uint32_t& s1, uint32_t& s2, uint32_t& s3,
                                        const K& k) {
    uint32_t e0, e1, e2, e3;
    if (!DEC) {
        e0 = tb.t(0, s0, 0) ^ tb.t(1, s1, 1) ^ tb.t(2, s2, 2) ^ tb.t(3, s3, 3) ^ k[0];
        e1 = tb.t(0, s1, 0) ^ tb.t(1, s2, 1) ^ tb.t(2, s3, 2) ^ tb.t(3, s0, 3) ^ k[1];
        e2 = tb.t(0, s2, 0) ^ tb.t(1, s3, 1) ^ tb.t(2, s0, 2) ^ tb.t(3, s1, 3) ^ k[2];
        e3 = tb.t(0, s3, 0) ^ tb.t(1, s0, 1) ^ tb.t(2, s1, 2) ^ tb.t(3, s2, 3) ^ k[3];
    } else {
        e0 = tb.t(0, s0, 0) ^ tb.t(1, s3, 1) ^ tb.t(2, s2, 2) ^ tb.t(3, s1, 3) ^ k[0];
        e1 = tb.t(0, s1, 0) ^ tb.t(1, s0, 1) ^ tb.t(2, s3, 2) ^ tb.t(3, s2, 3) ^ k[1];
        e2 = tb.t(0, s2, 0) ^ tb.t(1, s1, 1) ^ tb.t(2, s0, 2) ^ tb.t(3, s3, 3) ^ k[2];
        e3 = tb.t(0, s3, 0) ^ tb.t(1, s2, 1) ^ tb.t(2, s1, 2) ^ tb.t(3, s0, 3) ^ k[3];
    }
    s0 = e0; s1 = e1; s2 = e2; s3 = e3;
}

// A8: final round = SubBytes + ShiftRows + AddRoundKey, no MixColumns (R1, R14).
template <bool DEC, class TB, class K>
__device__ __forceinline__ uint4 final_round(const TB& tb, uint32_t s0, uint32_t s1, uint32_t s2, uint32_t s3,
                                             const K& k) {
    uint4 o;
    if (!DEC) {
        // S[x] sits in byte 0 of Te2, byte 1 of Te3, byte 2 of Te0, byte 3 of Te1
#define AES_FINAL_E(a, b, c, d) \
    (((tb.t(2, a, 0) & 0x000000FFu) | (tb.t(3, b, 1) & 0x0000FF00u) | (tb.t(0, c, 2) & 0x00FF0000u) | \
      (tb.t(1, d, 3) & 0xFF000000u)))
        o.x = AES_FINAL_E(s0, s1, s2, s3) ^ k[0];
        o.y = AES_FINAL_E(s1, s2, s3, s0) ^ k[1];
        o.z = AES_FINAL_E(s2, s3, s0, s1) ^ k[2];
        o.w = AES_FINAL_E(s3, s0, s1, s2) ^ k[3];
#undef AES_FINAL_E
    } else {
#define AES_FINAL_D(a, b, c, d) \
    (((tb.si(a, 0) & 0x000000FFu) | (tb.si(b, 1) & 0x0000FF00u) | (tb.si(c, 2) & 0x00FF0000u) | \
      (tb.si(d, 3) & 0xFF000000u)))
        o.x = AES_FINAL_D(s0, s3, s2, s1) ^ k[0];
        o.y = AES_FINAL_D(s1, s0, s3, s2) ^ k[1];
        o.z = AES_FINAL_D(s2, s1, s0, s3) ^ k[2];
        o.w = AES_FINAL_D(s3, s2, s1, s0) ^ k[3];
#undef AES_FINAL_D
    }
    return o;
}

// Round key r as an indexable view of the by-value parameter (constant bank).
struct KeyAt {
    const RK& rk;
    int r;
    __device__ __forceinline__ uint32_t operator[](int j) const { return rk.w[4 * r + j]; }
};

// One block: Algorithm 1 (corrected, R1) with the Eq 26 round.
template <int NR, bool DEC, class TB>
__device__ __forceinline__ uint4 cipher_block(const TB& tb, uint4 v, const RK& rk) {
    // A6: round-0 AddRoundKey (Eq 21)
    uint32_t s0 = v.x ^ rk.w[0], s1 = v.y ^ rk.w[1], s2 = v.z ^ rk.w[2], s3 = v.w ^ rk.w[3];
#pragma unroll
    for (int r = 1; r < NR; r++) t_round<DEC>(tb, s0, s1, s2, s3, KeyAt{rk, r});   // A7
    return final_round<DEC>(tb, s0, s1, s2, s3, KeyAt{rk, NR});                    // A8
}

// ---------------------------------------------------------------------------
// Kernels: persistent grid-stride, SPT states per thread per trip.
//   ecb_kernel          C_i = E(P_i) / P_i = D(C_i)                (Eq 1)
//   ctr_kernel          C_i = P_i ^ E(ctr0 + i), BE 128-bit counter  (Eq 5, R24)
//   cbc_decrypt_kernel  P_i = D(C_i) ^ C_{i-1}, C_{-1} = IV          (Eq 2, R25)
// ---------------------------------------------------------------------------
enum { M_ECB = 0, M_CTR = 1, M_CBCD = 2 };

struct ModeP {
    uint32_t iv[4];    // CBC: IV as LE column words
    uint64_t ctr_hi;   // CTR: counter of block 0 of this launch, big-endian value,
    uint64_t ctr_lo;   //      split into high / low 64 bits
};

__device__ __forceinline__ uint4 counter_block(const ModeP& mp, uint64_t i) {
    uint64_t lo = mp.ctr_lo + i;
    uint64_t hi = mp.ctr_hi + (lo < mp.ctr_lo ? 1ull : 0ull);   // carry, wraps mod 2^128
    // block bytes 0..7 = hi big-endian, 8..15 = lo big-endian; columns are LE words
    return make_uint4(__byte_perm((uint32_t)(hi >> 32), 0, 0x0123), __byte_perm((uint32_t)hi, 0, 0x0123),
                      __byte_perm((uint32_t)(lo >> 32), 0, 0x0123), __byte_perm((uint32_t)lo, 0, 0x0123));
}

__device__ __forceinline__ uint4 xor4(uint4 a, uint4 b) {
    return make_uint4(a.x ^ b.x, a.y ^ b.y, a.z ^ b.z, a.w ^ b.w);
}

template <int NR, bool DEC, int V, int SPT, int MODE>
__device__ __forceinline__ void aes_body(const uint4* __restrict__ in, uint4* __restrict__ out, uint64_t n,
                                         const RK& rk, const ModeP& mp) {
    extern __shared__ __align__(16) uint32_t smem[];
    const Tab<V> tb = Tab<V>::template setup<DEC>(smem);   // A4
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += SPT * T) {
        uint4 v[SPT], w[SPT];
#pragma unroll
        for (int k = 0; k < SPT; k++) {
            const uint64_t j = i + k * T;
            if (j < n) {                                                   // A5
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
        for (int k = 0; k < SPT; k++) {
            const uint64_t j = i + k * T;
            if (j < n) __stcs(out + j, MODE == M_ECB ? v[k] : xor4(v[k], w[k]));   // A9
        }
    }
}

template <int NR, bool DEC, int V, int SPT>
__global__ void __launch_bounds__(kThreads, 1)
    ecb_kernel(const uint4* __restrict__ in, uint4* __restrict__ out, uint64_t n, const __grid_constant__ RK rk) {
    aes_body<NR, DEC, V, SPT, M_ECB>(in, out, n, rk, ModeP{});
}

template <int NR>
__global__ void __launch_bounds__(kThreads, 1)
    ctr_kernel(const uint4* __restrict__ in, uint4* __restrict__ out, uint64_t n, const __grid_constant__ RK rk,
               const __grid_constant__ ModeP mp) {
    aes_body<NR, false, V_REPL, 1, M_CTR>(in, out, n, rk, mp);
}

template <int NR>
__global__ void __launch_bounds__(kThreads, 1)
    cbc_decrypt_kernel(const uint4* __restrict__ in, uint4* __restrict__ out, uint64_t n,
                       const __grid_constant__ RK rk, const __grid_constant__ ModeP mp) {
    aes_body<NR, true, V_REPL, 1, M_CBCD>(in, out, n, rk, mp);
}

// ---------------------------------------------------------------------------
// Batched multi-message ECB (aes_ecb_batch): many messages, each with its own
// key, in ONE launch -- the paper's file-sized workloads at
// bulk rate instead of one launch per file.  Segment s covers global blocks
// [first, first + n); a warp's 32 consecutive global blocks find their
// segment with one warp-uniform binary search (broadcast loads) plus a short
// forward walk; round keys are read per round from the (L1-resident)
// descriptor area: a broadcast when the warp is inside one message.
// ---------------------------------------------------------------------------
struct BatchSeg {
    uint64_t in_off, out_off;   // byte offsets from in_base / out_base
    uint64_t first, n;          // global block range
    uint32_t key, pad;          // index into the key words (60 per key)
};

struct KeyVec {
    uint4 k;   // one round key, fetched with a single LDS.128 (a broadcast within a message)
    __device__ __forceinline__ uint32_t operator[](int j) const { return j == 0 ? k.x : j == 1 ? k.y : j == 2 ? k.z : k.w; }
};

constexpr int kBatchMaxKeys = 128;   // 128 x 240 B = 30 KiB of key schedules staged in shared memory

// Each CTA owns one contiguous range of global blocks; its 1024 threads walk it
// 1024 consecutive blocks per trip, so the segment of a warp only moves
// forward: found once by a warp-uniform binary search, then advanced by a
// short forward walk (broadcast loads).
template <int NR, bool DEC>
__global__ void __launch_bounds__(kThreads, 1)
    batch_kernel(const char* __restrict__ in_base, char* __restrict__ out_base, const BatchSeg* __restrict__ segs,
                 uint32_t nsegs, uint64_t total, const uint32_t* __restrict__ keyw, int nkeys) {
    extern __shared__ __align__(16) uint32_t smem[];
    const Tab<V_REPL> tb = Tab<V_REPL>::template setup<DEC>(smem);   // ends with __syncthreads
    uint32_t* skeys = smem + (DEC ? kSmemReplDec : kSmemReplEnc) / 4;
    for (int w = threadIdx.x; w < 60 * nkeys; w += blockDim.x) skeys[w] = __ldg(keyw + w);
    __syncthreads();
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
    bool have = false;
    uint4 v = make_uint4(0, 0, 0, 0);
    uint4* op = nullptr;
    const uint4* kp = nullptr;
    auto fetch = [&](uint64_t base) {
        while (base >= __ldg(&segs[seg].first) + __ldg(&segs[seg].n)) seg++;   // warp-uniform advance
        const uint64_t i = base + lane;
        have = i < c1;
        if (!have) return;
        uint32_t sidx = seg;
        while (i >= __ldg(&segs[sidx].first) + __ldg(&segs[sidx].n)) sidx++;
        const BatchSeg* sg = segs + sidx;
        const uint64_t local = i - __ldg(&sg->first);
        v = __ldcs(reinterpret_cast<const uint4*>(in_base + __ldg(&sg->in_off)) + local);
        op = reinterpret_cast<uint4*>(out_base + __ldg(&sg->out_off)) + local;
        kp = reinterpret_cast<const uint4*>(skeys + 60u * __ldg(&sg->key));
    };
    fetch(w0);
    while (w0 < c1) {
        const bool chave = have;
        const uint4 cv = v;
        uint4* const cop = op;
        const uint4* const ckp = kp;
        w0 += blockDim.x;
        if (w0 < c1) fetch(w0);
        if (chave) {
            const uint4 k0 = ckp[0];
            uint32_t s0 = cv.x ^ k0.x, s1 = cv.y ^ k0.y, s2 = cv.z ^ k0.z, s3 = cv.w ^ k0.w;
#pragma unroll
            for (int r = 1; r < NR; r++) t_round<DEC>(tb, s0, s1, s2, s3, KeyVec{ckp[r]});
            __stcs(cop, final_round<DEC>(tb, s0, s1, s2, s3, KeyVec{ckp[NR]}));
        }
    }
}

// Debug/pin kernel (aes_ecb_trace): the state after ARK(0) and `rounds` rounds
// of the SAME t_round / final_round code the production kernels inline, one
// state per thread.  rounds = NR gives the full cipher.
template <int NR, bool DEC>
__global__ void __launch_bounds__(kThreads, 1)
    trace_kernel(const uint4* __restrict__ in, uint4* __restrict__ out, uint64_t n, const __grid_constant__ RK rk,
                 int rounds) {
    extern __shared__ __align__(16) uint32_t smem[];
    const Tab<V_REPL> tb = Tab<V_REPL>::template setup<DEC>(smem);
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
// Host side: kernel registry, per-device attribute cache, validation, launch
// ---------------------------------------------------------------------------
struct KernelInfo {
    const void* fn;
    size_t smem;
};

template <int NR, bool DEC, int V, int SPT>
KernelInfo kinfo() {
    size_t sm = V == V_REPL ? (DEC ? kSmemReplDec : kSmemReplEnc) : V == V_PLAIN ? kSmemPlain : 0;
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
        if (v == V_PLAIN) return kinfo<NR, DEC, V_PLAIN, 1>();
        if (v == V_CONST) return kinfo<NR, DEC, V_CONST, 1>();
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

KernelInfo pick_mode(int nr, int mode) {
    const void* f = nullptr;
    if (mode == M_CTR) {
        f = nr == 10 ? (const void*)&ctr_kernel<10> : nr == 12 ? (const void*)&ctr_kernel<12>
                                                               : (const void*)&ctr_kernel<14>;
        return {f, kSmemReplEnc};
    }
    f = nr == 10 ? (const void*)&cbc_decrypt_kernel<10> : nr == 12 ? (const void*)&cbc_decrypt_kernel<12>
                                                                   : (const void*)&cbc_decrypt_kernel<14>;
    return {f, kSmemReplDec};
}

thread_local int t_last_cuda_error = 0;

inline aes_status cuda_fail(cudaError_t e) {
    t_last_cuda_error = (int)e;
    return AES_ECUDA;
}

// Per-(device, kernel) resident-CTA count; set the dynamic-smem attribute once.
constexpr int kMaxDev = 64;
std::mutex g_attr_mu;
struct AttrEntry {
    const void* fn;
    int occ;
};
AttrEntry g_attr[kMaxDev][128];
int g_nsm[kMaxDev];

aes_status resident_ctas(int dev, const KernelInfo& ki, int* occ, int* nsm) {
    if (dev < 0 || dev >= kMaxDev) return AES_ERANGE;
    std::lock_guard<std::mutex> g(g_attr_mu);
    if (!g_nsm[dev]) {
        int v = 0;
        cudaError_t e = cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return cuda_fail(e);
        g_nsm[dev] = v;
    }
    *nsm = g_nsm[dev];
    int slot = -1;
    for (int s = 0; s < 128; s++) {
        if (g_attr[dev][s].fn == ki.fn) { *occ = g_attr[dev][s].occ; return AES_OK; }
        if (!g_attr[dev][s].fn) { slot = s; break; }
    }
    if (slot < 0) return AES_ERANGE;
    cudaError_t e = cudaFuncSetAttribute(ki.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ki.smem);
    if (e != cudaSuccess) return cuda_fail(e);
    int o = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, ki.fn, kThreads, ki.smem);
    if (e != cudaSuccess) return cuda_fail(e);
    if (o < 1) o = 1;
    g_attr[dev][slot].fn = ki.fn;
    g_attr[dev][slot].occ = o;
    *occ = o;
    return AES_OK;
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

aes_status launch(const aes_round_keys* rk, int nr, int decrypt, const void* in, void* out, uint64_t nblocks,
                  cudaStream_t stream, const aes_launch_config* cfg, bool check_ptrs, int mode = M_ECB,
                  const ModeP* mp = nullptr) {
    aes_status st = validate_keys(rk, nr);
    if (st) return st;
    int variant = cfg ? cfg->variant : AES_VAR_DEFAULT;
    int spt = cfg ? cfg->states_per_thread : 0;
    int grid_req = cfg ? cfg->grid : 0;
    if (variant == AES_VAR_DEFAULT) variant = V_REPL;   // measured best
    if (spt == 0) spt = 1;                              // S = 1, 2, 4 measure within 1 %
    if (grid_req < 0) return AES_ERANGE;
    KernelInfo ki = mode == M_ECB ? pick(nr, decrypt != 0, variant, spt) : pick_mode(nr, mode);
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
    // Spread small and medium buffers over every SM (at least one full warp of
    // states per CTA) instead of packing 1024 states into each CTA: the per-CTA
    // table fill is ~0.5 us, the lookups are what must be parallel.
    uint64_t per_cta = 32ull * spt;
    uint64_t want = (nblocks + per_cta - 1) / per_cta;
    uint64_t cap = grid_req ? (uint64_t)grid_req : (uint64_t)nsm * occ;
    unsigned grid = (unsigned)(want < cap ? want : cap);
    RK k;
    std::memcpy(k.w, decrypt ? rk->dk : rk->ek, sizeof k.w);
    const uint4* pin = static_cast<const uint4*>(in);
    uint4* pout = static_cast<uint4*>(out);
    ModeP m = mp ? *mp : ModeP{};
    void* args[] = {(void*)&pin, (void*)&pout, (void*)&nblocks, (void*)&k, (void*)&m};
    e = cudaLaunchKernel(ki.fn, dim3(grid), dim3(kThreads), args, ki.smem, stream);
    if (e != cudaSuccess) return cuda_fail(e);
    return AES_OK;
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
    e = cudaLaunchKernel(f, dim3((unsigned)(want < cap ? want : cap)), dim3(kThreads), args, ki.smem,
                         (cudaStream_t)stream);
    return e == cudaSuccess ? AES_OK : cuda_fail(e);
}

aes_status aes_ecb_batch(const aes_round_keys* keys, int nkeys, int decrypt, const aes_segment* segs, uint32_t nsegs,
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
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e);
    aes_status st;
    if ((st = check_device_ptr(in_base, dev))) return st;
    if (out_base != in_base && (st = check_device_ptr(out_base, dev))) return st;
    const void* f = nullptr;
    if (nr == 10) f = decrypt ? (const void*)&batch_kernel<10, true> : (const void*)&batch_kernel<10, false>;
    else if (nr == 12) f = decrypt ? (const void*)&batch_kernel<12, true> : (const void*)&batch_kernel<12, false>;
    else f = decrypt ? (const void*)&batch_kernel<14, true> : (const void*)&batch_kernel<14, false>;
    KernelInfo ki{f, (decrypt ? kSmemReplDec : kSmemReplEnc) + 240 * kBatchMaxKeys};
    if ((st = resident_ctas(dev, ki, &occ, &nsm))) return st;
    const size_t smem = (decrypt ? kSmemReplDec : kSmemReplEnc) + 240ull * nkeys;
    // descriptors: segments, then 60 key words per key (ek or dk), in one
    // stream-ordered allocation that is freed after the kernel on `stream`
    const size_t seg_bytes = sizeof(BatchSeg) * nsegs, key_bytes = 240ull * nkeys;
    std::vector<char> host(seg_bytes + key_bytes);
    std::memcpy(host.data(), hs.data(), seg_bytes);
    for (int k = 0; k < nkeys; k++)
        std::memcpy(host.data() + seg_bytes + 240ull * k, decrypt ? keys[k].dk : keys[k].ek, 240);
    cudaStream_t cs = (cudaStream_t)stream;
    cudaMemPool_t pool;
    if ((st = desc_pool(dev, &pool))) return st;
    void* d = nullptr;
    if ((e = cudaMallocFromPoolAsync(&d, host.size(), pool, cs)) != cudaSuccess) return cuda_fail(e);
    if ((e = cudaMemcpyAsync(d, host.data(), host.size(), cudaMemcpyHostToDevice, cs)) != cudaSuccess) {
        cudaFreeAsync(d, cs);
        return cuda_fail(e);
    }
    const char* pin = static_cast<const char*>(in_base);
    char* pout = static_cast<char*>(out_base);
    const BatchSeg* dsegs = static_cast<const BatchSeg*>(d);
    const uint32_t* dkeys = reinterpret_cast<const uint32_t*>(static_cast<char*>(d) + seg_bytes);
    void* args[] = {(void*)&pin, (void*)&pout, (void*)&dsegs, (void*)&nsegs, (void*)&total, (void*)&dkeys,
                    (void*)&nkeys};
    uint64_t want = (total + 31) / 32, cap = (uint64_t)nsm * occ;
    e = cudaLaunchKernel(f, dim3((unsigned)(want < cap ? want : cap)), dim3(kThreads), args, smem, cs);
    cudaError_t e2 = cudaFreeAsync(d, cs);
    if (e != cudaSuccess) return cuda_fail(e);
    return e2 == cudaSuccess ? AES_OK : cuda_fail(e2);
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

// --------------------------------------------------------------------------
// Host-resident pipeline (NEXT-3)
// --------------------------------------------------------------------------
struct aes_pipeline {
    int device;
    uint64_t chunk;
    int depth;
    void* dbuf[8];
    cudaStream_t st[8];
};

aes_status aes_pipeline_destroy(aes_pipeline* p) {
    if (!p) return AES_ENULL;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(p->device);
    for (int k = 0; k < p->depth; k++) {
        if (p->st[k]) cudaStreamSynchronize(p->st[k]), cudaStreamDestroy(p->st[k]);
        if (p->dbuf[k]) cudaFree(p->dbuf[k]);
    }
    cudaSetDevice(prev);
    delete p;
    return AES_OK;
}

aes_status aes_pipeline_create(uint64_t chunk_bytes, int depth, aes_pipeline** out) {
    if (!out) return AES_ENULL;
    *out = nullptr;
    if (chunk_bytes < 16 || (chunk_bytes & 15) || depth < 1 || depth > 8) return AES_ERANGE;
    aes_pipeline* p = new aes_pipeline();
    p->chunk = chunk_bytes;
    p->depth = depth;
    cudaError_t e = cudaGetDevice(&p->device);
    if (e != cudaSuccess) { delete p; return cuda_fail(e); }
    for (int k = 0; k < depth; k++) {
        e = cudaMalloc(&p->dbuf[k], chunk_bytes);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->st[k], cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            aes_pipeline_destroy(p);
            return cuda_fail(e);
        }
    }
    *out = p;
    return AES_OK;
}

aes_status aes_pipeline_run(aes_pipeline* p, const aes_round_keys* rk, int nr, int decrypt, const void* in_host,
                            void* out_host, uint64_t nblocks) {
    if (!p) return AES_ENULL;
    aes_status st = validate_keys(rk, nr);
    if (st) return st;
    if (nblocks == 0) return AES_OK;
    if (!in_host || !out_host) return AES_ENULL;
    if (nblocks > (UINT64_MAX >> 4)) return AES_ERANGE;
    uint64_t bytes = nblocks << 4;
    uintptr_t a = (uintptr_t)in_host, b = (uintptr_t)out_host;
    if (a > UINTPTR_MAX - bytes || b > UINTPTR_MAX - bytes) return AES_ERANGE;
    if (a != b && a < b + bytes && b < a + bytes) return AES_EOVERLAP;
    int prev = 0;
    cudaError_t e = cudaGetDevice(&prev);
    if (e != cudaSuccess) return cuda_fail(e);
    if (prev != p->device && (e = cudaSetDevice(p->device)) != cudaSuccess) return cuda_fail(e);
    const char* src = static_cast<const char*>(in_host);
    char* dst = static_cast<char*>(out_host);
    uint64_t nchunks = (bytes + p->chunk - 1) / p->chunk;
    for (uint64_t c = 0; c < nchunks && st == AES_OK; c++) {
        int k = (int)(c % (uint64_t)p->depth);
        uint64_t off = c * p->chunk;
        uint64_t len = bytes - off < p->chunk ? bytes - off : p->chunk;
        e = cudaMemcpyAsync(p->dbuf[k], src + off, len, cudaMemcpyHostToDevice, p->st[k]);
        if (e != cudaSuccess) { st = cuda_fail(e); break; }
        st = launch(rk, nr, decrypt, p->dbuf[k], p->dbuf[k], len >> 4, p->st[k], nullptr, false);
        if (st) break;
        e = cudaMemcpyAsync(dst + off, p->dbuf[k], len, cudaMemcpyDeviceToHost, p->st[k]);
        if (e != cudaSuccess) { st = cuda_fail(e); break; }
    }
    for (int k = 0; k < p->depth; k++) {
        e = cudaStreamSynchronize(p->st[k]);
        if (e != cudaSuccess && st == AES_OK) st = cuda_fail(e);
    }
    if (prev != p->device) cudaSetDevice(prev);
    return st;
}

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
    }
    return "AES_?: unknown status";
}

int aes_last_cuda_error(void) { return t_last_cuda_error; }
int aes_abi_version(void) { return AES_B200_ABI_VERSION; }

}  // extern "C"
