// aes_device.cuh -- device building blocks shared by every kernel TU of
// libaes_b200.so: compile-time table images (A3), the shared-memory table
// policies (A4), the Eq 26 round and the final round (A6-A8).
//
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
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "aes_host.h"
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

static __device__ const Tables4 g_tab = kTables4;     // L2-resident source of the smem fill
static __constant__ Tables4 c_tab = kTables4;         // AES_VAR_CONST (the paper's placement)

struct RK {
    uint32_t w[60];
};


// Replicated layout (bytes).  Region C (Si4) is only used by decryption.
constexpr uint32_t kRegion = 65536;
__host__ __device__ constexpr uint32_t off_t(int i) { return (uint32_t)(i >> 1) * kRegion + (uint32_t)(i & 1) * 128u; }
constexpr uint32_t kOffSi = 2 * kRegion;
constexpr size_t kSmemReplEnc = 2 * kRegion;
constexpr size_t kSmemReplDec = 2 * kRegion + 255 * 256 + 128;
constexpr size_t kSmemPlain = (4 * 256 + 256) * 4;
constexpr size_t kSmemRot = 255 * 256 + 256;   // one replicated table (+ Si4 for decryption) in a 64 KiB region

enum { V_REPL = 1, V_PLAIN = 2, V_CONST = 3, V_REPL_TMA = 4, V_ROT = 5, V_GLOBAL = 6, V_HYBRID = 7, V_BITSLICE = 8 };

// ---------------------------------------------------------------------------
// Programmatic dependent launch (PDL).  Every kernel lets the next kernel of
// its stream be scheduled at once (launch_dependents) and waits for the
// previous one only after its own table fill (pdl_wait), so back-to-back
// launches overlap the next launch's latency and 128-192 KiB prologue with
// this one's tail.  Both are no-ops when the launch carries no PDL attribute.
// All reads and writes of mutable global memory come after pdl_wait (the
// table fill before it reads only the immutable g_tab image).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ---------------------------------------------------------------------------
// Work split of n blocks over the grid (A10).  Whole trips of TS = SPT * grid
// threads are walked grid-stride (each warp access = 512 contiguous bytes, one
// moving DRAM window).  The remainder rem < TS -- the whole message when it is
// small -- is cut into per-CTA contiguous, warp-aligned chunks of
// c = ceil(rem / grid) rounded up to 32 blocks (c <= SPT * blockDim), so every
// CTA that paid its table fill gets work instead of the first rem/1024 CTAs
// taking all of it.
// ---------------------------------------------------------------------------
struct Split {
    uint64_t full;    // blocks [0, full) are walked grid-stride with stride TS
    uint64_t tbase;   // this CTA's tail chunk starts at tbase ...
    uint32_t tlen;    // ... and holds tlen blocks (0 <= tlen <= c)
};

__device__ __forceinline__ Split split_work(uint64_t n, uint64_t TS) {
    Split sp;
    sp.full = n - n % TS;
    const uint64_t rem = n - sp.full;
    const uint64_t c = ((rem + gridDim.x - 1) / gridDim.x + 31) & ~31ull;
    const uint64_t b0 = (uint64_t)blockIdx.x * c;
    sp.tbase = sp.full + b0;
    sp.tlen = b0 >= rem ? 0u : (uint32_t)(rem - b0 < c ? rem - b0 : c);
    return sp;
}

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

// One lane-replicated table T0 (Td0) and T_i[x] = rotl(T0[x], 8i) computed by a
// funnel shift per lookup ("a single Te0 x 32 replicas
// plus __byte_perm / funnel-shift rotations"): 4x less shared memory, one more
// ALU op for 3 of every 4 lookups.  Si4 sits in the other half of each row.
template <>
struct Tab<V_ROT> {
    const char* sb;
    uint32_t lo;
    __device__ __forceinline__ uint32_t t(int i, uint32_t s, int k) const {
        const uint32_t v = *reinterpret_cast<const uint32_t*>(sb + __byte_perm(lo, s, 0x1140 + 16 * k));
        return i ? __funnelshift_l(v, v, 8 * i) : v;
    }
    __device__ __forceinline__ uint32_t si(uint32_t s, int k) const {
        return *reinterpret_cast<const uint32_t*>(sb + 128 + __byte_perm(lo, s, 0x1140 + 16 * k));
    }
    template <bool DEC>
    __device__ __forceinline__ static Tab setup(uint32_t* smem) {
        const uint32_t* src = DEC ? &g_tab.td[0][0] : &g_tab.te[0][0];
        uint4* s4 = reinterpret_cast<uint4*>(smem);
#pragma unroll
        for (int it = 0; it < 2048 / kThreads; it++) {     // 256 rows x 8 uint4 of T0
            int q = threadIdx.x + it * kThreads, x = q >> 3, part = q & 7;
            uint32_t v = __ldg(src + x);
            s4[x * 16 + part] = make_uint4(v, v, v, v);
            if (DEC) {
                uint32_t u = __ldg(g_tab.si4 + x);
                s4[x * 16 + 8 + part] = make_uint4(u, u, u, u);
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

// Tables left in global memory and read through the read-only L1 path
// (__ldg, LDG.E.CONSTANT): the fourth placement of the NEXT-2 ablation.  The
// 4 KiB (+1 KiB Si4) image stays L1-resident; a warp's 32 divergent addresses
// cost one L1 tag lookup per distinct 128-byte line.
template <>
struct Tab<V_GLOBAL> {
    const uint32_t* t4;
    __device__ __forceinline__ uint32_t t(int i, uint32_t s, int k) const {
        return __ldg(t4 + i * 256 + ((s >> (8 * k)) & 255));
    }
    __device__ __forceinline__ uint32_t si(uint32_t s, int k) const { return __ldg(g_tab.si4 + ((s >> (8 * k)) & 255)); }
    template <bool DEC>
    __device__ __forceinline__ static Tab setup(uint32_t*) {
        Tab tb;
        tb.t4 = DEC ? &g_tab.td[0][0] : &g_tab.te[0][0];
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
// Modes (NEXT-1 CTR, NEXT-4 CBC decryption): parameters and shared pieces
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

// CTR with counter-mode caching (Bernstein-Schwabe): the counters of 256
// consecutive blocks differ only in byte 15 (row 3 of column 3), so in round 1
// only column 0 depends on it (one Te3 lookup) and in round 2 each column has
// exactly one varying input byte (four lookups); everything else is a
// per-256-block-group constant (8 words: P0, e1..e3 of round 1 and Q0..Q3 of
// round 2), so every block needs 1 + 4 + 16*(NR-3) + 16 lookups instead of
// 16*NR (133 vs 160 for AES-128).
constexpr size_t kCtrTableBytes = (kThreads / 32) * 32 * 8 * 4;   // 32 warps x 32 entries x 8 words = 32 KiB

// Group constants (8 words) of the 256-block counter group starting at the
// 128-bit counter (ghi:glo) with byte 15 = 0.
template <class TB>
__device__ __forceinline__ void ctr_group_constants(const TB& tb, const RK& rk, uint64_t ghi, uint64_t glo,
                                                    uint32_t* dst) {
    // representative counter (byte 15 = 0), round 0
    const uint32_t s0 = __byte_perm((uint32_t)(ghi >> 32), 0, 0x0123) ^ rk.w[0];
    const uint32_t s1 = __byte_perm((uint32_t)ghi, 0, 0x0123) ^ rk.w[1];
    const uint32_t s2 = __byte_perm((uint32_t)(glo >> 32), 0, 0x0123) ^ rk.w[2];
    const uint32_t s3 = __byte_perm((uint32_t)glo, 0, 0x0123) ^ rk.w[3];
    // round 1: e1..e3 do not see byte 15; e0 = P0 ^ Te3[byte 3 of s3]
    const uint32_t P0 = tb.t(0, s0, 0) ^ tb.t(1, s1, 1) ^ tb.t(2, s2, 2) ^ rk.w[4];
    const uint32_t e1 = tb.t(0, s1, 0) ^ tb.t(1, s2, 1) ^ tb.t(2, s3, 2) ^ tb.t(3, s0, 3) ^ rk.w[5];
    const uint32_t e2 = tb.t(0, s2, 0) ^ tb.t(1, s3, 1) ^ tb.t(2, s0, 2) ^ tb.t(3, s1, 3) ^ rk.w[6];
    const uint32_t e3 = tb.t(0, s3, 0) ^ tb.t(1, s0, 1) ^ tb.t(2, s1, 2) ^ tb.t(3, s2, 3) ^ rk.w[7];
    // round 2: f_j = Q_j ^ (the one lookup of a byte of e0)
    const uint32_t Q0 = tb.t(1, e1, 1) ^ tb.t(2, e2, 2) ^ tb.t(3, e3, 3) ^ rk.w[8];
    const uint32_t Q1 = tb.t(0, e1, 0) ^ tb.t(1, e2, 1) ^ tb.t(2, e3, 2) ^ rk.w[9];
    const uint32_t Q2 = tb.t(0, e2, 0) ^ tb.t(1, e3, 1) ^ tb.t(3, e1, 3) ^ rk.w[10];
    const uint32_t Q3 = tb.t(0, e3, 0) ^ tb.t(2, e1, 2) ^ tb.t(3, e2, 3) ^ rk.w[11];
    uint4* gw = reinterpret_cast<uint4*>(dst);
    gw[0] = make_uint4(P0, e1, e2, e3);
    gw[1] = make_uint4(Q0, Q1, Q2, Q3);
}


// Lane `lane` of a warp fills entry `lane` of the warp's 32-entry group table
// wt: the constants of group (lane & 1) (0: the group holding block tcb, 1: the
// next one) of the 32-block run starting at block tcb -- the run of trip
// (lane >> 1) of the warp's next 16.
template <class TB>
__device__ __forceinline__ void ctr_fill_group(const TB& tb, const RK& rk, const ModeP& mp, uint64_t tcb,
                                               uint32_t lane, uint32_t* wt) {
    const uint64_t lo_c = mp.ctr_lo + tcb;
    const uint64_t hi_c = mp.ctr_hi + (lo_c < mp.ctr_lo ? 1ull : 0ull);
    const uint64_t g0 = lo_c & ~0xffull;
    const uint64_t glo = g0 + 256ull * (lane & 1);
    ctr_group_constants(tb, rk, hi_c + (glo < g0 ? 1ull : 0ull), glo, wt + 8 * lane);
}

// Output block cb + lane of a 32-block run (trip `trip` of the table) in CTR
// mode with the cached group constants: 1 + 4 + 16*(NR-3) + 16 lookups.
template <int NR, class TB>
__device__ __forceinline__ uint4 ctr_cached_block(const TB& tb, const RK& rk, const ModeP& mp, const uint32_t* wt,
                                                  uint32_t trip, uint64_t cb, uint32_t lane, uint4 p) {
    const uint32_t off = (uint32_t)((mp.ctr_lo + cb) & 0xff) + lane;   // < 256 + 32
    const uint4* c = reinterpret_cast<const uint4*>(wt + 8 * (2 * trip + (off >> 8)));
    const uint4 c0 = c[0], c1 = c[1];
    const uint32_t x = (off & 0xff) ^ (rk.w[3] >> 24);                 // byte 15 of this counter ^ k0
    const uint32_t e0 = c0.x ^ tb.t(3, x << 24, 3);
    uint32_t f0 = c1.x ^ tb.t(0, e0, 0), f1 = c1.y ^ tb.t(3, e0, 3);
    uint32_t f2 = c1.z ^ tb.t(2, e0, 2), f3 = c1.w ^ tb.t(1, e0, 1);
#pragma unroll
    for (int r = 3; r < NR; r++) t_round<false>(tb, f0, f1, f2, f3, KeyAt{rk, r});
    return xor4(p, final_round<false>(tb, f0, f1, f2, f3, KeyAt{rk, NR}));
}

}  // namespace aesb200
