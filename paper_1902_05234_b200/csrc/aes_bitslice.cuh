// aes_bitslice.cuh -- bitsliced AES for the hybrid kernel's ALU-only warps.
//
// Why: the T-table rounds (Eq 26) are
// bound by the shared-memory data path (16*Nr lookups per block, 1 wavefront
// per clock per SM) and leave about a quarter of the ALU pipe idle.  A few
// warps per CTA that evaluate the same cipher WITHOUT any lookup -- SubBytes
// as a Boolean circuit over bitsliced words -- turn that idle ALU time into
// extra blocks.  The result is bit-identical to the T-table path (both are
// FIPS-197 Cipher / InvCipher; checked against the oracle by the GPU parity
// tests and here by static_asserts on the FIPS-197 App. C vectors).
//
// Representation ("row-sliced", 8 blocks per thread).  Thread holds 8 blocks
// j = 0..7 as 32 words R[r][b] (r = AES row 0..3, b = bit 0..7 of the byte,
// b = 0 the LSB): bit 8c + j of R[r][b] is bit b of byte (r, c) of block j
// (byte r + 4c of the block, R9).  Then
//   SubBytes      = the S-box circuit on the 8 words of each row (4 circuits
//                   cover all 16 bytes of all 8 blocks; aes_bs_sbox.inc),
//   ShiftRows     = rotate row r's words right by 8r bits (column c <- c + r),
//   MixColumns    = XORs between the row groups (no rotation: a column's
//                   four bytes sit at the same bit positions of the 4 rows),
//   AddRoundKey   = XOR with the bitsliced round key (field c of K[r][b] is
//                   0xFF when bit b of key byte (r, c) is set; built on the
//                   host and passed by value, so the XOR takes a constant-bank
//                   operand).
// Packing: an 8x8 bit transpose (3 SWAPMOVE stages) per column and a 4x4
// byte transpose (PRMT) per bit; unpacking is the same two involutions.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "aes_tables.h"

namespace aesb200 {

// One 3-input LUT (LOP3.LUT, immediate = truth table over a=0xF0, b=0xCC, c=0xAA).
// The device branch is inline PTX (not a constant expression); constexpr
// evaluation only ever runs the host branch.
#pragma nv_diag_suppress 2388
template <unsigned IMM>
__host__ __device__ __forceinline__ constexpr uint32_t bs_lop3(uint32_t a, uint32_t b, uint32_t c) {
#ifdef __CUDA_ARCH__
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(IMM));
    return d;
#else
    uint32_t r = 0;
    for (int i = 0; i < 8; i++)
        if (IMM >> i & 1) r |= (i & 4 ? a : ~a) & (i & 2 ? b : ~b) & (i & 1 ? c : ~c);
    return r;
#endif
}
#pragma nv_diag_default 2388

#include "aes_bs_sbox.inc"

// Bitsliced round keys: k[round][r * 8 + b], rounds 0..NR (encryption: ek;
// decryption: the equivalent-inverse dk in application order), and the
// power-of-two multipliers that move the packing shifts and the ShiftRows
// rotations onto the FMA pipe (IMAD / IMAD.HI / IMAD.WIDE): passed at run time
// so ptxas cannot strength-reduce them back to ALU shifts (the ALU pipe is
// what the bitsliced warps compete for).
struct BSK {
    uint32_t k[15][32];
    uint32_t shl[5];     // shl[s] = 2^s           (s = 1, 2, 4): x << s = x * shl[s]
    uint32_t shr[5];     // shr[s] = 2^(32 - s):  x >> s = hi(x * shr[s])
    uint32_t rot[4];     // rot[r] = 2^(32 - 8r): rotr(x, 8r) = lo(x * rot[r]) + hi(x * rot[r])
    uint32_t one;        // 1: the final add of a rotation stays an IMAD
};

__host__ __device__ constexpr uint32_t bs_mulhi(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
    return __umulhi(a, b);
#else
    return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}


__host__ __device__ constexpr uint32_t bs_perm(uint32_t a, uint32_t b, uint32_t s) {
#ifdef __CUDA_ARCH__
    return __byte_perm(a, b, s);
#else
    const uint64_t v = ((uint64_t)b << 32) | a;
    uint32_t r = 0;
    for (int i = 0; i < 4; i++) r |= (uint32_t)((v >> (8 * ((s >> (4 * i)) & 7))) & 0xFF) << (8 * i);
    return r;
#endif
}

// swap bit (p + s) of a with bit p of b for every p with (p & s) == 0 in its
// byte; the two shifts are IMAD.HI / IMAD (FMA pipe), the rest 3 LOP3
__host__ __device__ constexpr void bs_swapmove(uint32_t& a, uint32_t& b, uint32_t m, int s, const BSK& bk) {
    const uint32_t t = (bs_mulhi(a, bk.shr[s]) ^ b) & m;
    b ^= t;
    a ^= t * bk.shl[s];
}

// 8x8 bit transpose inside each byte lane: bit b of byte r of w[j] <-> bit j of byte r of w[b]
__host__ __device__ constexpr void bs_transpose8(uint32_t (&w)[8], const BSK& bk) {
    bs_swapmove(w[0], w[1], 0x55555555u, 1, bk);
    bs_swapmove(w[2], w[3], 0x55555555u, 1, bk);
    bs_swapmove(w[4], w[5], 0x55555555u, 1, bk);
    bs_swapmove(w[6], w[7], 0x55555555u, 1, bk);
    bs_swapmove(w[0], w[2], 0x33333333u, 2, bk);
    bs_swapmove(w[1], w[3], 0x33333333u, 2, bk);
    bs_swapmove(w[4], w[6], 0x33333333u, 2, bk);
    bs_swapmove(w[5], w[7], 0x33333333u, 2, bk);
    bs_swapmove(w[0], w[4], 0x0F0F0F0Fu, 4, bk);
    bs_swapmove(w[1], w[5], 0x0F0F0F0Fu, 4, bk);
    bs_swapmove(w[2], w[6], 0x0F0F0F0Fu, 4, bk);
    bs_swapmove(w[3], w[7], 0x0F0F0F0Fu, 4, bk);
}

// 4x4 byte transpose: byte c of y[r] = byte r of x[c]
__host__ __device__ constexpr void bs_transpose4(uint32_t& x0, uint32_t& x1, uint32_t& x2, uint32_t& x3) {
    const uint32_t p0 = bs_perm(x0, x1, 0x5140), p1 = bs_perm(x0, x1, 0x7362);
    const uint32_t p2 = bs_perm(x2, x3, 0x5140), p3 = bs_perm(x2, x3, 0x7362);
    x0 = bs_perm(p0, p2, 0x5410);
    x1 = bs_perm(p0, p2, 0x7632);
    x2 = bs_perm(p1, p3, 0x5410);
    x3 = bs_perm(p1, p3, 0x7632);
}

// v[j][c] = column word c of block j  ->  R[r][b]
__host__ __device__ constexpr void bs_pack(const uint32_t (&v)[8][4], uint32_t (&R)[4][8], const BSK& bk) {
    uint32_t X[4][8] = {};
    for (int c = 0; c < 4; c++) {
        uint32_t w[8] = {v[0][c], v[1][c], v[2][c], v[3][c], v[4][c], v[5][c], v[6][c], v[7][c]};
        bs_transpose8(w, bk);                              // w[b]: byte r, bit j = bit b of byte r of block j
        for (int b = 0; b < 8; b++) X[c][b] = w[b];
    }
    for (int b = 0; b < 8; b++) {
        bs_transpose4(X[0][b], X[1][b], X[2][b], X[3][b]);   // X[r][b]: byte c = byte r of old X[c][b]
        for (int r = 0; r < 4; r++) R[r][b] = X[r][b];
    }
}

__host__ __device__ constexpr void bs_unpack(uint32_t (&R)[4][8], uint32_t (&v)[8][4], const BSK& bk) {
    for (int b = 0; b < 8; b++) bs_transpose4(R[0][b], R[1][b], R[2][b], R[3][b]);   // R[c][b] = old X[c][b]
    for (int c = 0; c < 4; c++) {
        uint32_t w[8] = {R[c][0], R[c][1], R[c][2], R[c][3], R[c][4], R[c][5], R[c][6], R[c][7]};
        bs_transpose8(w, bk);
        for (int j = 0; j < 8; j++) v[j][c] = w[j];
    }
}

template <class K>
__host__ __device__ constexpr void bs_ark(uint32_t (&R)[4][8], const K& k) {
    for (int r = 0; r < 4; r++)
        for (int b = 0; b < 8; b++) R[r][b] ^= k[r * 8 + b];
}

__host__ __device__ constexpr void bs_sub_bytes(uint32_t (&R)[4][8]) {
    for (int r = 0; r < 4; r++) bs_sbox(R[r]);
}

__host__ __device__ constexpr void bs_inv_sub_bytes(uint32_t (&R)[4][8]) {
    for (int r = 0; r < 4; r++) bs_inv_sbox(R[r]);
}

// rotr(x, 8r) on the FMA pipe: IMAD.WIDE.U32 (x * 2^(32-8r) = hi:lo) + IMAD (lo * 1 + hi)
__host__ __device__ constexpr uint32_t bs_rotr8(uint32_t x, int r, const BSK& bk) {
    const uint64_t p = (uint64_t)x * bk.rot[r];
    return (uint32_t)p * bk.one + (uint32_t)(p >> 32);
}

// ShiftRows (Eq 19): row r, column c <- column c + r  ==  rotate right by 8r
__host__ __device__ constexpr void bs_shift_rows(uint32_t (&R)[4][8], const BSK& bk) {
    for (int r = 1; r < 4; r++)
        for (int b = 0; b < 8; b++) R[r][b] = bs_rotr8(R[r][b], r, bk);
}

// InvShiftRows: rotate row r right by 32 - 8r
__host__ __device__ constexpr void bs_inv_shift_rows(uint32_t (&R)[4][8], const BSK& bk) {
    for (int r = 1; r < 4; r++)
        for (int b = 0; b < 8; b++) R[r][b] = bs_rotr8(R[r][b], 4 - r, bk);
}

// xtime on a bitsliced byte, bit b of the result
__host__ __device__ constexpr uint32_t bs_xt(const uint32_t (&t)[8], int b) {
    return b == 0 ? t[7] : (b == 1 || b == 3 || b == 4) ? t[b - 1] ^ t[7] : t[b - 1];
}

// MixColumns (matrix A) fused with AddRoundKey:
//   out_r = 02 a_r ^ 03 a_{r+1} ^ a_{r+2} ^ a_{r+3} ^ k_r
//         = xtime(a_r ^ a_{r+1}) ^ a_{r+1} ^ (a_{r+2} ^ a_{r+3}) ^ k_r
template <class K>
__host__ __device__ constexpr void bs_mix_columns_ark(uint32_t (&R)[4][8], const K& k) {
    uint32_t t[4][8] = {};
    for (int r = 0; r < 4; r++)
        for (int b = 0; b < 8; b++) t[r][b] = R[r][b] ^ R[(r + 1) & 3][b];
    uint32_t o[4][8] = {};
    for (int r = 0; r < 4; r++)
        for (int b = 0; b < 8; b++) o[r][b] = bs_xt(t[r], b) ^ R[(r + 1) & 3][b] ^ t[(r + 2) & 3][b] ^ k[r * 8 + b];
    for (int r = 0; r < 4; r++)
        for (int b = 0; b < 8; b++) R[r][b] = o[r][b];
}

// InvMixColumns = MixColumns o P, P: a_0,a_2 ^= 04 (a_0 ^ a_2); a_1,a_3 ^= 04 (a_1 ^ a_3)
// (circulants: (02 03 01 01)(05 00 04 00) = (0E 0B 0D 09)).
template <class K>
__host__ __device__ constexpr void bs_inv_mix_columns_ark(uint32_t (&R)[4][8], const K& k) {
    for (int h = 0; h < 2; h++) {
        uint32_t d[8] = {};
        for (int b = 0; b < 8; b++) d[b] = R[h][b] ^ R[h + 2][b];
        const uint32_t z[8] = {d[6], d[7] ^ d[6], d[0] ^ d[7], d[1] ^ d[6], d[2] ^ d[7] ^ d[6], d[3] ^ d[7], d[4], d[5]};
        for (int b = 0; b < 8; b++) {
            R[h][b] ^= z[b];
            R[h + 2][b] ^= z[b];
        }
    }
    bs_mix_columns_ark(R, k);
}

// Round keys (host): round i of `w` (4(NR+1) LE column words) -> bk.k[i]
__host__ __device__ constexpr void bs_expand_round_keys(const uint32_t* w, int nr, BSK& bk) {
    for (int q = 0; q < 5; q++) {
        bk.shl[q] = 1u << q;
        bk.shr[q] = q ? 1u << (32 - q) : 0u;
    }
    for (int r = 0; r < 4; r++) bk.rot[r] = r ? 1u << (32 - 8 * r) : 1u;
    bk.one = 1;
    for (int i = 0; i <= nr; i++)
        for (int r = 0; r < 4; r++)
            for (int b = 0; b < 8; b++) {
                uint32_t m = 0;
                for (int c = 0; c < 4; c++)
                    if ((w[4 * i + c] >> (8 * r + b)) & 1) m |= 0xFFu << (8 * c);
                bk.k[i][r * 8 + b] = m;
            }
}

struct BSKeyAt {
    const BSK& bk;
    int i;
    __host__ __device__ constexpr uint32_t operator[](int q) const { return bk.k[i][q]; }
};

// FIPS-197 Cipher on 8 blocks (Algorithm 1, corrected: DESIGN.md R1)
template <int NR>
__host__ __device__ constexpr void bs_encrypt(uint32_t (&R)[4][8], const BSK& bk) {
    bs_ark(R, BSKeyAt{bk, 0});
#ifdef __CUDA_ARCH__
#pragma unroll 1
#endif
    for (int i = 1; i < NR; i++) {
        bs_sub_bytes(R);
        bs_shift_rows(R, bk);
        bs_mix_columns_ark(R, BSKeyAt{bk, i});
    }
    bs_sub_bytes(R);
    bs_shift_rows(R, bk);
    bs_ark(R, BSKeyAt{bk, NR});
}

// FIPS-197 5.3.5 equivalent inverse cipher (R12), keys = dk in application order
template <int NR>
__host__ __device__ constexpr void bs_decrypt(uint32_t (&R)[4][8], const BSK& bk) {
    bs_ark(R, BSKeyAt{bk, 0});
#ifdef __CUDA_ARCH__
#pragma unroll 1
#endif
    for (int i = 1; i < NR; i++) {
        bs_inv_sub_bytes(R);
        bs_inv_shift_rows(R, bk);
        bs_inv_mix_columns_ark(R, BSKeyAt{bk, i});
    }
    bs_inv_sub_bytes(R);
    bs_inv_shift_rows(R, bk);
    bs_ark(R, BSKeyAt{bk, NR});
}

// ---------------------------------------------------------------------------
// Compile-time checks: both circuits on all 256 inputs against the product's
// tables, and the whole bitsliced cipher on FIPS-197 App. C.1 / C.3.
// ---------------------------------------------------------------------------
namespace bs_check {

constexpr bool sboxes_ok() {
    for (int x = 0; x < 256; x++) {
        uint32_t a[8] = {}, b[8] = {};
        for (int i = 0; i < 8; i++) a[i] = b[i] = (uint32_t)((x >> i) & 1);
        bs_sbox(a);
        bs_inv_sbox(b);
        int s = 0, si = 0;
        for (int i = 0; i < 8; i++) {
            s |= (int)(a[i] & 1) << i;
            si |= (int)(b[i] & 1) << i;
        }
        if (s != kTables.s[x] || si != kTables.si[x]) return false;
    }
    return true;
}
#ifndef __CUDA_ARCH__   // evaluated by the host pass (the device pass has no constexpr PRMT/SHF)
static_assert(sboxes_ok(), "bitsliced S-box / inverse S-box circuits == S / Si on all 256 inputs");
#endif

struct Sched {
    uint32_t ek[60], dk[60];
};
constexpr uint32_t sub_word(uint32_t w) {
    return (uint32_t)kTables.s[w & 0xFF] | ((uint32_t)kTables.s[(w >> 8) & 0xFF] << 8) |
           ((uint32_t)kTables.s[(w >> 16) & 0xFF] << 16) | ((uint32_t)kTables.s[w >> 24] << 24);
}
constexpr uint32_t inv_mix(uint32_t w) {
    uint32_t r = 0;
    for (int row = 0; row < 4; row++) {
        const uint8_t a0 = (uint8_t)(w >> (8 * row)), a1 = (uint8_t)(w >> (8 * ((row + 1) & 3))),
                      a2 = (uint8_t)(w >> (8 * ((row + 2) & 3))), a3 = (uint8_t)(w >> (8 * ((row + 3) & 3)));
        r |= (uint32_t)(gmul(a0, 14) ^ gmul(a1, 11) ^ gmul(a2, 13) ^ gmul(a3, 9)) << (8 * row);
    }
    return r;
}
// FIPS-197 5.2 / 5.3.5 (the same rule aes_expand_key implements at run time)
constexpr Sched expand(int nk) {
    Sched s{};
    const int nr = nk + 6, nw = 4 * (nr + 1);
    for (int i = 0; i < nk; i++)   // App. C key 00 01 02 ... as LE words
        s.ek[i] = (uint32_t)(4 * i) | (uint32_t)(4 * i + 1) << 8 | (uint32_t)(4 * i + 2) << 16 | (uint32_t)(4 * i + 3) << 24;
    uint8_t rcon = 1;
    for (int i = nk; i < nw; i++) {
        uint32_t t = s.ek[i - 1];
        if (i % nk == 0) {
            t = sub_word((t >> 8) | (t << 24)) ^ rcon;
            rcon = xt(rcon);
        } else if (nk == 8 && i % nk == 4) {
            t = sub_word(t);
        }
        s.ek[i] = s.ek[i - nk] ^ t;
    }
    for (int j = 0; j < 4; j++) {
        s.dk[j] = s.ek[4 * nr + j];
        s.dk[4 * nr + j] = s.ek[j];
    }
    for (int r = 1; r < nr; r++)
        for (int j = 0; j < 4; j++) s.dk[4 * r + j] = inv_mix(s.ek[4 * (nr - r) + j]);
    return s;
}
// one App. C plaintext (00112233...ff) in block slot `slot`, random-ish blocks elsewhere;
// returns column word c of the result in slot `slot`
template <int NR>
constexpr uint32_t run(bool dec, const uint32_t (&in)[4], int slot, int c) {
    const Sched s = expand(NR - 6);
    BSK bk{};
    bs_expand_round_keys(dec ? s.dk : s.ek, NR, bk);
    uint32_t v[8][4] = {};
    for (int j = 0; j < 8; j++)
        for (int q = 0; q < 4; q++) v[j][q] = j == slot ? in[q] : 0x9E3779B9u * (uint32_t)(4 * j + q + 1);
    uint32_t R[4][8] = {};
    bs_pack(v, R, bk);
    if (dec) bs_decrypt<NR>(R, bk);
    else bs_encrypt<NR>(R, bk);
    bs_unpack(R, v, bk);
    return v[slot][c];
}
constexpr uint32_t kPt[4] = {0x33221100u, 0x77665544u, 0xBBAA9988u, 0xFFEEDDCCu};
constexpr uint32_t kCt128[4] = {0xD8E0C469u, 0x30047B6Au, 0x80B7CDD8u, 0x5AC5B470u};   // 69c4e0d8 6a7b0430 d8cdb780 70b4c55a
constexpr uint32_t kCt256[4] = {0xCAB7A28Eu, 0xBF456751u, 0x9049FCEAu, 0x8960494Bu};   // 8ea2b7ca 516745bf eafc4990 4b496089
#ifndef __CUDA_ARCH__
static_assert(run<10>(false, kPt, 3, 0) == kCt128[0] && run<10>(false, kPt, 3, 3) == kCt128[3], "FIPS-197 C.1 encrypt");
static_assert(run<10>(true, kCt128, 6, 1) == kPt[1] && run<10>(true, kCt128, 6, 2) == kPt[2], "FIPS-197 C.1 decrypt");
static_assert(run<14>(false, kPt, 0, 2) == kCt256[2], "FIPS-197 C.3 encrypt");
static_assert(run<14>(true, kCt256, 7, 0) == kPt[0], "FIPS-197 C.3 decrypt");
#endif

}  // namespace bs_check

}  // namespace aesb200
