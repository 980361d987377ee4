// aes_keysched.cpp -- host key schedule behind aes_expand_key (steps A1, A2).
//
// A1: KeyExpansion, PAPER.md:327 ("key expansion and round key selection",
//     Nr+1 round keys = 1408 bits for AES-128) + FIPS-197 5.2 for the rule the
//     paper leaves out (R2, R3: w[i] = w[i-Nk] ^ temp; R4: Nk = 4/6/8).
// A2: equivalent-inverse schedule for the Td-table decryption (FIPS-197 5.3.5,
//     DESIGN.md R12): dk[0] = ek[Nr], dk[r] = InvMixColumns(ek[Nr-r]),
//     dk[Nr] = ek[0].
// Words are little-endian memory-order (R7/R21): byte k of a word is
// row k of that column.
#include <cstring>

#include "aes_b200.h"
#include "aes_tables.h"

namespace {
using aesb200::kTables;

inline uint32_t sub_word(uint32_t w) {
    return (uint32_t)kTables.s[w & 0xFF] | ((uint32_t)kTables.s[(w >> 8) & 0xFF] << 8) |
           ((uint32_t)kTables.s[(w >> 16) & 0xFF] << 16) | ((uint32_t)kTables.s[w >> 24] << 24);
}

// RotWord [a0,a1,a2,a3] -> [a1,a2,a3,a0]: in LE words that is a right rotate by 8.
inline uint32_t rot_word(uint32_t w) { return (w >> 8) | (w << 24); }

// InvMixColumns on one LE column word.
inline uint32_t inv_mix_column(uint32_t w) {
    uint8_t a[4] = {(uint8_t)w, (uint8_t)(w >> 8), (uint8_t)(w >> 16), (uint8_t)(w >> 24)};
    static constexpr uint8_t M[4][4] = {
        {14, 11, 13, 9}, {9, 14, 11, 13}, {13, 9, 14, 11}, {11, 13, 9, 14}};
    uint32_t r = 0;
    for (int row = 0; row < 4; row++) {
        uint8_t acc = 0;
        for (int k = 0; k < 4; k++) acc ^= aesb200::gmul(M[row][k], a[k]);
        r |= (uint32_t)acc << (8 * row);
    }
    return r;
}
}  // namespace

extern "C" aes_status aes_expand_key(const uint8_t* key, int keybits, aes_round_keys* out) {
    if (!key || !out) return AES_ENULL;
    int nk, nr;
    switch (keybits) {
        case 128: nk = 4; nr = 10; break;
        case 192: nk = 6; nr = 12; break;
        case 256: nk = 8; nr = 14; break;
        default: return AES_EKEYBITS;
    }
    aes_round_keys rk;
    std::memset(&rk, 0, sizeof rk);
    const int nw = 4 * (nr + 1);
    for (int i = 0; i < nk; i++)
        rk.ek[i] = (uint32_t)key[4 * i] | ((uint32_t)key[4 * i + 1] << 8) |
                   ((uint32_t)key[4 * i + 2] << 16) | ((uint32_t)key[4 * i + 3] << 24);
    uint8_t rcon = 1;
    for (int i = nk; i < nw; i++) {
        uint32_t t = rk.ek[i - 1];
        if (i % nk == 0) {
            t = sub_word(rot_word(t)) ^ rcon;
            rcon = aesb200::xt(rcon);
        } else if (nk == 8 && i % nk == 4) {
            t = sub_word(t);
        }
        rk.ek[i] = rk.ek[i - nk] ^ t;
    }
    for (int j = 0; j < 4; j++) {
        rk.dk[j] = rk.ek[4 * nr + j];
        rk.dk[4 * nr + j] = rk.ek[j];
    }
    for (int r = 1; r < nr; r++)
        for (int j = 0; j < 4; j++) rk.dk[4 * r + j] = inv_mix_column(rk.ek[4 * (nr - r) + j]);
    rk.nr = nr;
    rk.keybits = keybits;
    *out = rk;
    return AES_OK;
}
