/*
 * aes_oracle.c -- plain, slow, byte-oriented CPU AES (TEST INFRASTRUCTURE ONLY).
 *
 * This file is the parity oracle for the B200 ECB path.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  The product library (paper_1902_05234_b200/) never includes,
 * links or calls anything in oracle/, and this file includes nothing from the
 * product: no shared tables, headers, generators or helpers.
 *
 * What it computes: ECB, C_i = Cipher(P_i) for every 16-byte block
 * (Eq 1), with Cipher written out exactly as the paper's
 * transforms define it -- SubBytes (Def 4), ShiftRows
 * (Def 5, Eq 19), MixColumns (Def 6, Eq 20,
 * PAPER.md:302-318), AddRoundKey (Def 7, Eq 21) -- in the
 * round order of Algorithm 1 as corrected by DESIGN.md
 * reading R1 (FIPS-197 sec 5.1: the last round has no MixColumns).  There are
 * NO T-tables here: the GPU's Eqs 22-26 are checked against this definition.
 *
 * Decryption is the straightforward InvCipher of FIPS-197 sec 5.3 (reading R12),
 * deliberately NOT the equivalent inverse cipher the GPU uses.
 *
 * Every function cites the passage it follows.  Readings of silent or garbled
 * passages are numbered R1..R23 in DESIGN.md ("Readings of the paper").
 *
 * Parity pins: tests/test_oracle_pins.py (GF worked examples of PAPER.md
 * Eqs 7-17, exhaustive field checks, S-box closed-form values, FIPS-197
 * App A/B/C, SP 800-38A F.1 (ECB), F.5 (CTR), F.2 (CBC), OpenSSL cross-checks,
 * the InvCipher trace against the forward trace).  No function here is
 * "parity unpinned".
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#include <pthread.h>

/* ------------------------------------------------------------------------- */
/* GF(2^8)                                                  */
/* ------------------------------------------------------------------------- */

/* Definition 1 / Eq 7: addition adds coefficients mod 2. */
uint8_t oracle_gf_add(uint8_t a, uint8_t b) { return (uint8_t)(a ^ b); }

/* Definition 3 / Eqs 15-17: xtime(a) = x*a mod m(x):
 * shift left, and if x^8 appeared subtract (= xor) m(x) = x^8+x^4+x^3+x+1
 * (Eq 8), i.e. xor 0x1B into the low byte.  Bit k = coefficient of x^k (R16). */
uint8_t oracle_xtime(uint8_t a) {
    uint8_t r = (uint8_t)(a << 1);
    if (a & 0x80) r ^= 0x1B;
    return r;
}

/* Definition 2 / Eqs 8-14: product mod m(x), written as
 * the sum over the set bits b_k of b of x^k * a ("all elements of AES can be
 * written as a sum of powers of x ... repeated use of ... M"). */
uint8_t oracle_gf_mul(uint8_t a, uint8_t b) {
    uint8_t acc = 0;
    uint8_t xk_a = a;           /* x^k * a, starting at k = 0 */
    for (int k = 0; k < 8; k++) {
        if (b & (1u << k)) acc = oracle_gf_add(acc, xk_a);
        xk_a = oracle_xtime(xk_a);
    }
    return acc;
}

/* Multiplicative inverse by its definition: the b with a*b = 1; inv(0) = 0
 * (FIPS-197 sec 5.1.1; the paper only says "a 256-byte look-up table",
 * reading R5). */
uint8_t oracle_gf_inv(uint8_t a) {
    if (a == 0) return 0;
    for (int b = 1; b < 256; b++)
        if (oracle_gf_mul(a, (uint8_t)b) == 1) return (uint8_t)b;
    return 0; /* unreachable for a field */
}

/* ------------------------------------------------------------------------- */
/* S-box, Definition 4, construction per FIPS-197 5.1.1   */
/* ------------------------------------------------------------------------- */

/* Affine map over GF(2): b'_i = b_i ^ b_{i+4} ^ b_{i+5} ^ b_{i+6} ^ b_{i+7} ^ c_i,
 * indices mod 8, c = 0x63 (reading R5). */
static uint8_t affine(uint8_t b) {
    uint8_t out = 0;
    for (int i = 0; i < 8; i++) {
        int bit = ((b >> i) & 1) ^ ((b >> ((i + 4) % 8)) & 1) ^ ((b >> ((i + 5) % 8)) & 1)
                ^ ((b >> ((i + 6) % 8)) & 1) ^ ((b >> ((i + 7) % 8)) & 1) ^ ((0x63 >> i) & 1);
        out |= (uint8_t)(bit << i);
    }
    return out;
}

uint8_t oracle_sbox(uint8_t a) { return affine(oracle_gf_inv(a)); }

/* Inverse S-box: the inverse permutation of oracle_sbox, found by search. */
uint8_t oracle_inv_sbox(uint8_t y) {
    for (int a = 0; a < 256; a++)
        if (oracle_sbox((uint8_t)a) == y) return (uint8_t)a;
    return 0; /* unreachable: sbox is a bijection (pinned) */
}

/* The oracle evaluates S and Si through the definitions above once, into
 * plain 256-entry arrays (the paper's own "256-byte look-up table named
 * sbox").  This is memoisation of the definition, not a T-table. */
static uint8_t S[256], SI[256];
static pthread_once_t sbox_once = PTHREAD_ONCE_INIT;
static void sbox_init(void) {
    for (int a = 0; a < 256; a++) S[a] = oracle_sbox((uint8_t)a);
    for (int a = 0; a < 256; a++) SI[S[a]] = (uint8_t)a;
}
static void ensure_sbox(void) { pthread_once(&sbox_once, sbox_init); }

/* ------------------------------------------------------------------------- */
/* State, round transforms (Defs 4-7)                                         */
/* ------------------------------------------------------------------------- */

/* state[r][c] <- in[r + 4c]: column-major bytes (reading R9). */
typedef struct { uint8_t s[4][4]; } state_t;

static void load_state(state_t *st, const uint8_t in[16]) {
    for (int c = 0; c < 4; c++)
        for (int r = 0; r < 4; r++) st->s[r][c] = in[r + 4 * c];
}
static void store_state(uint8_t out[16], const state_t *st) {
    for (int c = 0; c < 4; c++)
        for (int r = 0; r < 4; r++) out[r + 4 * c] = st->s[r][c];
}

/* Eq 18: state_{i,j} = sbox_t, t = state_{i,j}. */
static void sub_bytes(state_t *st) {
    for (int r = 0; r < 4; r++)
        for (int c = 0; c < 4; c++) st->s[r][c] = S[st->s[r][c]];
}
static void inv_sub_bytes(state_t *st) {
    for (int r = 0; r < 4; r++)
        for (int c = 0; c < 4; c++) st->s[r][c] = SI[st->s[r][c]];
}

/* Eq 19: state'_{i,j} = state_{i,t}, t = (i + j) mod 4. */
static void shift_rows(state_t *st) {
    state_t t = *st;
    for (int i = 0; i < 4; i++)
        for (int j = 0; j < 4; j++) st->s[i][j] = t.s[i][(i + j) % 4];
}
/* Inverse of Eq 19: state'_{i,(i+j) mod 4} = state_{i,j}. */
static void inv_shift_rows(state_t *st) {
    state_t t = *st;
    for (int i = 0; i < 4; i++)
        for (int j = 0; j < 4; j++) st->s[i][(i + j) % 4] = t.s[i][j];
}

/* Eq 20: state' = A (x) state, A the circulant (02 03 01 01) matrix printed at
 * PAPER.md:309-316, products in GF(2^8) (Def 2), sums are xor (Def 1). */
static const uint8_t A_MIX[4][4] = {
    {0x02, 0x03, 0x01, 0x01},
    {0x01, 0x02, 0x03, 0x01},
    {0x01, 0x01, 0x02, 0x03},
    {0x03, 0x01, 0x01, 0x02}};
/* FIPS-197 5.3.3 inverse matrix (0E 0B 0D 09), reading R12. */
static const uint8_t A_INVMIX[4][4] = {
    {0x0E, 0x0B, 0x0D, 0x09},
    {0x09, 0x0E, 0x0B, 0x0D},
    {0x0D, 0x09, 0x0E, 0x0B},
    {0x0B, 0x0D, 0x09, 0x0E}};

static void mat_columns(state_t *st, const uint8_t M[4][4]) {
    for (int c = 0; c < 4; c++) {
        uint8_t col[4];
        for (int r = 0; r < 4; r++) col[r] = st->s[r][c];
        for (int r = 0; r < 4; r++) {
            uint8_t acc = 0;
            for (int k = 0; k < 4; k++) acc = oracle_gf_add(acc, oracle_gf_mul(M[r][k], col[k]));
            st->s[r][c] = acc;
        }
    }
}
static void mix_columns(state_t *st) { mat_columns(st, A_MIX); }
static void inv_mix_columns(state_t *st) { mat_columns(st, A_INVMIX); }

/* Eq 21: state' = state xor epdkey.  Round key r is words w[4r..4r+3] of the
 * expanded key ("the first round key consists of the first Nb words",
 * PAPER.md:327); word 4r+c is column c, its byte k is row k. */
static void add_round_key(state_t *st, const uint8_t *w /* bytes of expanded key */, int r) {
    for (int c = 0; c < 4; c++)
        for (int k = 0; k < 4; k++) st->s[k][c] ^= w[16 * r + 4 * c + k];
}

/* ------------------------------------------------------------------------- */
/* Key schedule (PAPER.md:327 + FIPS-197 sec 5.2; readings R2, R3, R4)         */
/* ------------------------------------------------------------------------- */

/* Returns Nr for keybits in {128,192,256}, else 0. */
int oracle_nr(int keybits) {
    switch (keybits) { case 128: return 10; case 192: return 12; case 256: return 14; }
    return 0;
}

/* w_out receives 16*(Nr+1) bytes: word i = w_out[4i..4i+3] (byte 0 first). */
int oracle_key_expansion(const uint8_t *key, int keybits, uint8_t *w_out) {
    ensure_sbox();
    int nr = oracle_nr(keybits);
    if (!nr) return -1;
    int nk = keybits / 32;
    int nwords = 4 * (nr + 1);
    uint8_t (*w)[4] = (uint8_t (*)[4])w_out;
    for (int i = 0; i < nk; i++)
        for (int k = 0; k < 4; k++) w[i][k] = key[4 * i + k];
    uint8_t rcon = 0x01;                         /* Rcon[1] = x^0 */
    for (int i = nk; i < nwords; i++) {
        uint8_t temp[4];
        for (int k = 0; k < 4; k++) temp[k] = w[i - 1][k];
        if (i % nk == 0) {
            uint8_t t0 = temp[0];                /* RotWord */
            temp[0] = temp[1]; temp[1] = temp[2]; temp[2] = temp[3]; temp[3] = t0;
            for (int k = 0; k < 4; k++) temp[k] = S[temp[k]];   /* SubWord */
            temp[0] ^= rcon;                     /* Rcon[i/Nk] = x^(i/Nk - 1) in byte 0 */
            rcon = oracle_xtime(rcon);
        } else if (nk == 8 && i % nk == 4) {
            for (int k = 0; k < 4; k++) temp[k] = S[temp[k]];
        }
        for (int k = 0; k < 4; k++) w[i][k] = (uint8_t)(w[i - nk][k] ^ temp[k]);   /* w[i-Nk], R3 */
    }
    return nr;
}

/* ------------------------------------------------------------------------- */
/* Cipher / InvCipher (Algorithm 1 corrected, R1; InvCipher R12)              */
/* ------------------------------------------------------------------------- */

/* trace (optional, 16*(nr+1) bytes): state after AddRoundKey(r), r = 0..Nr,
 * i.e. FIPS-197 App B's "start of round r+1" column; trace[Nr] = output. */
static void cipher_block(const uint8_t in[16], uint8_t out[16], const uint8_t *w, int nr,
                         uint8_t *trace) {
    state_t st;
    load_state(&st, in);
    add_round_key(&st, w, 0);
    if (trace) store_state(trace, &st);
    for (int r = 1; r <= nr - 1; r++) {
        sub_bytes(&st);
        shift_rows(&st);
        mix_columns(&st);
        add_round_key(&st, w, r);
        if (trace) store_state(trace + 16 * r, &st);
    }
    sub_bytes(&st);
    shift_rows(&st);
    add_round_key(&st, w, nr);
    if (trace) store_state(trace + 16 * nr, &st);
    store_state(out, &st);
}

/* trace (optional, 16*(nr+1) bytes): trace[0] = state after AddRoundKey(Nr);
 * trace[i], 1 <= i <= Nr-1 = state after the loop iteration for round Nr-i
 * (after InvMixColumns); trace[Nr] = output. */
static void inv_cipher_block_t(const uint8_t in[16], uint8_t out[16], const uint8_t *w, int nr,
                               uint8_t *trace) {
    state_t st;
    load_state(&st, in);
    add_round_key(&st, w, nr);
    if (trace) store_state(trace, &st);
    for (int r = nr - 1; r >= 1; r--) {
        inv_shift_rows(&st);
        inv_sub_bytes(&st);
        add_round_key(&st, w, r);
        inv_mix_columns(&st);
        if (trace) store_state(trace + 16 * (nr - r), &st);
    }
    inv_shift_rows(&st);
    inv_sub_bytes(&st);
    add_round_key(&st, w, 0);
    if (trace) store_state(trace + 16 * nr, &st);
    store_state(out, &st);
}

static void inv_cipher_block(const uint8_t in[16], uint8_t out[16], const uint8_t *w, int nr) {
    inv_cipher_block_t(in, out, w, nr, NULL);
}

/* ------------------------------------------------------------------------- */
/* ECB over a buffer (Eq 1), threaded over contiguous slices                  */
/* ------------------------------------------------------------------------- */

typedef struct {
    const uint8_t *in; uint8_t *out; const uint8_t *w; int nr; int decrypt;
    uint64_t b0, b1;
} job_t;

static void *ecb_worker(void *arg) {
    job_t *j = (job_t *)arg;
    for (uint64_t b = j->b0; b < j->b1; b++) {
        if (j->decrypt) inv_cipher_block(j->in + 16 * b, j->out + 16 * b, j->w, j->nr);
        else cipher_block(j->in + 16 * b, j->out + 16 * b, j->w, j->nr, NULL);
    }
    return NULL;
}

/* oracle_aes_ecb: decrypt = 0 encrypts, 1 decrypts.  in == out is allowed
 * (each block is read fully before it is written).  Returns 0 or -1. */
int oracle_aes_ecb(const uint8_t *key, int keybits, int decrypt, const uint8_t *in, uint8_t *out,
                   uint64_t nblocks, int nthreads) {
    uint8_t w[16 * 15];
    int nr = oracle_key_expansion(key, keybits, w);
    if (nr <= 0) return -1;
    if (nblocks == 0) return 0;
    if (nthreads < 1) nthreads = 1;
    if ((uint64_t)nthreads > nblocks) nthreads = (int)nblocks;
    if (nthreads > 1024) nthreads = 1024;
    pthread_t tid[1024];
    job_t jobs[1024];
    for (int t = 0; t < nthreads; t++) {
        jobs[t].in = in; jobs[t].out = out; jobs[t].w = w; jobs[t].nr = nr; jobs[t].decrypt = decrypt;
        jobs[t].b0 = nblocks * (uint64_t)t / (uint64_t)nthreads;
        jobs[t].b1 = nblocks * (uint64_t)(t + 1) / (uint64_t)nthreads;
    }
    if (nthreads == 1) { ecb_worker(&jobs[0]); return 0; }
    int started = 0;
    for (int t = 0; t < nthreads; t++) {
        if (pthread_create(&tid[t], NULL, ecb_worker, &jobs[t]) != 0) { ecb_worker(&jobs[t]); tid[t] = 0; }
        else started++;
    }
    for (int t = 0; t < nthreads; t++) if (tid[t]) pthread_join(tid[t], NULL);
    (void)started;
    return 0;
}

/* Per-round trace of one block (for the FIPS-197 App B pins). */
int oracle_cipher_trace(const uint8_t *key, int keybits, const uint8_t in[16], uint8_t *trace) {
    uint8_t w[16 * 15], out[16];
    int nr = oracle_key_expansion(key, keybits, w);
    if (nr <= 0) return -1;
    cipher_block(in, out, w, nr, trace);
    return nr;
}

/* Per-iteration trace of one block through InvCipher (see inv_cipher_block_t). */
int oracle_inv_cipher_trace(const uint8_t *key, int keybits, const uint8_t in[16], uint8_t *trace) {
    uint8_t w[16 * 15], out[16];
    int nr = oracle_key_expansion(key, keybits, w);
    if (nr <= 0) return -1;
    inv_cipher_block_t(in, out, w, nr, trace);
    return nr;
}

/* ------------------------------------------------------------------------- */
/* Single-transform entry points, for the pins only                           */
/* ------------------------------------------------------------------------- */

void oracle_sbox_table(uint8_t out[256]) { ensure_sbox(); memcpy(out, S, 256); }
void oracle_inv_sbox_table(uint8_t out[256]) { ensure_sbox(); memcpy(out, SI, 256); }

/* op: 0 SubBytes, 1 ShiftRows, 2 MixColumns, 3 InvSubBytes, 4 InvShiftRows,
 *     5 InvMixColumns.  Operates on 16 bytes in block order (R9). */
int oracle_transform(int op, uint8_t blk[16]) {
    ensure_sbox();
    state_t st;
    load_state(&st, blk);
    switch (op) {
        case 0: sub_bytes(&st); break;
        case 1: shift_rows(&st); break;
        case 2: mix_columns(&st); break;
        case 3: inv_sub_bytes(&st); break;
        case 4: inv_shift_rows(&st); break;
        case 5: inv_mix_columns(&st); break;
        default: return -1;
    }
    store_state(blk, &st);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* CTR and CBC (NEXT-1 / NEXT-4 of SURVEY.md 8(f))                            */
/* ------------------------------------------------------------------------- */

/* CTR, Eq 5: C_i = P_i xor CTR(R+i).  Reading R24: CTR(.)
 * is Cipher_K of the counter block, the counter is the whole 16-byte block read
 * as a big-endian 128-bit integer and incremented by one per block mod 2^128
 * (SP 800-38A 6.5, B.1).  Block j (0-based, j >= 0) of this call uses counter
 * iv + block_offset + j.  Encryption and decryption are the same operation. */
static void counter_add(uint8_t ctr[16], uint64_t add) {
    /* big-endian 128-bit add, carry propagated byte by byte */
    unsigned carry = 0;
    for (int b = 15; b >= 0; b--) {
        unsigned v = ctr[b] + (unsigned)(add & 0xFF) + carry;
        ctr[b] = (uint8_t)v;
        carry = v >> 8;
        add >>= 8;
    }
}

typedef struct {
    const uint8_t *in; uint8_t *out; const uint8_t *w; int nr;
    uint8_t iv[16]; uint64_t off; uint64_t b0, b1;
} ctr_job_t;

static void *ctr_worker(void *arg) {
    ctr_job_t *j = (ctr_job_t *)arg;
    for (uint64_t b = j->b0; b < j->b1; b++) {
        uint8_t ctr[16], ks[16];
        memcpy(ctr, j->iv, 16);
        counter_add(ctr, j->off);
        counter_add(ctr, b);
        cipher_block(ctr, ks, j->w, j->nr, NULL);
        for (int k = 0; k < 16; k++) j->out[16 * b + k] = (uint8_t)(j->in[16 * b + k] ^ ks[k]);
    }
    return NULL;
}

int oracle_aes_ctr(const uint8_t *key, int keybits, const uint8_t iv[16], uint64_t block_offset,
                   const uint8_t *in, uint8_t *out, uint64_t nblocks, int nthreads) {
    uint8_t w[16 * 15];
    int nr = oracle_key_expansion(key, keybits, w);
    if (nr <= 0) return -1;
    if (nblocks == 0) return 0;
    if (nthreads < 1) nthreads = 1;
    if ((uint64_t)nthreads > nblocks) nthreads = (int)nblocks;
    if (nthreads > 1024) nthreads = 1024;
    pthread_t tid[1024];
    ctr_job_t jobs[1024];
    for (int t = 0; t < nthreads; t++) {
        jobs[t].in = in; jobs[t].out = out; jobs[t].w = w; jobs[t].nr = nr;
        memcpy(jobs[t].iv, iv, 16); jobs[t].off = block_offset;
        jobs[t].b0 = nblocks * (uint64_t)t / (uint64_t)nthreads;
        jobs[t].b1 = nblocks * (uint64_t)(t + 1) / (uint64_t)nthreads;
    }
    if (nthreads == 1) { ctr_worker(&jobs[0]); return 0; }
    for (int t = 0; t < nthreads; t++)
        if (pthread_create(&tid[t], NULL, ctr_worker, &jobs[t]) != 0) { ctr_worker(&jobs[t]); tid[t] = 0; }
    for (int t = 0; t < nthreads; t++) if (tid[t]) pthread_join(tid[t], NULL);
    return 0;
}

/* CBC, Eq 2, printed as C_i = P_i xor C_{i-1} without the
 * cipher call.  Reading R25: C_i = Cipher_K(P_i xor C_{i-1}), C_0 = IV
 * (SP 800-38A 6.2); decryption P_i = InvCipher_K(C_i) xor C_{i-1}.
 * Sequential, single-threaded, exactly as the equations read.  in == out is
 * allowed (each C_{i-1} is saved before block i is overwritten). */
int oracle_aes_cbc(const uint8_t *key, int keybits, const uint8_t iv[16], int decrypt,
                   const uint8_t *in, uint8_t *out, uint64_t nblocks) {
    uint8_t w[16 * 15];
    int nr = oracle_key_expansion(key, keybits, w);
    if (nr <= 0) return -1;
    uint8_t prev[16];
    memcpy(prev, iv, 16);
    for (uint64_t b = 0; b < nblocks; b++) {
        uint8_t x[16], y[16];
        memcpy(x, in + 16 * b, 16);
        if (!decrypt) {
            for (int k = 0; k < 16; k++) y[k] = (uint8_t)(x[k] ^ prev[k]);
            cipher_block(y, out + 16 * b, w, nr, NULL);
            memcpy(prev, out + 16 * b, 16);
        } else {
            inv_cipher_block(x, y, w, nr);
            for (int k = 0; k < 16; k++) out[16 * b + k] = (uint8_t)(y[k] ^ prev[k]);
            memcpy(prev, x, 16);
        }
    }
    return 0;
}
