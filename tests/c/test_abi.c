/* Plain-C user of the C ABI (include/aes_b200.h): proves the library is
 * usable without Python or torch.  Part 1 (always): aes_expand_key against
 * FIPS-197 App A.1 and the error codes decided before any CUDA call.
 * Part 2 (argv[1] == "gpu"): the FIPS-197 App C vectors encrypted and
 * decrypted on the device with cudaMalloc'd buffers and a user stream (the
 * T-table, hybrid and bitsliced kernels), a 128 MiB round trip on the default
 * (hybrid) kernel, plus CTR (SP 800-38A F.5.1 block 1), all through the ABI.
 * Exit 0 = pass. */
#include <stdio.h>
#include <string.h>
#include <cuda_runtime.h>
#include "aes_b200.h"

#define CHECK(c) do { if (!(c)) { printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); return 1; } } while (0)

static void hex2bin(const char *h, unsigned char *o, int n) {
    for (int i = 0; i < n; i++) { unsigned v; sscanf(h + 2 * i, "%2x", &v); o[i] = (unsigned char)v; }
}

int main(int argc, char **argv) {
    aes_round_keys rk;
    unsigned char key[32];
    hex2bin("2b7e151628aed2a6abf7158809cf4f3c", key, 16);
    CHECK(aes_expand_key(key, 128, &rk) == AES_OK);
    CHECK(rk.nr == 10 && rk.keybits == 128);
    CHECK(rk.ek[40] == 0xa8f914d0u);           /* FIPS-197 A.1 w40 = d014f9a8 (LE word) */
    CHECK(rk.ek[43] == 0xa60c63b6u);           /* w43 = b6630ca6 */
    CHECK(aes_expand_key(key, 100, &rk) == AES_EKEYBITS);
    CHECK(aes_expand_key(NULL, 128, &rk) == AES_ENULL);
    CHECK(aes_expand_key(key, 128, &rk) == AES_OK);
    CHECK(aes_ecb_encrypt(&rk, 12, (void *)16, (void *)16, 1, NULL) == AES_ENR);
    CHECK(aes_ecb_encrypt(&rk, 10, (void *)16, (void *)16, 0, NULL) == AES_OK);
    CHECK(aes_ecb_encrypt(&rk, 10, (void *)16, (void *)32, 4, NULL) == AES_EOVERLAP);
    CHECK(aes_ecb_encrypt(&rk, 10, (void *)24, (void *)4096, 4, NULL) == AES_EALIGN);
    CHECK(strncmp(aes_status_string(AES_EOVERLAP), "AES_EOVERLAP", 12) == 0);
    CHECK(aes_abi_version() == AES_B200_ABI_VERSION);
    if (argc < 2 || strcmp(argv[1], "gpu") != 0) { printf("c-abi cpu ok\n"); return 0; }

    const char *kat[3][2] = {
        {"000102030405060708090a0b0c0d0e0f", "69c4e0d86a7b0430d8cdb78070b4c55a"},
        {"000102030405060708090a0b0c0d0e0f1011121314151617", "dda97ca4864cdfe06eaf70a0ec0d7191"},
        {"000102030405060708090a0b0c0d0e0f101112131415161718191a1b1c1d1e1f", "8ea2b7ca516745bfeafc49904b496089"}};
    unsigned char pt[16], ct[16], want[16], back[16];
    hex2bin("00112233445566778899aabbccddeeff", pt, 16);
    void *d_in = NULL, *d_out = NULL;
    cudaStream_t st;
    CHECK(cudaMalloc(&d_in, 4096) == cudaSuccess && cudaMalloc(&d_out, 4096) == cudaSuccess);
    CHECK(cudaStreamCreate(&st) == cudaSuccess);
    for (int k = 0; k < 3; k++) {
        int kb = 128 + 64 * k;
        hex2bin(kat[k][0], key, kb / 8);
        hex2bin(kat[k][1], want, 16);
        CHECK(aes_expand_key(key, kb, &rk) == AES_OK);
        CHECK(cudaMemcpy(d_in, pt, 16, cudaMemcpyHostToDevice) == cudaSuccess);
        CHECK(aes_ecb_encrypt(&rk, rk.nr, d_in, d_out, 1, st) == AES_OK);
        CHECK(aes_ecb_decrypt(&rk, rk.nr, d_out, d_in, 1, st) == AES_OK);
        CHECK(cudaStreamSynchronize(st) == cudaSuccess);
        CHECK(cudaMemcpy(ct, d_out, 16, cudaMemcpyDeviceToHost) == cudaSuccess);
        CHECK(cudaMemcpy(back, d_in, 16, cudaMemcpyDeviceToHost) == cudaSuccess);
        CHECK(memcmp(ct, want, 16) == 0);
        CHECK(memcmp(back, pt, 16) == 0);
    }
    /* the same App C vectors through aes_ecb_launch with the hybrid and the
       bitsliced-only kernels (AES_VAR_HYBRID / AES_VAR_BITSLICE) */
    for (int v = AES_VAR_HYBRID; v <= AES_VAR_BITSLICE; v++) {
        aes_launch_config cfg = {v, 0, 0, 0};
        for (int k = 0; k < 3; k++) {
            int kb = 128 + 64 * k;
            hex2bin(kat[k][0], key, kb / 8);
            hex2bin(kat[k][1], want, 16);
            CHECK(aes_expand_key(key, kb, &rk) == AES_OK);
            CHECK(cudaMemcpy(d_in, pt, 16, cudaMemcpyHostToDevice) == cudaSuccess);
            CHECK(aes_ecb_launch(&rk, rk.nr, 0, d_in, d_out, 1, st, &cfg) == AES_OK);
            CHECK(aes_ecb_launch(&rk, rk.nr, 1, d_out, d_in, 1, st, &cfg) == AES_OK);
            CHECK(cudaStreamSynchronize(st) == cudaSuccess);
            CHECK(cudaMemcpy(ct, d_out, 16, cudaMemcpyDeviceToHost) == cudaSuccess);
            CHECK(cudaMemcpy(back, d_in, 16, cudaMemcpyDeviceToHost) == cudaSuccess);
            CHECK(memcmp(ct, want, 16) == 0);
            CHECK(memcmp(back, pt, 16) == 0);
        }
    }
    /* a message past the hybrid crossover (2^23 blocks, 128 MiB): the default
       entry points take the hybrid kernel; decrypt(encrypt(x)) == x, and block
       5 of an all-App-C-plaintext buffer encrypts to the App C ciphertext */
    {
        const unsigned long long nb = 1ull << 23;
        void *big = NULL, *big2 = NULL;
        CHECK(cudaMalloc(&big, nb * 16) == cudaSuccess && cudaMalloc(&big2, nb * 16) == cudaSuccess);
        for (unsigned long long j = 0; j < 64; j++)
            CHECK(cudaMemcpy((char *)big + 16 * j, pt, 16, cudaMemcpyHostToDevice) == cudaSuccess);
        CHECK(cudaMemset((char *)big + 1024, 0x5a, nb * 16 - 1024) == cudaSuccess);
        hex2bin(kat[0][0], key, 16);
        hex2bin(kat[0][1], want, 16);
        CHECK(aes_expand_key(key, 128, &rk) == AES_OK);
        CHECK(aes_ecb_encrypt(&rk, rk.nr, big, big2, nb, st) == AES_OK);
        CHECK(cudaMemcpyAsync(ct, (char *)big2 + 16 * 5, 16, cudaMemcpyDeviceToHost, st) == cudaSuccess);
        CHECK(aes_ecb_decrypt(&rk, rk.nr, big2, big2, nb, st) == AES_OK);   /* in place */
        CHECK(cudaStreamSynchronize(st) == cudaSuccess);
        CHECK(memcmp(ct, want, 16) == 0);
        static unsigned char h1[4096], h2[4096];
        for (unsigned long long off = 0; off < nb * 16; off += (nb * 16) / 7 - 16) {
            unsigned long long o = off & ~15ull;
            if (o + sizeof h1 > nb * 16) o = nb * 16 - sizeof h1;
            CHECK(cudaMemcpy(h1, (char *)big + o, sizeof h1, cudaMemcpyDeviceToHost) == cudaSuccess);
            CHECK(cudaMemcpy(h2, (char *)big2 + o, sizeof h2, cudaMemcpyDeviceToHost) == cudaSuccess);
            CHECK(memcmp(h1, h2, sizeof h1) == 0);
        }
        cudaFree(big); cudaFree(big2);
    }
    hex2bin("000102030405060708090a0b0c0d0e0f", key, 16);
    CHECK(aes_expand_key(key, 128, &rk) == AES_OK);
    /* host pointers are rejected: no CPU fallback */
    CHECK(aes_ecb_encrypt(&rk, rk.nr, pt, ct, 1, st) == AES_ENOTDEVICE);
    /* CTR, SP 800-38A F.5.1 block 1 */
    unsigned char iv[16], p1[16], c1[16], got[16];
    hex2bin("2b7e151628aed2a6abf7158809cf4f3c", key, 16);
    hex2bin("f0f1f2f3f4f5f6f7f8f9fafbfcfdfeff", iv, 16);
    hex2bin("6bc1bee22e409f96e93d7e117393172a", p1, 16);
    hex2bin("874d6191b620e3261bef6864990db6ce", c1, 16);
    CHECK(aes_expand_key(key, 128, &rk) == AES_OK);
    CHECK(cudaMemcpy(d_in, p1, 16, cudaMemcpyHostToDevice) == cudaSuccess);
    CHECK(aes_ctr_xcrypt(&rk, 10, iv, 0, d_in, d_out, 1, st) == AES_OK);
    CHECK(cudaStreamSynchronize(st) == cudaSuccess);
    CHECK(cudaMemcpy(got, d_out, 16, cudaMemcpyDeviceToHost) == cudaSuccess);
    CHECK(memcmp(got, c1, 16) == 0);
    cudaFree(d_in); cudaFree(d_out); cudaStreamDestroy(st);
    printf("c-abi gpu ok\n");
    return 0;
}
