/*
 * aes_b200.h -- C ABI of the B200 (sm_100a) AES-ECB library  libaes_b200.so
 *
 * The hot path of arXiv 1902.05234 ("one state per thread", T-box rounds):
 * given a cipher key and a message P = P_1..P_n of 16-byte states, produce
 * C_i = Cipher_K(P_i) for every i (ECB, Eq 1), and the inverse.
 * Rounds are computed as the paper's T-table round (Eq 26, PAPER.md:423-427;
 * tables Eqs 22-25), one state per thread (sec 4.1,
 * PAPER.md:435-436).  Decryption uses the equivalent inverse cipher
 * (FIPS-197 5.3.5; reading R12), keys of 128/192/256 bits (R4).
 *
 * Conventions (R7, R9, R21):
 *  - A 16-byte block is a 4x4 state, byte r+4c = row r of column c.
 *  - Column c is the little-endian uint32 word c of the block.
 *  - Round-key words are little-endian memory-order words: for the key
 *    00 01 02 03 ..., ek[0] == 0x03020100.
 *
 * Thread safety: every entry point is re-entrant; the library keeps no
 * per-call global mutable state (a per-device launch-attribute cache is
 * initialised once under a lock).  No CUDA or torch types appear here: a
 * stream is passed as `void *` holding a cudaStream_t (NULL = legacy default).
 *
 * Errors: status codes only -- no exceptions cross the ABI, nothing aborts.
 * Argument validation happens before any launch.  On error `out` is left
 * unspecified (no partial-output guarantee: the GPU analogue of SPEC.md:491).
 * Kernel faults surface at the caller's next synchronisation.
 * There is NO CPU fallback: host pointers passed to the device entry points
 * are rejected with AES_ENOTDEVICE.
 */
#ifndef AES_B200_H
#define AES_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AES_B200_ABI_VERSION 3   /* 2: AES_VAR_GLOBAL, aes_launch_config.flags, AES_ECAPTURE; 3: AES_VAR_HYBRID, AES_VAR_BITSLICE (hybrid default from 2^23 blocks) */

typedef enum {
    AES_OK = 0,
    AES_EKEYBITS = 1,   /* keybits not in {128, 192, 256}                        */
    AES_ENR = 2,        /* nr not in {10,12,14}, or nr != rk->nr                  */
    AES_ENULL = 3,      /* a required pointer is NULL                             */
    AES_EALIGN = 4,     /* in/out not 16-byte aligned                             */
    AES_EOVERLAP = 5,   /* in and out partially overlap (in == out is allowed)    */
    AES_ERANGE = 6,     /* 16*nblocks overflows, or a config value out of range   */
    AES_ENOTDEVICE = 7, /* in/out not device memory of the current device         */
    AES_ECUDA = 8,      /* a CUDA runtime call failed; see aes_last_cuda_error()  */
    AES_EVARIANT = 9,   /* unknown kernel variant / states-per-thread             */
    AES_ECAPTURE = 10   /* aes_ecb_batch called on a stream under graph capture   */
} aes_status;

/* Expanded key.  Plain old data, caller-owned, 488 bytes.
 *  ek: FIPS-197 KeyExpansion ("1408 bits" for AES-128), 4*(nr+1)
 *      words used; round key r = ek[4r .. 4r+3] ("round keys are sequentially
 *      taken from the expanded key").
 *  dk: equivalent-inverse schedule in application order:
 *      dk[0..3] = ek[4nr..], dk[4r+j] = InvMixColumns(ek[4(nr-r)+j]) for
 *      1 <= r <= nr-1, dk[4nr..] = ek[0..3]  (FIPS-197 5.3.5; R12). */
typedef struct {
    uint32_t ek[60];
    uint32_t dk[60];
    int32_t nr;       /* 10 | 12 | 14 */
    int32_t keybits;  /* 128 | 192 | 256 */
} aes_round_keys;

/* aes_expand_key: host only, no CUDA calls.  key: keybits/8 bytes, read only
 * during the call.  out: caller-owned, fully written on AES_OK.
 * Errors: AES_ENULL, AES_EKEYBITS.  Steps A1 + A2 of SURVEY.md 8(a). */
aes_status aes_expand_key(const uint8_t *key, int keybits, aes_round_keys *out);

/* aes_ecb_encrypt / aes_ecb_decrypt: enqueue C_i = E_K(P_i) (resp. P_i =
 * D_K(C_i)) for i < nblocks on `stream`, asynchronously.
 *  rk      : host pointer, read during the call only (round keys are copied
 *            by value into the kernel parameters -> constant bank, PAPER.md
 *            sec 4.3 "round keys in the constant memory", 452-454).
 *  nr      : must equal rk->nr (guards against a stale/mismatched schedule).
 *  in, out : device pointers of the current device, 16-byte aligned,
 *            16*nblocks bytes each; in == out (in place) is allowed, any
 *            other overlap is AES_EOVERLAP.  Caller keeps them alive until the
 *            stream work completes.
 *  nblocks : number of 16-byte states (64-bit; > 2^32 supported).  0 -> AES_OK
 *            without a launch.
 *  stream  : cudaStream_t as void*, NULL = legacy default stream.
 * Errors: AES_ENULL, AES_ENR, AES_EALIGN, AES_EOVERLAP, AES_ERANGE,
 *         AES_ENOTDEVICE, AES_ECUDA.  Uses the tuned default kernel variant. */
aes_status aes_ecb_encrypt(const aes_round_keys *rk, int nr, const void *in, void *out,
                           uint64_t nblocks, void *stream);
aes_status aes_ecb_decrypt(const aes_round_keys *rk, int nr, const void *in, void *out,
                           uint64_t nblocks, void *stream);

/* aes_ctr_xcrypt: CTR mode (Eq 5,
 * C_i = P_i xor CTR(R+i), "Suitable" for parallelism in Table 1), reading R24:
 * the keystream block of block j (0-based) of this call is
 * Cipher_K(iv + block_offset + j), the counter being the whole 16-byte block as
 * a big-endian 128-bit integer, wrapping mod 2^128 (SP 800-38A 6.5 / B.1).
 * Encryption and decryption are the same call.  block_offset lets a shard
 * (rank r of a multi-GPU job) continue the global counter stream.
 *  iv : host pointer to 16 bytes (initial counter block T_1), read during the call.
 *  in/out/nblocks/stream : as aes_ecb_encrypt (in == out allowed).
 * Implementation: counter-mode caching -- the 256 counters of a group differ
 * only in byte 15, so rounds 1-2 take 5 lookups instead of 32 per block
 * (environment AES_B200_CTR_KERNEL=plain selects the uncached kernel, for A/B
 * measurements only; results are identical).
 * Errors: as aes_ecb_encrypt, plus AES_ENULL for iv. */
aes_status aes_ctr_xcrypt(const aes_round_keys *rk, int nr, const uint8_t *iv, uint64_t block_offset,
                          const void *in, void *out, uint64_t nblocks, void *stream);

/* aes_cbc_decrypt: CBC decryption (Eq 2,
 * printed without the cipher call -- reading R25: C_i = Cipher_K(P_i xor
 * C_{i-1}), C_0 = IV), P_i = InvCipher_K(C_i) xor C_{i-1}.  Decryption is
 * parallel (every C_{i-1} is already known); CBC ENCRYPTION is a sequential
 * chain ("Unsuitable", Table 1) and is not offered.
 *  iv : host pointer to 16 bytes, the block preceding in[0] (the IV for the
 *       first shard, the last ciphertext block of the previous shard otherwise).
 *  in == out is NOT allowed (AES_EOVERLAP): block i reads C_{i-1} after block
 *  i-1 may have been overwritten.  Otherwise as aes_ecb_decrypt. */
aes_status aes_cbc_decrypt(const aes_round_keys *rk, int nr, const uint8_t *iv, const void *in, void *out,
                           uint64_t nblocks, void *stream);

/* aes_ecb_batch: many messages, each with its own key, in one launch
 * (ECB of Eq 1 applied per message; the paper's workloads are files of
 * 1,202 .. 1,190,402 bytes, which one launch each would
 * leave launch-bound).  Message i = segs[i]: nblocks 16-byte blocks read at
 * in_base + in_offset and written at out_base + out_offset with round keys
 * keys[key_index] (ek, or dk when decrypt = 1).
 *  keys  : host array of 1..128 round keys (passed by value in the kernel parameters), all
 *          with the same nr (else AES_ENR).
 *  segs  : host array of nsegs descriptors; read during the call only (they are
 *          copied into a library-owned page-locked staging slot -- a ring of
 *          slots per device, each reused only after its previous copy has run --
 *          and from there into a stream-ordered device allocation freed after
 *          the kernel).  Offsets must be multiples of 16 (AES_EALIGN); a segment's
 *          output must equal or be disjoint from its own input (AES_EOVERLAP);
 *          outputs of DIFFERENT segments must not overlap other segments'
 *          inputs or outputs (not checked: O(n^2)); empty segments are allowed.
 *  in_base/out_base : device pointers of the current device, 16-byte aligned.
 * Asynchronous on `stream`; NOT capturable into a CUDA graph (the staged
 * descriptors live in a reused host slot): a stream under capture returns
 * AES_ECAPTURE.  Errors: AES_ENULL, AES_ERANGE (nkeys not in 1..128, key_index
 * out of range, size overflow), AES_ENR, AES_EALIGN, AES_EOVERLAP,
 * AES_ENOTDEVICE, AES_ECUDA, AES_ECAPTURE. */
typedef struct {
    uint64_t in_offset;   /* bytes from in_base  */
    uint64_t out_offset;  /* bytes from out_base */
    uint64_t nblocks;
    uint32_t key_index;
    uint32_t reserved;
} aes_segment;
aes_status aes_ecb_batch(const aes_round_keys *keys, int nkeys, int decrypt, const aes_segment *segs, uint32_t nsegs,
                         const void *in_base, void *out_base, void *stream);

/* Kernel variants (T-table placement).  All variants
 * produce bit-identical output; they differ only in speed.
 *  AES_VAR_DEFAULT    : tuned choice: AES_VAR_HYBRID for ECB messages of 2^23
 *                       blocks (128 MiB) or more, AES_VAR_SMEM_REPL below.
 *  AES_VAR_SMEM_REPL  : Te0..Te3 (Td0..Td3, Si) replicated 32x in shared
 *                       memory, bank == lane, conflict-free by construction.
 *  AES_VAR_SMEM_PLAIN : one copy of each table in shared memory (Li et al.,
 *                       PAPER.md:41); data-dependent bank conflicts.
 *  AES_VAR_CONST      : tables in __constant__ memory (the paper's choice,
 *                       PAPER.md:443); serialises divergent addresses.
 *  AES_VAR_SMEM_REPL_TMA : as SMEM_REPL, with the input states staged into
 *                       shared memory by bulk copies (cp.async.bulk + mbarrier)
 *                       in a 2-stage ring per warp.  states_per_thread must be 1.
 *  AES_VAR_SMEM_ROT   : ONE lane-replicated table (Te0 / Td0) and the other three
 *                       as funnel-shift rotations (Eqs 23-25 are byte rotations
 *                       of Eq 22): 64 KiB of shared memory instead of 128/192.
 *  AES_VAR_GLOBAL     : tables left in global memory, read through the
 *                       read-only L1 path (__ldg); no shared memory.
 *  AES_VAR_HYBRID     : SMEM_REPL T-table warps plus, in the same CTA, warps
 *                       that run a bitsliced (lookup-free, Boolean-circuit
 *                       S-box) cipher on the integer pipe the table lookups
 *                       leave idle; both take 32-block units from a per-CTA
 *                       queue.  states_per_thread must be 1.
 *  AES_VAR_BITSLICE   : every warp bitsliced (8 blocks per thread), no tables;
 *                       the ALU-only point of the ablation (about half the
 *                       T-table rate; no data-dependent memory access or
 *                       branch).  states_per_thread must be 1. */
typedef enum {
    AES_VAR_DEFAULT = 0,
    AES_VAR_SMEM_REPL = 1,
    AES_VAR_SMEM_PLAIN = 2,
    AES_VAR_CONST = 3,
    AES_VAR_SMEM_REPL_TMA = 4,
    AES_VAR_SMEM_ROT = 5,
    AES_VAR_GLOBAL = 6,
    AES_VAR_HYBRID = 7,
    AES_VAR_BITSLICE = 8
} aes_variant;

/* aes_launch_config.flags (bitwise OR):
 *  AES_LAUNCH_TRUSTED_PTRS : skip the two cudaPointerGetAttributes queries
 *                            that classify in/out (AES_ENOTDEVICE); for callers
 *                            that already know both are device memory of the
 *                            current device (e.g. a prepared call that checked
 *                            them once).  A host pointer passed with this flag
 *                            faults in the kernel instead of being rejected.
 *                            Alignment/overlap/size checks still run.
 *  AES_LAUNCH_NO_PDL       : launch without programmatic dependent launch.  By
 *                            default every kernel is launched with the PDL
 *                            attribute: it starts (and fills its shared-memory
 *                            tables) while the previous kernel on the stream
 *                            drains, and waits for that kernel (griddepcontrol
 *                            .wait) before touching in/out.  Results are
 *                            identical either way. */
#define AES_LAUNCH_TRUSTED_PTRS 1
#define AES_LAUNCH_NO_PDL 2

typedef struct {
    int32_t variant;           /* aes_variant                                      */
    int32_t states_per_thread; /* 0 = default; else 1, 2 or 4 (granularity, 8(a) A10) */
    int32_t grid;              /* 0 = persistent default (SMs x resident CTAs)     */
    int32_t flags;             /* AES_LAUNCH_* bits; 0 = checked pointers + PDL    */
} aes_launch_config;

/* Same contract as aes_ecb_encrypt/decrypt (decrypt = 0/1) with an explicit
 * variant; cfg may be NULL (= defaults).  AES_EVARIANT for an unknown variant
 * or states_per_thread value, AES_ERANGE for a negative grid or unknown flag
 * bits.  Work split (every variant): whole trips of grid x 1024 x S blocks
 * grid-stride, the remainder (all of a small message) as one contiguous
 * warp-aligned chunk per CTA, so every launched CTA has work. */
aes_status aes_ecb_launch(const aes_round_keys *rk, int nr, int decrypt, const void *in,
                          void *out, uint64_t nblocks, void *stream,
                          const aes_launch_config *cfg);

/* Host-resident end-to-end path (the paper's timing
 * boundary, "we get back the encrypted data from GPU memory").
 * A pipeline owns `depth` device staging buffers of chunk_bytes each and
 * `depth` streams on the device that is current at creation.  Run copies host
 * -> device, ciphers, and copies device -> host chunk by chunk, with the
 * three stages of different chunks overlapped; it returns when out_host is
 * complete (synchronous).  in_host/out_host: host memory, 16*nblocks bytes,
 * ideally page-locked (pageable memory works but does not overlap);
 * in_host == out_host allowed.  chunk_bytes: multiple of 16, >= 16; depth 1..8.
 * Messages up to 8 MiB whose host buffers are both page-locked and mapped
 * (e.g. cudaHostAlloc / torch pin_memory) skip the staging: the kernel reads
 * and writes them over the link directly (one launch, no copies).
 * A pipeline object is not re-entrant (its staging buffers are shared): use
 * one per host thread.  Pipelines on different devices are independent.
 * Errors: AES_ENULL, AES_ERANGE, AES_ENR, AES_EOVERLAP, AES_ECUDA. */
typedef struct aes_pipeline aes_pipeline;
aes_status aes_pipeline_create(uint64_t chunk_bytes, int depth, aes_pipeline **out);
aes_status aes_pipeline_run(aes_pipeline *p, const aes_round_keys *rk, int nr, int decrypt,
                            const void *in_host, void *out_host, uint64_t nblocks);
aes_status aes_pipeline_destroy(aes_pipeline *p);

/* aes_ecb_trace: parity pin for single rounds (SURVEY.md 8(c) "per-round
 * states"; FIPS-197 App B).  Writes, for each block, the state after
 * AddRoundKey(0) and `rounds` Eq 26 rounds (0 <= rounds <= nr; rounds == nr
 * is the full cipher incl. the final round) computed by the same round code
 * the production kernels use.  decrypt = 1 runs the equivalent inverse cipher
 * with dk.  Same buffer contract as aes_ecb_encrypt; AES_ERANGE for a bad
 * `rounds`.  Test/debug use; not tuned. */
aes_status aes_ecb_trace(const aes_round_keys *rk, int nr, int decrypt, int rounds, const void *in, void *out,
                         uint64_t nblocks, void *stream);

/* Shared-memory gather microbenchmark (the binding roofline):
 * `grid` CTAs x 1024 threads each perform `iters` x 16 conflict-free 32-bit
 * lookups into a lane-replicated 128 KiB table with the same one-PRMT address
 * form as the AES rounds, on `stream`.  sink: device pointer, >= 4*grid*1024
 * bytes, receives a checksum (keeps the loads live).  Time it with events. */
aes_status aes_mb_lds_gather(void *sink, int grid, int iters, void *stream);

const char *aes_status_string(aes_status s);
/* cudaError_t (as int) behind the last AES_ECUDA returned on this thread. */
int aes_last_cuda_error(void);
int aes_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* AES_B200_H */
