/* sfxb_cuda.h — C ABI of the B200-native Paillier plugin (libsfxb_cuda.so).
 *
 * This is the thin layer between host code and the sm_100a kernels.  It
 * replaces the three scalar-path virtuals of the reference's
 * `sfxb::EncryptionPlugin` (/root/reference/proj/include/sfxb/
 * secure_processor.hpp:112-143) as implemented by `PaillierPlugin`
 * (proj/src/secure_processor.cpp:553-746), and the HE primitives they bottom
 * out in (proj/src/he.cpp:87-143).  The C++ adapter that re-exposes these as an
 * EncryptionPlugin lives in paper_2504_03909_b200/host/ (INTEGRATION.md).
 *
 * Conventions
 *   - Big integers are little-endian arrays of uint32_t limbs.  A value mod n
 *     takes `n_words` limbs, a ciphertext (mod n²) takes 2·n_words limbs.
 *   - All pointers are caller-owned and only used for the duration of the
 *     call.  Host-pointer entry points are synchronous.  `*_dev` entry points
 *     take device pointers on the context's device, are ordered on the
 *     context's stream and return after enqueueing unless stated otherwise.
 *   - Every entry point returns SFXB_OK (0) or a negative code; the message
 *     is in sfxb_last_error(ctx) and repeats the reference's exception text
 *     where one exists (e.g. "not coprime", "bin index out of range in
 *     accumulate", "decrypt requested without private key material").
 *   - A context is used by one host thread at a time (the reference calls one
 *     plugin instance from one thread at a time, federation.cpp:509-516);
 *     distinct contexts may be used concurrently.
 *   - There is no CPU fallback: without a usable sm_100 device every call
 *     fails with SFXB_ERR_CUDA.
 */
#ifndef SFXB_CUDA_H
#define SFXB_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    SFXB_OK = 0,
    SFXB_ERR_ARG = -1,         /* bad argument / shape (reference: sfxb::Error)        */
    SFXB_ERR_CUDA = -2,        /* CUDA runtime failure or no device                     */
    SFXB_ERR_AUTH = -3,        /* private key required (reference: AuthorizationError) */
    SFXB_ERR_RANGE = -4,       /* value out of range (plaintext, blinding, ciphertext)  */
    SFXB_ERR_COPRIME = -5,     /* value not coprime to n                                */
    SFXB_ERR_UNSUPPORTED = -6, /* key size / shape outside the built size classes      */
};

typedef struct sfxb_ctx sfxb_ctx;

/* ---- key context -------------------------------------------------------
 * Replaces make_paillier_plugin(const PaillierPublicKey&, ...) and
 * make_paillier_plugin(const PaillierKeypair&, ...)
 * (secure_processor.hpp:155-158, secure_processor.cpp:754-762).
 * p, q: NULL for a public-key-only holder (passive party,
 * federation.cpp:83-85); otherwise pq_words limbs each.  n up to 3072 bits. */
int sfxb_ctx_create(sfxb_ctx **out, int device, const uint32_t *n, uint32_t n_words,
                    const uint32_t *p, const uint32_t *q, uint32_t pq_words);
/* One key on several GPUs of this process (SURVEY §8e inside the reference's
 * single-process plugin; replaces the same factories).  `devices` lists 1–16
 * CUDA devices, one shard each (a device may repeat: its shards then share
 * that GPU — the logic check used on one-GPU machines).  Distinct devices need
 * peer access (NVLink/NVSwitch); otherwise SFXB_ERR_UNSUPPORTED.
 * The host-buffer entry points use every shard:
 *   sfxb_encrypt / sfxb_encrypt_plain / sfxb_add / sfxb_decrypt — contiguous
 *     element ranges, one per GPU (≥ 4096 exponentiations per GPU);
 *   sfxb_gh_upload — gh rows in contiguous row shards, one per GPU;
 *   sfxb_accumulate / sfxb_accumulate_gh / sfxb_accumulate_tree_gh — each GPU
 *     builds partial histograms of its rows (Montgomery form); GPU k then
 *     multiplies slot slice k of every node across all GPUs, reading the
 *     peers' partials over NVLink in one kernel (a modular product: no NCCL
 *     reduction op can combine ciphertexts), applies sibling subtraction on
 *     its slice and writes its slice of the caller's output;
 *   sfxb_decrypt_tree — every node's slots in per-GPU slices.
 * Results and counters are identical to a single-device context.  The
 * encrypt/decrypt/reduce *_dev entry points act on shard 0 only (device
 * pointers of devices[0]); sfxb_gh_from_dev and sfxb_accumulate*_dev return
 * SFXB_ERR_UNSUPPORTED on a group (its gradient handle is host-API only). */
int sfxb_ctx_create_multi(sfxb_ctx **out, const int *devices, uint32_t n_devices, const uint32_t *n,
                          uint32_t n_words, const uint32_t *p, const uint32_t *q, uint32_t pq_words);
/* Page-locked host memory for callers' marshalling buffers: host-pointer
 * entry points copy from / to it at full PCIe speed (pageable buffers are
 * staged by the driver).  NULL on failure. */
void *sfxb_host_alloc(size_t bytes);
void sfxb_host_free(void *p);
/* visible CUDA devices (0 without a driver/GPU) */
int sfxb_device_count(void);
/* shards of a context (1 for sfxb_ctx_create) and the device of shard k */
uint32_t sfxb_ctx_n_shards(const sfxb_ctx *ctx);
/* Encryptions whose exponentiations run concurrently on the context's GPU(s)
 * (one wave of the encrypt kernels; summed over shards): batches that are
 * whole multiples of it leave no partial last wave.  0 on error. */
size_t sfxb_ctx_enc_wave(const sfxb_ctx *ctx);
int sfxb_ctx_shard_device(const sfxb_ctx *ctx, uint32_t k);
void sfxb_ctx_destroy(sfxb_ctx *ctx);
const char *sfxb_last_error(const sfxb_ctx *ctx);
/* error text of the last failed sfxb_ctx_create on this thread */
const char *sfxb_create_error(void);
uint32_t sfxb_ctx_n_words(const sfxb_ctx *ctx);
uint32_t sfxb_ctx_ct_words(const sfxb_ctx *ctx);
int sfxb_ctx_has_private(const sfxb_ctx *ctx);
/* key_id_of(n): FNV-1a-64 over the lower-case hex digits of n (he.cpp:30-38) */
uint64_t sfxb_ctx_key_id(const sfxb_ctx *ctx);
/* number of our kernels launched by this context so far (bench evidence) */
uint64_t sfxb_ctx_launches(const sfxb_ctx *ctx);

/* ---- encrypt -------------------------------------------------------------
 * Batch of encrypt_with_r (he.cpp:87-99) as driven by PaillierPlugin::
 * encrypt_gh (secure_processor.cpp:574-585):
 *     c_i = ((1 + m_i·n) mod n²) · (r_i^n mod n²) mod n²
 * with m_i = q_i mod n, q_i the fixed-point value fixed_encode_ll(x, scale)
 * (fixed_point.hpp:13-15; encode_fixed's range checks he.cpp:125-136 are the
 * caller's, see sfxb_encode_check).  r: count × n_words limbs, 1 < r < n.
 * With p, q present the kernel uses CRT (mod p², q²); otherwise r^n mod n².
 * r_flags (optional, count bytes): set to 1 where r shares a factor with n
 * (only detectable with p, q; the call then fails with SFXB_ERR_COPRIME so the
 * caller can re-draw per the reference's rejection rule, he.cpp:19-28). */
int sfxb_encrypt(sfxb_ctx *ctx, const int64_t *q_fixed, const uint32_t *r, size_t count,
                 uint32_t *out_cts, uint8_t *r_flags);
/* encrypt_with_r for arbitrary plaintexts m ∈ [0, n) given as count × n_words
 * little-endian words (the packed-vector path: pack_encrypt, he.cpp:220-232,
 * plaintexts from pack_plain).  Same r semantics, flags and errors as
 * sfxb_encrypt, plus "encrypt: plaintext out of range [0, n)" (he.cpp:88). */
int sfxb_encrypt_plain(sfxb_ctx *ctx, const uint32_t *m_words, const uint32_t *r_words, size_t count,
                       uint32_t *out_cts, uint8_t *r_flags);
int sfxb_encrypt_dev(sfxb_ctx *ctx, const int64_t *d_q_fixed, const uint32_t *d_r, size_t count,
                     uint32_t *d_out_cts, uint8_t *d_r_flags);

/* ---- offline / online encryption ----------------------------------------
 * The blinding power r^n mod n² of encrypt_with_r (he.cpp:87-99) does not
 * depend on the plaintext, so it can be computed ahead of the call that
 * needs it — e.g. while the host runs the protocol between trees — and the
 * call then only does c = (1 + m·n)·r^n mod n² (3 multiplications mod n²
 * instead of the exponentiation).  Ciphertexts are bit-identical as long as
 * the queued powers are consumed in the order their r were drawn (the
 * adapter draws them from the reference's HeRng stream, he.cpp:11-28).
 * A queue lives on one device for one key; appends and encrypts may use
 * different contexts of that key on that device (e.g. a low-priority
 * background context).  Single-device contexts only. */
typedef struct sfxb_blind sfxb_blind;
int sfxb_blind_create(sfxb_ctx *ctx, size_t capacity, sfxb_blind **out);
void sfxb_blind_free(sfxb_blind *b);
size_t sfxb_blind_size(const sfxb_blind *b);
/* append r_i^n mod n² for `count` host blinding factors (n_words limbs each,
 * 1 < r < n); synchronous.  r_flags as sfxb_encrypt; on SFXB_ERR_COPRIME
 * nothing is appended. */
int sfxb_blind_append(sfxb_ctx *ctx, sfxb_blind *b, const uint32_t *r, size_t count, uint8_t *r_flags);
/* drop the first `count` queued powers (their r were consumed elsewhere) */
int sfxb_blind_pop(sfxb_blind *b, size_t count);
/* c_i = (1 + m_i·n)·Y_i mod n² with Y_i the first `count` queued powers
 * (consumed); m_i from q_fixed (as sfxb_encrypt) or m_words (as
 * sfxb_encrypt_plain, with its range check) — exactly one of the two. */
int sfxb_encrypt_blind(sfxb_ctx *ctx, sfxb_blind *b, const int64_t *q_fixed, const uint32_t *m_words, size_t count,
                       uint32_t *out_cts);
/* recreate the context's stream at the lowest priority (background work
 * that should yield to other contexts' kernels at block boundaries) */
int sfxb_ctx_set_low_priority(sfxb_ctx *ctx);

/* encode_fixed's checks (he.cpp:125-136) without the mpz work: returns
 * SFXB_OK and q = llround(ldexp(x, scale)), or SFXB_ERR_RANGE with the
 * reference's message. */
int sfxb_encode_check(sfxb_ctx *ctx, double x, uint32_t scale_bits, int64_t *q_out);
/* Gradients on the device: compute_gradients (gbdt.cpp:
 * 69-80) from probabilities and 0/1 labels, quantize_gradients (:82-87) and
 * encode_fixed (he.cpp:125-136) — d_q: 2n fixed-point plaintexts (g, h
 * interleaved) for sfxb_encrypt_dev; d_gh (optional): the 2n quantized
 * doubles.  Bit-identical to the reference's host arithmetic (one IEEE
 * operation per step).  *first_bad = the first value failing encode_fixed's
 * checks (2n when none; the call then returns SFXB_ERR_RANGE with its
 * message).  Device pointers; synchronous. */
int sfxb_gradients_dev(sfxb_ctx *ctx, const double *d_prob, const uint8_t *d_labels, size_t n, uint32_t scale_bits,
                       int64_t *d_q, double *d_gh, size_t *first_bad);
/* The same for `count` values on all host threads (encrypt_gh's encode of a
 * whole GhPayload): q_out[i] for every value before the first failing one;
 * *first_bad = index of the first value that fails (count when none) and the
 * call returns SFXB_ERR_RANGE with that value's message. */
int sfxb_encode_batch(sfxb_ctx *ctx, const double *x, size_t count, uint32_t scale_bits, int64_t *q_out,
                      size_t *first_bad);

/* ---- ciphertext addition (add_ciphertexts, he.cpp:117-121), batched -------- */
int sfxb_add(sfxb_ctx *ctx, const uint32_t *a, const uint32_t *b, size_t count, uint32_t *out);

/* ---- encrypted histogram ---------------------------------------------------
 * PaillierPlugin::accumulate_rows (secure_processor.cpp:587-620) for one
 * party and one frontier:
 *   gh_cts      2·n_samples ciphertexts, interleaved Enc(g_i), Enc(h_i)
 *   bins        n_features columns of n_samples uint16 (column-major,
 *               dataset.hpp:55-57), feature order = output order
 *   node_offsets[n_nodes+1] / rows: the rows of each frontier node
 *   out_slots   n_nodes × n_features × n_bins × 2 ciphertexts; slot
 *               ((node·J + f)·K + b)·2 + {0:G, 1:H}; empty slots are the
 *               literal 1 (trivial_zero, he.cpp:123)
 *   additions   += the reference's ciphertext_additions for this call,
 *               Σ_slots max(count − 1, 0) (fold_into, :724-732)
 * Errors: "bin index out of range in accumulate", row index out of range. */
int sfxb_accumulate(sfxb_ctx *ctx, const uint32_t *gh_cts, uint32_t n_samples,
                    const uint16_t *bins, uint32_t n_features, const uint32_t *node_offsets,
                    uint32_t n_nodes, const uint32_t *rows, uint32_t n_bins, uint32_t *out_slots,
                    uint64_t *additions);

/* Device-resident gradient ciphertexts (Montgomery form), reusable across
 * the levels of a tree; the C++ adapter keys it on content. */
typedef struct sfxb_gh sfxb_gh;
int sfxb_gh_upload(sfxb_ctx *ctx, const uint32_t *gh_cts, uint32_t n_samples, sfxb_gh **out);
int sfxb_gh_from_dev(sfxb_ctx *ctx, const uint32_t *d_gh_cts, uint32_t n_samples, sfxb_gh **out);
void sfxb_gh_free(sfxb_gh *gh);

/* accumulate_rows with HOST bins / frontier / output over a resident gh
 * (the C++ adapter's call: the 2·n_samples ciphertexts cross PCIe once per
 * GhPayload, not once per tree level). */
int sfxb_accumulate_gh(sfxb_ctx *ctx, const sfxb_gh *gh, const uint16_t *bins, uint32_t n_features,
                       const uint32_t *node_offsets, uint32_t n_nodes, const uint32_t *rows,
                       uint32_t n_bins, uint32_t *out_slots, uint64_t *additions);

/* Histogram over a resident gh with device-resident bins and frontier.
 * mont_out != 0 leaves the slots in Montgomery form (partials for the
 * multi-GPU reduce); additions is synchronous (host) and may be NULL. */
int sfxb_accumulate_dev(sfxb_ctx *ctx, const sfxb_gh *gh, const uint16_t *d_bins,
                        uint32_t n_features, const uint32_t *d_node_offsets, uint32_t n_nodes,
                        const uint32_t *d_rows, uint32_t n_rows, uint32_t n_bins,
                        uint32_t *d_out_slots, int mont_out, uint64_t *additions);

/* Tree mode — sibling subtraction: parent[i] is the index of
 * frontier node i's parent in the previous tree-mode call on this context
 * (−1: none; the caller guarantees rows(parent) = rows(child a) ∪ rows(child b)
 * for parents with exactly two children listed).  For such siblings only the
 * child with fewer rows is multiplied out; the other is derived as
 * hist(parent)·hist(small)⁻¹ mod n² (one batch inversion per call).  Results,
 * `additions` and the output layout are identical to sfxb_accumulate — the
 * residues are unique.  The context caches the last tree-mode call's
 * histograms; sfxb_tree_reset, freeing the gh handle or a call with another
 * gh / feature count / bin count forgets them. */
int sfxb_accumulate_tree_dev(sfxb_ctx *ctx, const sfxb_gh *gh, const uint16_t *d_bins,
                             uint32_t n_features, const uint32_t *d_node_offsets,
                             const uint32_t *h_node_offsets, uint32_t n_nodes, const uint32_t *d_rows,
                             uint32_t n_rows, uint32_t n_bins, const int32_t *h_parent,
                             uint32_t *d_out_slots, int mont_out, uint64_t *additions);
int sfxb_accumulate_tree_gh(sfxb_ctx *ctx, const sfxb_gh *gh, const uint16_t *bins, uint32_t n_features,
                            const uint32_t *node_offsets, uint32_t n_nodes, const uint32_t *rows,
                            uint32_t n_bins, const int32_t *parent, uint32_t *out_slots,
                            uint64_t *additions);
int sfxb_tree_reset(sfxb_ctx *ctx);
/* Device-resident bin columns (n_features × n_samples u16, column-major,
 * dataset.hpp:55-57): the reference's bins are fixed for a whole training
 * run, so the adapter uploads them once (keyed on their content) instead of
 * once per accumulate_rows call.  sfxb_accumulate_tree_bins is
 * sfxb_accumulate_tree_gh with the handle's columns (feature count =
 * the handle's).  Single-device contexts only. */
typedef struct sfxb_bins sfxb_bins;
int sfxb_bins_upload(sfxb_ctx *ctx, const uint16_t *bins, uint32_t n_features, uint32_t n_samples, sfxb_bins **out);
void sfxb_bins_free(sfxb_bins *b);
int sfxb_accumulate_tree_bins(sfxb_ctx *ctx, const sfxb_gh *gh, const sfxb_bins *bins, const uint32_t *node_offsets,
                              uint32_t n_nodes, const uint32_t *rows, uint32_t n_bins, const int32_t *parent,
                              uint32_t *out_slots, uint64_t *additions);
/* number of frontier nodes obtained by sibling subtraction on this context */
uint64_t sfxb_ctx_tree_derived(const sfxb_ctx *ctx);

/* K4: element-wise product of `parts` partial histograms (Montgomery form,
 * each n_slots ciphertexts, contiguous) into d_out (plain form, n_slots).
 * Used after the all-gather of per-GPU row-shard partials (homomorphic
 * addition is a modular product, so an NCCL sum cannot combine them). */
int sfxb_reduce_partials_dev(sfxb_ctx *ctx, const uint32_t *d_parts, uint32_t parts,
                             size_t n_slots, uint32_t *d_out);

/* ---- rank-sliced histograms (one process per GPU; SURVEY §8e under torchrun) ----
 * The device group's algorithm with the exchange left to the caller's
 * collective (NCCL all_to_all).  Per level and party, on every rank:
 *   1. sfxb_accumulate_part_dev: Montgomery-form partial histograms of this
 *      rank's rows (frontier renumbered to the rank's gh rows; host offsets
 *      h_node_offsets), nodes that sibling subtraction will derive skipped,
 *      written as `world` slot slices, rank-major:
 *      d_send[k][node][j] = partial slot k·jl + j of node, jl =
 *      sfxb_slice_width(J, K, world), world × n_nodes × jl ciphertexts;
 *      d_real: 2·n_nodes·J·K per-slot counts of non-trivial ciphertexts.
 *   2. the caller: all_to_all of d_send (slice k to rank k) and a SUM
 *      all_reduce of d_real; sfxb_count_additions_dev on the summed counts
 *      gives the reference's ciphertext_additions.
 *   3. sfxb_combine_slices_dev: product of the world received slices
 *      (d_recv, rank-major), sibling subtraction on this rank's slice against
 *      the slice it cached at the previous level, plain slice n_nodes × jl to
 *      d_out.
 * h_parent (tree mode, NULL = direct) indexes the previous level's nodes;
 * h_node_sizes are the GLOBAL row counts of this level's nodes (every rank
 * must choose the same smaller sibling).  All device pointers on the
 * context's device; synchronous. */
uint32_t sfxb_slice_width(uint32_t n_features, uint32_t n_bins, uint32_t world);
int sfxb_accumulate_part_dev(sfxb_ctx *ctx, const sfxb_gh *gh, const uint16_t *d_bins, uint32_t n_features,
                             const uint32_t *d_node_offsets, const uint32_t *h_node_offsets, uint32_t n_nodes,
                             const uint32_t *d_rows, uint32_t n_rows, uint32_t n_bins, const int32_t *h_parent,
                             const uint32_t *h_node_sizes, uint32_t world, uint32_t *d_send, uint32_t *d_real);
int sfxb_combine_slices_dev(sfxb_ctx *ctx, const sfxb_gh *gh, const uint32_t *d_recv, uint32_t world, uint32_t rank,
                            uint32_t n_nodes, uint32_t n_features, uint32_t n_bins, const int32_t *h_parent,
                            const uint32_t *h_node_sizes, uint32_t *d_out);
int sfxb_count_additions_dev(sfxb_ctx *ctx, const uint32_t *d_real, size_t n, uint64_t *additions);

/* ---- decrypt -----------------------------------------------------------------
 * PaillierPlugin::decrypt_histogram / decrypt_slot (secure_processor.cpp:
 * 679-719, :734-738) + decrypt (he.cpp:105-115) + decode_fixed (:138-143):
 * slots equal to 1 decode to 0.0 and are not counted; others are decrypted
 * (CRT mod p², q²; bit-identical to the reference's c^λ mod n² path) and
 * decoded exactly like mpz_get_d (truncation) then ldexp(−scale).
 * out_plain (optional): count × n_words decrypted plaintexts.
 * Errors: SFXB_ERR_AUTH without p, q; "ciphertext out of range";
 * "ciphertext not coprime to modulus". */
int sfxb_decrypt(sfxb_ctx *ctx, const uint32_t *cts, size_t count, uint32_t scale_bits,
                 double *out_values, uint32_t *out_plain, uint64_t *decryptions);
int sfxb_decrypt_dev(sfxb_ctx *ctx, const uint32_t *d_cts, size_t count, uint32_t scale_bits,
                     double *d_out_values, uint32_t *d_out_plain, uint64_t *decryptions);
/* Tree-level decrypt with verified sibling reuse (B200-side extension of
 * decrypt_histogram, secure_processor.cpp:679-719; same outputs and counter).
 * cts: n_nodes × slots_per_node ciphertexts of one histogram stream `tag`
 * (node-major).  parent[i] (optional, −1 = none) indexes the nodes of the
 * previous call with the same tag.  For two children a, b of one parent P the
 * context checks, per slot, ct_a·ct_b ≡ ct_P (mod n²) on the GPU; where it
 * holds, Dec(ct_b) = Dec(ct_P) − Dec(ct_a) mod n (Paillier is a group
 * homomorphism Z*_{n²} → Z_n) replaces the CRT exponentiations.  Slots whose
 * check fails are decrypted normally, so a wrong or hostile `parent` costs
 * time, never correctness.  `decryptions` counts every non-trivial slot, as
 * the reference does.  Each call becomes the cached parent level of `tag`. */
int sfxb_decrypt_tree(sfxb_ctx *ctx, uint64_t tag, const uint32_t *cts, uint32_t n_nodes,
                      uint32_t slots_per_node, const int32_t *parent, uint32_t scale_bits,
                      double *out_values, uint64_t *decryptions);
/* slots sfxb_decrypt_tree obtained by verified sibling reuse on this context */
uint64_t sfxb_ctx_dec_derived(const sfxb_ctx *ctx);

/* ---- stream / timing helpers (bench + tests) ---------------------------------- */
void *sfxb_ctx_stream(sfxb_ctx *ctx); /* cudaStream_t of the context */
int sfxb_ctx_sync(sfxb_ctx *ctx);
/* CUDA-event timing of the hot kernel families on the context stream
 * (0: K2 segmented product, 1: K1 encrypt exponentiations, 2: K3 decrypt
 * exponentiation).  Enabling resets the accumulators. */
int sfxb_ctx_profile(sfxb_ctx *ctx, int enable);
int sfxb_ctx_kernel_time(sfxb_ctx *ctx, int family, uint64_t *launches, double *ms);
/* as above plus the Montgomery multiplications those launches executed:
 * families 0, 3 (3: sibling-subtraction batch inversion / derivation) count
 * multiplications mod n²; families 1, 2 count multiplications mod p² (the
 * CRT exponentiations; encrypt step 1 mod p counts 1/4). */
int sfxb_ctx_kernel_stats(sfxb_ctx *ctx, int family, uint64_t *launches, double *ms, uint64_t *modmuls);
/* integer-multiply peak microbenchmark: IMAD.WIDE.U32(.X) 32×32→64 products/s */
int sfxb_imad_peak(int device, double *products_per_s, double *sm_clock_mhz);

#ifdef __cplusplus
}
#endif

#endif /* SFXB_CUDA_H */
