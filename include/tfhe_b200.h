/*
 * tfhe_b200.h -- C ABI of the sm_100a batched RNS-CKKS hot path.
 *
 * Drop-in boundary for the reference's operator layer (rnsckks,
 * /root/reference/pkg/src/rnsckks).  The reference has no native FFI of its
 * own: its plugin point is the NTT backend string dispatched in
 * `ntt.transform_rows` (ntt.py:30, 347-363).  Each entry point below replaces
 * one reference operator; the Python host layer (paper_2212_14191_b200/) binds
 * them with ctypes and keeps the reference's names, argument meaning and
 * exceptions.  INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - All data pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors),
 *    u32 canonical residues.  Buffers are level-major (rows, batch, n), one
 *    prime per row (batch.py:22-47 BatchBuffer layout); a ciphertext batch is
 *    (2, level+1, batch, n): component b then a (ckks.py:34-43).
 *  - Small index arrays (limb/prime maps, scalars) are HOST pointers.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *    asynchronous and stream-ordered; nothing synchronises the host.
 *  - The caller owns every buffer, including workspaces (query the size
 *    first); the context owns only its constant tables.
 *  - Return 0 on success, TFHE_EINVAL for bad arguments, TFHE_ECUDA for a
 *    CUDA error; tfhe_last_error() describes the last failure (thread-local).
 *    No exceptions cross the ABI.
 *  - Primes must satisfy q = 1 mod 2n and q < 2^31.
 */
#ifndef TFHE_B200_H
#define TFHE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TFHE_ABI_VERSION 3
#define TFHE_OK 0
#define TFHE_EINVAL 2
#define TFHE_ECUDA 3

/* element-wise op codes for tfhe_eltwise */
#define TFHE_OP_ADD 0    /* ele_add          kernels.py:33-35 */
#define TFHE_OP_SUB 1    /* ele_sub          kernels.py:38-40 */
#define TFHE_OP_MUL 2    /* hada_mult        kernels.py:43-47 */
#define TFHE_OP_NEG 3    /* negate           kernels.py:61-67 */
#define TFHE_OP_SCALAR 4 /* scalar_rows_mult kernels.py:50-58 */

typedef struct TfheCtx TfheCtx;

int tfhe_abi_version(void);
const char* tfhe_last_error(void);

/* Context for degree n = 2^log_n over primes[0..n_chain+n_special): the
 * chain q_0..q_L followed by the special primes (CkksParams.ext_basis,
 * ckks.py:73).  psis[i] is the negacyclic root of primes[i]
 * (params.find_negacyclic_root, params.py:51-62).  Builds and uploads every
 * twiddle table (params.build_twiddles, params.py:198-228; ntt.TwiddleTable,
 * ntt.py:115-165).  n_special may be 0 for transform-only contexts. */
int tfhe_ctx_create(int device, int log_n, const uint32_t* primes, const uint32_t* psis,
                    int n_chain, int n_special, TfheCtx** out);
void tfhe_ctx_destroy(TfheCtx* ctx);
/* n1 x n2 plan actually used (params.build_ntt_plan, params.py:170-175) */
int tfhe_ctx_plan(const TfheCtx* ctx, int* n1, int* n2);
/* How the device factors one transform into tensor-core contractions (any
 * exact factorisation gives the reference's bits): the contraction lengths
 * k0, k1, k2 of its GEMM stages (k2 = 0 for two stages).  n = 2^16 on the
 * three-factor plan: (32, 32, 64) -- a 1024-point column transform split
 * 32 x 32 on chip, then 64-point rows; n = 2^14 / 2^15: (n1, n2, 0) on the
 * twiddle-resident kernel; n = 4096: (64, 64, 0).  int8 tensor work per
 * limb-transform = 32 n (k0 + k1 + k2). */
int tfhe_ctx_transform_plan(const TfheCtx* ctx, int* k0, int* k1, int* k2);

/* ---- transforms --------------------------------------------------------
 * Replaces ntt.transform_rows (ntt.py:347-363), ntt_forward/ntt_inverse
 * (ntt.py:366-385) and batched_apply("ntt"/"intt") (batch.py:88-98).
 * Output row l (of n_limbs) is the transform of input row in_rows[l] taken
 * mod primes[limb_prime[l]], written to output row out_rows[l] (NULL maps =
 * identity).  Input residues may be any u32 (they are reduced implicitly),
 * which is how ModUp/ModDown reuse one source row for many target primes.
 * inverse != 0 includes the n^-1 factor.  `ws` >= tfhe_ntt_workspace_bytes. */
size_t tfhe_ntt_workspace_bytes(const TfheCtx* ctx, int n_limbs, int batch);
int tfhe_ntt(TfheCtx* ctx, const uint32_t* in, uint32_t* out, const int32_t* limb_prime,
             const int32_t* in_rows, const int32_t* out_rows, int n_limbs, int batch,
             int inverse, void* ws, size_t ws_bytes, void* stream);

/* Host-to-host form of tfhe_ntt (the e2e path of ntt.transform_rows /
 * batched_apply on host buffers): rows of host_in (n_limbs, batch, n) are
 * streamed through `staging` (device, >= tfhe_ntt_host_staging_bytes) in
 * chunks, H2D copy / transform / D2H copy overlapped on two internal copy
 * streams and the caller's stream; the call is stream-ordered -- host_out
 * is complete once `stream` reaches this point.  Pinned host buffers give
 * full copy/compute overlap; pageable ones are bounced through pinned slots
 * by a parallel host memcpy, which makes the call host-blocking. */
size_t tfhe_ntt_host_staging_bytes(const TfheCtx* ctx, int n_limbs, int batch);
int tfhe_ntt_host(TfheCtx* ctx, const uint32_t* host_in, uint32_t* host_out,
                  const int32_t* limb_prime, int n_limbs, int batch, int inverse, void* staging,
                  size_t staging_bytes, void* stream);

/* ---- element-wise / automorphism / base conversion ---------------------
 * tfhe_eltwise: out[r] = a[r] op b[r] (or op a[r]) for rows r < rows of
 * per_row elements (per_row % 4 == 0), prime primes[row_prime[r]];
 * `scalars` (host, one per row) for TFHE_OP_SCALAR.
 * Replaces kernels.ele_add/ele_sub/hada_mult/negate/scalar_rows_mult
 * (kernels.py:33-67) and batched_apply's binary kernels (batch.py:107-127). */
int tfhe_eltwise(TfheCtx* ctx, int op, const uint32_t* a, const uint32_t* b, uint32_t* out,
                 const int32_t* row_prime, int rows, int64_t per_row, const uint32_t* scalars,
                 void* stream);
/* x -> x^t on (rows, batch, n); ntt_domain selects the gather form
 * (kernels.py:88-96) or the coefficient-domain signed scatter (:97-107).
 * Replaces apply_automorphism / forbenius_map / conjugate and
 * batched_apply("forbenius_map") (batch.py:99-106). out must not alias in. */
int tfhe_automorphism(TfheCtx* ctx, const uint32_t* in, uint32_t* out, uint32_t galois_t,
                      int ntt_domain, const int32_t* row_prime, int rows, int batch,
                      void* stream);
/* fast_basis_conv (rns.py:118-152): (n_src, batch, n) coefficient rows over
 * primes[src_prime[]] -> (n_dst, batch, n) over primes[dst_prime[]]. */
int tfhe_bconv(TfheCtx* ctx, const uint32_t* in, uint32_t* out, const int32_t* src_prime,
               int n_src, const int32_t* dst_prime, int n_dst, int batch, void* stream);

/* ---- CKKS evaluation (ckks.py:246-381) -----------------------------------
 * Ciphertext batches are (2, level+1, batch, n), NTT domain, over the chain
 * primes q_0..q_level.  Switching keys are (dnum, 2, L+1+K, n), NTT domain,
 * over the full extended basis (SwitchingKey, ckks.py:57-60), shared by the
 * whole batch.  Each call equals the reference's per-member call bit for bit.
 * Workspace: tfhe_ckks_workspace_bytes(ctx, level, batch). */
size_t tfhe_ckks_workspace_bytes(const TfheCtx* ctx, int level, int batch);
/* key_switch (ckks.py:321-352): d (level+1, batch, n) -> out (2, level+1,
 * batch, n) = (ksb, ksa); when `add` is non-NULL it is a (2, level+1, batch,
 * n) buffer added component-wise to the result. */
int tfhe_keyswitch(TfheCtx* ctx, const uint32_t* d, int level, int batch, const uint32_t* key,
                   int dnum, uint32_t* out, const uint32_t* add, void* ws, size_t ws_bytes,
                   void* stream);
/* hmult (ckks.py:265-274): tensor product + relinearising key switch */
int tfhe_hmult(TfheCtx* ctx, const uint32_t* ct0, const uint32_t* ct1, int level, int batch,
               const uint32_t* rlk, int dnum, uint32_t* out, void* ws, size_t ws_bytes,
               void* stream);
/* HMULT + relinearisation + rescale in one pipeline: out (2, level, B, n) equals
 * tfhe_rescale(tfhe_hmult(ct0, ct1)) bit for bit (ref ckks.py:265-274 then
 * :291-311) with 2*level fewer limb-NTTs -- ModDown's and the rescale's forward
 * NTTs merge by linearity (capi.cu: moddown_rescale).  level >= 1.
 * Workspace: tfhe_ckks_workspace_bytes(ctx, level, batch). */
int tfhe_hmult_rescale(TfheCtx* ctx, const uint32_t* ct0, const uint32_t* ct1, int level,
                       int batch, const uint32_t* rlk, int dnum, uint32_t* out, void* ws,
                       size_t ws_bytes, void* stream);
/* rescale (ckks.py:291-311): (2, level+1, batch, n) -> (2, level, batch, n) */
int tfhe_rescale(TfheCtx* ctx, const uint32_t* ct, int level, int batch, uint32_t* out, void* ws,
                 size_t ws_bytes, void* stream);
/* hrotate / hconjugate (ckks.py:276-289): automorphism x -> x^galois_t then
 * key switch of the a component; galois_t = 5^r mod 2n, or 2n-1 to conjugate */
int tfhe_hrotate(TfheCtx* ctx, const uint32_t* ct, int level, int batch, uint32_t galois_t,
                 const uint32_t* key, int dnum, uint32_t* out, void* ws, size_t ws_bytes,
                 void* stream);
/* hadd / hsub (ckks.py:246-256) are tfhe_eltwise over the 2*(level+1) rows. */

/* ---- limb-partitioned evaluation (optional multi-GPU mode) ----
 * Each of G ranks owns the chain rows [row_lo, row_lo + n_rows) of every
 * ciphertext.  Only the key switch needs other ranks' data: the caller
 * INTTs its own rows of d (tfhe_ntt, inverse), all-gathers them (one NCCL
 * all-gather per key switch) into y_full = (level+1, batch, n) coefficient
 * rows, and every rank then raises ALL slices to its own rows plus the K
 * specials (specials computed redundantly, no second collective) and does
 * ModDown locally.  Concatenating the ranks' outputs equals the
 * unpartitioned call (ckks.key_switch, ckks.py:321-381) bit for bit.
 *
 * tfhe_tensor_product: hmult's d0 = b0 b1, d1 = a0 b1 + a1 b0, d2 = a0 a1
 *   (ckks.py:265-271) over local rows: ct (2, n_rows, batch, n) ->
 *   out (3, n_rows, batch, n).
 * tfhe_keyswitch_part: d_local (n_rows, batch, n) NTT domain, y_full as
 *   above -> out (2, n_rows, batch, n); with `add`, its first add_components
 *   (1: b only, as hrotate's phi(b); 2: both, as hmult's d0/d1) of
 *   (2, n_rows, batch, n) are added.
 * tfhe_rescale_part: ct_local (2, n_rows, batch, n) and top_coeff = the
 *   INTT of both components' top limb (2, batch, n), broadcast by its owner
 *   -> out (2, n_keep, batch, n), n_keep = local rows below `level`
 *   (_rescale_poly, ckks.py:301-311). */
int tfhe_tensor_product(TfheCtx* ctx, const uint32_t* ct0, const uint32_t* ct1, int row_lo,
                        int n_rows, int batch, uint32_t* out, void* stream);
int tfhe_keyswitch_part(TfheCtx* ctx, const uint32_t* d_local, const uint32_t* y_full, int level,
                        int batch, const uint32_t* key, int dnum, int row_lo, int n_rows,
                        uint32_t* out, const uint32_t* add, int add_components, void* ws,
                        size_t ws_bytes, void* stream);
int tfhe_rescale_part(TfheCtx* ctx, const uint32_t* ct_local, const uint32_t* top_coeff,
                      int level, int batch, int row_lo, int n_rows, uint32_t* out, void* ws,
                      size_t ws_bytes, void* stream);

/* ---- diagnostics -----------------------------------------------------------
 * Fault injection for the selftest (ref cli.py:77-87 corrupts the twiddle
 * tables its backend actually uses): flips one byte of prime `prime`'s
 * FORWARD twiddle tables on the device (every stage table the context built
 * for it), so every later forward transform mod that prime is wrong.  Only
 * for a private context the caller then destroys. */
int tfhe_debug_corrupt_twiddle(TfheCtx* ctx, int prime);

/* ---- client-side CRT (ref rns.py:77-115, ckks.py:194-213) -----------------
 * tfhe_crt_decompose: n signed coefficients (device; kind 0 = int64, kind 1 =
 * float64 rounded half to even like np.rint, any finite magnitude) -> n_limbs
 * canonical residue rows `out` (n_limbs, n), row l mod prime limb_prime[l]:
 * crt_decompose of the encode / _encode_signed path.
 * tfhe_crt_compose: residue rows (n_limbs, n) -> the CRT representative
 * centred in (-Q/2, Q/2] (ckks._centered), as float64 rounded half to even
 * (Python float(int); +-inf past the double range) into out_f64 (nullable) and
 * as n_words-word little-endian two's complement into out_words (nullable,
 * layout (n_words, n)).  tfhe_crt_words: words of Q for that basis (use
 * n_words >= words + 1 for the sign). */
int tfhe_crt_decompose(TfheCtx* ctx, const void* coeffs, int kind, int64_t n,
                       const int32_t* limb_prime, int n_limbs, uint32_t* out, void* stream);
int tfhe_crt_words(const TfheCtx* ctx, const int32_t* limb_prime, int n_limbs);
int tfhe_crt_compose(TfheCtx* ctx, const uint32_t* rows, const int32_t* limb_prime, int n_limbs,
                     int64_t n, double* out_f64, uint32_t* out_words, int n_words, void* stream);

/* ---- per-kernel device timing (measurement aid) ---------------------------
 * While enabled (process-wide), every launch of the library's NTT-pass,
 * fused-NTT and base-conversion kernels is bracketed by two CUDA events
 * recorded on its launching stream.  tfhe_profile_read waits for those events
 * and writes one line per kernel family, "name<TAB>launches<TAB>total_ms\n",
 * into buf (NUL-terminated, truncated to len), then forgets the records.
 * Returns the number of families, or a negative code. */
int tfhe_profile_enable(int enable);
int tfhe_profile_read(char* buf, size_t len);

#ifdef __cplusplus
}
#endif
#endif /* TFHE_B200_H */
