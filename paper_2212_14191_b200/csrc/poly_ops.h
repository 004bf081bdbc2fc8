// Launchers for the HBM-bound polynomial kernels (poly_ops.cu) and the base
// conversion (bconv_tc.cu: int8 tensor cores, element-wise for tiny shapes).
#pragma once
#include <vector>
#include "tfhe_internal.h"

namespace tfhe {

constexpr int kMaxRows = 256;         // rows addressed by one element-wise launch
constexpr int kMaxBconvSrc = 16;
constexpr int kMaxBconvDst = 128;

enum PolyOp : int { OP_ADD = 0, OP_SUB = 1, OP_MUL = 2, OP_NEG = 3, OP_SCALAR = 4 };

struct BconvArgs {
  int n_src, n_dst;
  int16_t src_prime[kMaxBconvSrc];
  int16_t dst_prime[kMaxBconvDst];
  int16_t copy_from[kMaxBconvDst];            // >=0: dst row copies src row (shared prime)
  uint32_t qhat_inv[kMaxBconvSrc], qhat_inv_shoup[kMaxBconvSrc];
  uint32_t factor[kMaxBconvSrc * kMaxBconvDst];  // (Q/q_s) mod p_t, indexed s*kMaxBconvDst+t
};

int launch_binary(const Ctx& c, int op, const uint32_t* a, const uint32_t* b, uint32_t* out,
                  const int16_t* row_prime, int rows, int64_t per_row, cudaStream_t st);
int launch_unary(const Ctx& c, int op, const uint32_t* a, uint32_t* out, const int16_t* row_prime,
                 const uint32_t* scalars, int rows, int64_t per_row, cudaStream_t st);
// optional slice-row key-switch MAC fused into the tensor product: for rows
// r < rows of d2, acc_b[r] = d2[r] kb[key_off[r] + coef], acc_a likewise
struct TensorMac {
  const uint32_t* kb;
  const uint32_t* ka;
  uint32_t* acc_b;
  uint32_t* acc_a;
  int rows, log_n;
  int64_t key_off[kMaxRows];
};
int launch_tensor(const Ctx& c, const uint32_t* b0, const uint32_t* a0, const uint32_t* b1,
                  const uint32_t* a1, uint32_t* d0, uint32_t* d1, uint32_t* d2,
                  const int16_t* row_prime, int rows, int64_t per_row, cudaStream_t st,
                  const TensorMac* mac = nullptr);
int launch_ks_mac(const Ctx& c, const uint32_t* x, const uint32_t* kb, const uint32_t* ka,
                  uint32_t* acc_b, uint32_t* acc_a, const int16_t* row_prime,
                  const int64_t* key_off, int rows, int batch, int first, cudaStream_t st);
// hoisted HROTATE slice MAC: acc_b = phi_t(x) kb + pmod phi_t(base), acc_a = phi_t(x) ka
// (NTT-domain phi; perm_x = 0 reads x unpermuted)
int launch_ks_mac_rot(const Ctx& c, const uint32_t* x, const uint32_t* base, const uint32_t* kb,
                      const uint32_t* ka, uint32_t* acc_b, uint32_t* acc_a,
                      const int16_t* row_prime, const int64_t* key_off, const uint32_t* pmod,
                      int rows, int batch, uint32_t t, int perm_x, cudaStream_t st);
int launch_automorph(const Ctx& c, const uint32_t* in, uint32_t* out, uint32_t t, int ntt_domain,
                     const int16_t* row_prime, int rows, int batch, cudaStream_t st);
// CRT (de)composition rows: prime index per residue row (csrc/crt.cu)
constexpr int kMaxCrtRows = 128;
struct CrtRows {
  int n;
  int16_t prime[kMaxCrtRows];
};
// kind 0: int64 coefficients; kind 1: float64, rounded half to even (np.rint)
int launch_crt_decompose(const Ctx& c, const void* in, int kind, int64_t n, const CrtRows& rows,
                         uint32_t* out, cudaStream_t st);
// constants for crt_compose (host): returns W = words of Q
int crt_compose_constants(const Ctx& c, const int16_t* prime_ids, int L, std::vector<uint32_t>& out);
int crt_compose_words(const Ctx& c, const int16_t* prime_ids, int L);
int launch_crt_compose(const Ctx& c, const uint32_t* rows, int64_t n, const uint32_t* d_cst, int W,
                       const CrtRows& lr, double* out_f, uint32_t* out_w, int n_words,
                       cudaStream_t st);
// exact_copies = false: rows of targets that are source primes may be left
// with don't-care values (callers that never read them)
// n_comp > 1: that many independent conversions with the same bases, inputs /
// outputs `in_cstride` / `out_cstride` elements apart (one launch when the
// element-wise path applies)
int launch_bconv(const Ctx& c, const uint32_t* in, uint32_t* out, const BconvArgs& ba, int batch,
                 cudaStream_t st, bool exact_copies = true, int n_comp = 1,
                 int64_t in_cstride = 0, int64_t out_cstride = 0);

// Fused ModDown + rescale preparation, per row l = (component, chain row i < top):
//   X = acc[acc_row] * P^-1 + base[base_row]     (in place; base_row < 0: none)
//   W = conv[conv_row] * P^-1 + (T[t_row] mod q_i)   -> w[w_row]  (may be in place)
// so that NTT_i(W) = NTT_i(conv) P^-1 + NTT_i(T) and
// (X - NTT_i(W)) q_top^-1 = rescale(ModDown(.)) exactly (see capi.cu).
struct MdRsArgs {
  int16_t prime[kMaxRows];
  int16_t acc_row[kMaxRows], base_row[kMaxRows], conv_row[kMaxRows], t_row[kMaxRows];
  int16_t w_row[kMaxRows];
  uint32_t pinv[kMaxRows], pinv_shoup[kMaxRows];
};
int launch_md_rescale_prep(const Ctx& c, uint32_t* acc, const uint32_t* base, const uint32_t* conv,
                           const uint32_t* t, uint32_t* w, const MdRsArgs& ar, int rows,
                           int64_t per_row, cudaStream_t st);

}  // namespace tfhe
