// CRT decomposition / composition on the device: the integer steps of the
// client-side encode and decode.
//
//  * crt_decompose (ref rns.py:77-90, called by ckks.py:194-198 encode and
//    ckks.py:100-109 _encode_signed): signed coefficients -> canonical residue
//    rows.  The encode path feeds float64 values and rounds them here with
//    rint (round half to even, as np.rint); any finite double is an exact
//    integer m 2^e, so its residue is (m mod q)(2^e mod q) mod q -- exact for
//    every magnitude, like Python's int(c) % q.
//  * crt_compose (ref rns.py:93-115) + centring (ckks.py:207-213 _centered)
//    + float(c) (ckks.py:203-205 _decode_ints): residue rows -> the centred
//    integer in (-Q/2, Q/2] as multi-word two's complement (optional) and as
//    the correctly rounded float64 (round half to even, as Python's
//    float(int); +-inf where Python raises OverflowError).
//    Per coefficient: t_i = r_i y_i mod q_i (y_i = (Q/q_i)^-1 mod q_i),
//    acc = sum_i t_i M_i with M_i = Q/q_i in W 32-bit words (acc < L Q),
//    k = floor(sum_i t_i / q_i) (= floor(acc / Q) up to one, fixed by a
//    compare), v = acc - k Q, centred against (Q - 1) / 2 (Q is odd), then
//    the top 64 bits (+ sticky) rounded once.
// Both are one thread per coefficient; the multi-word arithmetic is fully
// unrolled over a compile-time word bound (registers, no local memory).
#include <cmath>
#include <string>
#include <vector>

#include "common.cuh"
#include "poly_ops.h"
#include "tfhe_internal.h"

namespace tfhe {

namespace {

TFHE_DEV uint32_t pow2_mod(uint32_t e, uint32_t q, uint64_t mu) {
  uint32_t r = 1 % q, x = 2 % q;
  while (e) {
    if (e & 1) r = mul_mod(r, x, q, mu);
    x = mul_mod(x, x, q, mu);
    e >>= 1;
  }
  return r;
}

// residue of the (already integral) magnitude |d| of a finite double
TFHE_DEV uint32_t f64_mag_mod(double ad, uint32_t q, uint64_t mu) {
  if (ad < 18446744073709551616.0) return reduce64((uint64_t)ad, q, mu);
  const uint64_t bits = (uint64_t)__double_as_longlong(ad);
  const uint32_t e = (uint32_t)((bits >> 52) & 0x7ff) - 1075u;   // >= 12 here
  const uint64_t m = (bits & ((1ull << 52) - 1)) | (1ull << 52);
  return mul_mod(reduce64(m, q, mu), pow2_mod(e, q, mu), q, mu);
}

__global__ void __launch_bounds__(256)
    crt_decompose_kernel(const void* __restrict__ in, int kind, int64_t n,
                         const PrimeConst* __restrict__ pcs, CrtRows rows,
                         uint32_t* __restrict__ out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    bool neg;
    uint64_t a = 0;
    double ad = 0.0;
    if (kind == 0) {
      const int64_t c = static_cast<const int64_t*>(in)[j];
      neg = c < 0;
      a = neg ? 0ull - (uint64_t)c : (uint64_t)c;
    } else {
      const double d = rint(static_cast<const double*>(in)[j]);   // np.rint: half to even
      neg = d < 0.0;
      ad = fabs(d);
    }
    for (int l = 0; l < rows.n; ++l) {
      const PrimeConst pc = pcs[rows.prime[l]];
      const uint32_t r = kind == 0 ? reduce64(a, pc.q, pc.mu) : f64_mag_mod(ad, pc.q, pc.mu);
      out[(int64_t)l * n + j] = neg && r ? pc.q - r : r;
    }
  }
}

// constants (words): Q[W] | half[W] = (Q-1)/2 | M_0[W] .. M_{L-1}[W] | y[L]
template <int WM>
__global__ void __launch_bounds__(128)
    crt_compose_kernel(const uint32_t* __restrict__ rows, int64_t n, const uint32_t* __restrict__ cst,
                       int W, const PrimeConst* __restrict__ pcs, CrtRows lr,
                       double* __restrict__ out_f, uint32_t* __restrict__ out_w, int n_words) {
  const int L = lr.n;
  const uint32_t* Q = cst;
  const uint32_t* H = cst + W;
  const uint32_t* Mw = cst + 2 * W;   // M_i = Q / q_i
  const uint32_t* Y = cst + (2 + L) * W;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    uint32_t acc[WM + 1];
#pragma unroll
    for (int w = 0; w <= WM; ++w) acc[w] = 0;
    double kf = 0.0;
    for (int i = 0; i < L; ++i) {
      const PrimeConst pc = pcs[lr.prime[i]];
      const uint32_t r = mul_mod(rows[(int64_t)i * n + j], Y[i], pc.q, pc.mu);
      const uint32_t* Mi = Mw + (size_t)i * W;
      uint64_t carry = 0;
#pragma unroll
      for (int w = 0; w < WM; ++w) {
        if (w < W) {
          const uint64_t t = (uint64_t)r * Mi[w] + acc[w] + carry;
          acc[w] = (uint32_t)t;
          carry = t >> 32;
        }
      }
#pragma unroll
      for (int w = 1; w <= WM; ++w)   // the top word (index W) takes the carry
        if (w == W) acc[w] += (uint32_t)carry;
      kf += (double)r / (double)pc.q;
    }
    // v = acc - k Q with k = floor(acc / Q) up to one; sign word = acc[W]
    const uint32_t k = (uint32_t)floor(kf);
    {
      int64_t borrow = 0;
      uint64_t carry = 0;
#pragma unroll
      for (int w = 0; w <= WM; ++w) {
        if (w <= W) {
          const uint64_t kq = (uint64_t)k * (w < W ? Q[w] : 0u) + carry;
          carry = kq >> 32;
          const int64_t t = (int64_t)acc[w] - (int64_t)(uint32_t)kq - borrow;
          acc[w] = (uint32_t)t;
          borrow = t < 0;
        }
      }
    }
    // correction: v < 0 -> v += Q ; v >= Q -> v -= Q
    uint32_t top = 0;
#pragma unroll
    for (int w = 0; w <= WM; ++w)
      if (w == W) top = acc[w];
    if ((int32_t)top < 0) {
      uint64_t c = 0;
#pragma unroll
      for (int w = 0; w <= WM; ++w)
        if (w <= W) {
          const uint64_t t = (uint64_t)acc[w] + (w < W ? Q[w] : 0u) + c;
          acc[w] = (uint32_t)t;
          c = t >> 32;
        }
    } else {
      // v >= Q ?  (top word 0 here unless v >= 2^(32 W) > Q)
      int cmp = top != 0 ? 1 : 0;
#pragma unroll
      for (int w = WM - 1; w >= 0; --w)
        if (w < W && cmp == 0) cmp = acc[w] > Q[w] ? 1 : (acc[w] < Q[w] ? -1 : 0);
      if (cmp >= 0) {
        int64_t b = 0;
#pragma unroll
        for (int w = 0; w <= WM; ++w)
          if (w <= W) {
            const int64_t t = (int64_t)acc[w] - (w < W ? (int64_t)Q[w] : 0) - b;
            acc[w] = (uint32_t)t;
            b = t < 0;
          }
      }
    }
    // centre: v > (Q - 1) / 2  ->  v - Q (magnitude Q - v)
    int cmp = 0;
#pragma unroll
    for (int w = WM - 1; w >= 0; --w)
      if (w < W && cmp == 0) cmp = acc[w] > H[w] ? 1 : (acc[w] < H[w] ? -1 : 0);
    const bool neg = cmp > 0;
    uint32_t mag[WM];
    {
      int64_t b = 0;
#pragma unroll
      for (int w = 0; w < WM; ++w) {
        if (w < W) {
          if (neg) {
            const int64_t t = (int64_t)Q[w] - acc[w] - b;
            mag[w] = (uint32_t)t;
            b = t < 0;
          } else {
            mag[w] = acc[w];
          }
        } else {
          mag[w] = 0;
        }
      }
    }
    // float64, round half to even (Python float(int))
    int msw = -1;
    uint32_t mtop = 0;
#pragma unroll
    for (int w = 0; w < WM; ++w)
      if (mag[w] != 0) {
        msw = w;
        mtop = mag[w];
      }
    double f = 0.0;
    if (msw >= 0) {
      const int bitpos = 32 * msw + 31 - __clz(mtop);
      if (bitpos < 64) {
        const uint64_t v = (uint64_t)mag[0] | ((WM > 1 ? (uint64_t)mag[1] : 0ull) << 32);
        f = __ull2double_rn(v);
      } else {
        // 64 bits from bitpos - 63 upwards, sticky = any bit below them
        const int lo = bitpos - 63, lw = lo >> 5, ls = lo & 31;
        uint64_t hi64 = 0;
        bool sticky = false;
#pragma unroll
        for (int w = 0; w < WM; ++w) {
          const uint64_t m = mag[w];
          if (w == lw) {
            hi64 |= m >> ls;
            sticky |= ls && (m & ((1u << ls) - 1u));
          } else if (w == lw + 1) {
            hi64 |= ls ? m << (32 - ls) : m << 32;
          } else if (w == lw + 2 && ls) {
            hi64 |= m << (64 - ls);
          } else if (w < lw) {
            sticky |= m != 0;
          }
        }
        f = ldexp(__ull2double_rn(hi64 | (sticky ? 1ull : 0ull)), lo);
      }
    }
    if (out_f) out_f[j] = neg ? -f : f;
    if (out_w) {
      // two's complement of the centred value, n_words words, sign-extended
      uint64_t c = 1;
#pragma unroll
      for (int w = 0; w < WM; ++w) {
        if (w < n_words) {
          uint32_t m = w < W ? mag[w] : 0u;
          if (neg) {
            const uint64_t t = (uint64_t)(~m) + c;
            m = (uint32_t)t;
            c = t >> 32;
          }
          out_w[(int64_t)w * n + j] = m;
        }
      }
      for (int w = WM; w < n_words; ++w) out_w[(int64_t)w * n + j] = neg ? 0xffffffffu : 0u;
    }
  }
}

// ---- host multi-word helpers (little-endian 32-bit words) ----
void mw_mul_small(std::vector<uint32_t>& a, uint32_t m) {
  uint64_t c = 0;
  for (auto& w : a) {
    const uint64_t t = (uint64_t)w * m + c;
    w = (uint32_t)t;
    c = t >> 32;
  }
  if (c) a.push_back((uint32_t)c);
}
uint32_t mw_div_small(std::vector<uint32_t>& a, uint32_t d) {   // a /= d, returns a % d
  uint64_t r = 0;
  for (size_t i = a.size(); i-- > 0;) {
    const uint64_t cur = (r << 32) | a[i];
    a[i] = (uint32_t)(cur / d);
    r = cur % d;
  }
  while (a.size() > 1 && a.back() == 0) a.pop_back();
  return (uint32_t)r;
}
uint32_t inv_mod(uint64_t a, uint32_t q) {
  uint64_t r = 1, x = a % q, e = q - 2;
  while (e) {
    if (e & 1) r = r * x % q;
    x = x * x % q;
    e >>= 1;
  }
  return (uint32_t)r;
}

}  // namespace

int crt_compose_words(const Ctx& c, const int16_t* prime_ids, int L) {
  std::vector<uint32_t> Q(1, 1);
  for (int i = 0; i < L; ++i) mw_mul_small(Q, c.primes[prime_ids[i]]);
  return (int)Q.size();
}

int crt_compose_constants(const Ctx& c, const int16_t* prime_ids, int L, std::vector<uint32_t>& out) {
  std::vector<uint32_t> Q(1, 1);
  for (int i = 0; i < L; ++i) mw_mul_small(Q, c.primes[prime_ids[i]]);
  const int W = (int)Q.size();
  out.assign((size_t)(2 + L) * W + L, 0);
  for (int w = 0; w < W; ++w) out[w] = Q[w];
  std::vector<uint32_t> H = Q;            // (Q - 1) / 2: Q is odd
  mw_div_small(H, 2);
  for (int w = 0; w < (int)H.size(); ++w) out[W + w] = H[w];
  for (int i = 0; i < L; ++i) {
    const uint32_t qi = c.primes[prime_ids[i]];
    std::vector<uint32_t> M = Q;          // Q / q_i
    mw_div_small(M, qi);
    std::vector<uint32_t> Mm = M;         // (Q / q_i) mod q_i
    const uint32_t mmod = mw_div_small(Mm, qi);
    const uint32_t y = inv_mod(mmod, qi);
    for (int w = 0; w < (int)M.size() && w < W; ++w) out[(size_t)(2 + i) * W + w] = M[w];
    out[(size_t)(2 + L) * W + i] = y;
  }
  return W;
}

int launch_crt_decompose(const Ctx& c, const void* in, int kind, int64_t n, const CrtRows& rows,
                         uint32_t* out, cudaStream_t st) {
  if (n <= 0 || rows.n <= 0) return 0;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)c.sms * 8);
  crt_decompose_kernel<<<(int)blocks, 256, 0, st>>>(in, kind, n, c.d_pc, rows, out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("crt_decompose launch: ") + cudaGetErrorString(e));
    return 3;
  }
  return 0;
}

int launch_crt_compose(const Ctx& c, const uint32_t* rows, int64_t n, const uint32_t* d_cst, int W,
                       const CrtRows& lr, double* out_f, uint32_t* out_w, int n_words,
                       cudaStream_t st) {
  if (n <= 0) return 0;
  const int64_t blocks = std::min<int64_t>((n + 127) / 128, (int64_t)c.sms * 16);
  if (W <= 4)
    crt_compose_kernel<4><<<(int)blocks, 128, 0, st>>>(rows, n, d_cst, W, c.d_pc, lr, out_f,
                                                        out_w, n_words);
  else if (W <= 16)
    crt_compose_kernel<16><<<(int)blocks, 128, 0, st>>>(rows, n, d_cst, W, c.d_pc, lr, out_f,
                                                         out_w, n_words);
  else if (W <= 64)
    crt_compose_kernel<64><<<(int)blocks, 128, 0, st>>>(rows, n, d_cst, W, c.d_pc, lr, out_f,
                                                         out_w, n_words);
  else {
    set_error("crt_compose: modulus wider than 2048 bits");
    return 2;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("crt_compose launch: ") + cudaGetErrorString(e));
    return 3;
  }
  return 0;
}

}  // namespace tfhe
