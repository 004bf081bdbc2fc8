// HBM-bound element-wise and automorphism kernels (base conversion lives in
// bconv_tc.cu).
//
// All operate on level-major buffers (rows, batch, n) of canonical u32
// residues, one prime per row (reference layout, batch.py:22-47).  Row r of a
// launch uses prime `row_prime[r]`; the prime table lives in the context.
//
//   ele_add / ele_sub / hada_mult / negate / scalar_rows_mult  kernels.py:33-67
//   tensor product (hmult's d0, d1, d2)                       ckks.py:265-271
//   key-switch inner product acc += raised * key              ckks.py:345-351
//   NTT-domain automorphism gather / coeff-domain signed scatter kernels.py:77-107
//
// Each thread moves 16-byte vectors (uint4) with a grid-stride loop; grids
// are sized as a multiple of the SM count.
#include <cstring>

#include "common.cuh"
#include "poly_ops.h"

namespace tfhe {

namespace {

struct RowPrimes {
  int16_t prime[kMaxRows];
};

TFHE_DEV uint4 ld4(const uint32_t* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }
TFHE_DEV void st4(uint32_t* p, uint4 v) { *reinterpret_cast<uint4*>(p) = v; }

template <int OP>
TFHE_DEV uint32_t binop(uint32_t x, uint32_t y, const PrimeConst& pc) {
  if (OP == OP_ADD) return add_mod(x, y, pc.q);
  if (OP == OP_SUB) return sub_mod(x, y, pc.q);
  return mul_mod(x, y, pc.q, pc.mu);
}

// out = a (op) b, row-wise primes; per_row elements per row (multiple of 4)
template <int OP>
__global__ void binary_kernel(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                              uint32_t* __restrict__ out, const PrimeConst* __restrict__ pcs,
                              const __grid_constant__ RowPrimes rp, int64_t per_row) {
  const int row = blockIdx.y;
  const PrimeConst pc = pcs[rp.prime[row]];
  const int64_t base = (int64_t)row * per_row;
  // two 4-element groups per iteration, loads first (memory-level parallelism)
  const int64_t step = (int64_t)gridDim.x * blockDim.x * 4;
  for (int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4; i0 < per_row;
       i0 += 2 * step) {
    uint4 x[2], y[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t i = i0 + h * step < per_row ? i0 + h * step : i0;
      x[h] = ld4(a + base + i);
      y[h] = ld4(b + base + i);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t i = i0 + h * step;
      if (i >= per_row) break;
      uint4 r;
      r.x = binop<OP>(x[h].x, y[h].x, pc);
      r.y = binop<OP>(x[h].y, y[h].y, pc);
      r.z = binop<OP>(x[h].z, y[h].z, pc);
      r.w = binop<OP>(x[h].w, y[h].w, pc);
      st4(out + base + i, r);
    }
  }
}

struct ScalarArgs {
  int16_t prime[kMaxRows];
  uint32_t s[kMaxRows], s_shoup[kMaxRows];
};

// out = a * s_row (OP_SCALAR) or q - a (OP_NEG)
template <int OP>
__global__ void unary_kernel(const uint32_t* __restrict__ a, uint32_t* __restrict__ out,
                             const PrimeConst* __restrict__ pcs,
                             const __grid_constant__ ScalarArgs sa, int64_t per_row) {
  const int row = blockIdx.y;
  const uint32_t q = pcs[sa.prime[row]].q;
  const uint32_t s = sa.s[row], sp = sa.s_shoup[row];
  const int64_t base = (int64_t)row * per_row;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4; i < per_row;
       i += (int64_t)gridDim.x * blockDim.x * 4) {
    uint4 x = ld4(a + base + i), r;
    if (OP == OP_NEG) {
      r.x = x.x ? q - x.x : 0;
      r.y = x.y ? q - x.y : 0;
      r.z = x.z ? q - x.z : 0;
      r.w = x.w ? q - x.w : 0;
    } else {
      r.x = mul_shoup(x.x, s, sp, q);
      r.y = mul_shoup(x.y, s, sp, q);
      r.z = mul_shoup(x.z, s, sp, q);
      r.w = mul_shoup(x.w, s, sp, q);
    }
    st4(out + base + i, r);
  }
}

// hmult tensor product: d0 = b0 b1, d1 = a0 b1 + a1 b0, d2 = a0 a1
__global__ void tensor_kernel(const uint32_t* __restrict__ b0, const uint32_t* __restrict__ a0,
                              const uint32_t* __restrict__ b1, const uint32_t* __restrict__ a1,
                              uint32_t* __restrict__ d0, uint32_t* __restrict__ d1,
                              uint32_t* __restrict__ d2, const PrimeConst* __restrict__ pcs,
                              const __grid_constant__ RowPrimes rp, int64_t per_row,
                              const __grid_constant__ TensorMac mac) {
  const int row = blockIdx.y;
  const PrimeConst pc = pcs[rp.prime[row]];
  const int64_t base = (int64_t)row * per_row;
  // two 4-element groups per iteration, loads first (memory-level parallelism)
  const int64_t step = (int64_t)gridDim.x * blockDim.x * 4;
  for (int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4; i0 < per_row;
       i0 += 2 * step) {
    uint4 xb0[2], xa0[2], xb1[2], xa1[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t o = base + (i0 + h * step < per_row ? i0 + h * step : i0);
      xb0[h] = ld4(b0 + o);
      xa0[h] = ld4(a0 + o);
      xb1[h] = ld4(b1 + o);
      xa1[h] = ld4(a1 + o);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (i0 + h * step >= per_row) break;
      const int64_t o = base + i0 + h * step;
      uint4 r0, r1, r2;
      // d1's two products (< 2^62 each) are summed before one reduction
#define TFHE_TP(c)                                                                          \
  r0.c = mul_mod(xb0[h].c, xb1[h].c, pc.q, pc.mu);                                          \
  r1.c = reduce64((uint64_t)xa0[h].c * xb1[h].c + (uint64_t)xa1[h].c * xb0[h].c, pc.q, pc.mu); \
  r2.c = mul_mod(xa0[h].c, xa1[h].c, pc.q, pc.mu);
      TFHE_TP(x) TFHE_TP(y) TFHE_TP(z) TFHE_TP(w)
#undef TFHE_TP
      st4(d0 + o, r0);
      st4(d1 + o, r1);
      st4(d2 + o, r2);
      if (row < mac.rows) {
        // the key switch's slice-row MAC on d2 (ckks.py:361-364, keys broadcast
        // over the batch): acc_b = d2 kb, acc_a = d2 ka, overwriting
        const int coef = (int)((i0 + h * step) & ((1 << mac.log_n) - 1));
        const uint4 wb = ld4(mac.kb + mac.key_off[row] + coef);
        const uint4 wa = ld4(mac.ka + mac.key_off[row] + coef);
        uint4 ob, oa;
#define TFHE_TM(c)                          \
  ob.c = mul_mod(r2.c, wb.c, pc.q, pc.mu);  \
  oa.c = mul_mod(r2.c, wa.c, pc.q, pc.mu);
        TFHE_TM(x) TFHE_TM(y) TFHE_TM(z) TFHE_TM(w)
#undef TFHE_TM
        st4(mac.acc_b + o, ob);
        st4(mac.acc_a + o, oa);
      }
    }
  }
}

struct MacArgs {
  int16_t prime[kMaxRows];
  int64_t key_off[kMaxRows];  // element offset of this row's key row (from kb / ka)
  uint32_t pmod[kMaxRows], pmod_shoup[kMaxRows];   // ks_mac_rot: P mod q_r
};

// acc_b[r] (+)= x[r] * kb[key_row[r]], acc_a[r] (+)= x[r] * ka[key_row[r]];
// keys are (rows, n) and broadcast over the batch.  first != 0 overwrites.
__global__ void ks_mac_kernel(const uint32_t* __restrict__ x, const uint32_t* __restrict__ kb,
                              const uint32_t* __restrict__ ka, uint32_t* __restrict__ acc_b,
                              uint32_t* __restrict__ acc_a, const PrimeConst* __restrict__ pcs,
                              const __grid_constant__ MacArgs ma, int batch, int n, int first) {
  const int row = blockIdx.y;
  const PrimeConst pc = pcs[ma.prime[row]];
  const int64_t per_row = (int64_t)batch * n;
  const int64_t base = (int64_t)row * per_row;
  const uint32_t* kbr = kb + ma.key_off[row];
  const uint32_t* kar = ka + ma.key_off[row];
  // two 4-coefficient groups per iteration, all loads issued before the
  // arithmetic (memory-level parallelism)
  const int64_t step = (int64_t)gridDim.x * blockDim.x * 4;
  for (int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4; i0 < per_row;
       i0 += 2 * step) {
    uint4 v[2], wb[2], wa[2], ob[2], oa[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t i = i0 + h * step;
      const bool ok = i < per_row;
      const int64_t o = base + (ok ? i : 0);
      const int coef = (int)(i & (n - 1));   // n is a power of two
      v[h] = ld4(x + o);
      wb[h] = ld4(kbr + coef);
      wa[h] = ld4(kar + coef);
      ob[h] = first ? make_uint4(0, 0, 0, 0) : ld4(acc_b + o);
      oa[h] = first ? make_uint4(0, 0, 0, 0) : ld4(acc_a + o);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t i = i0 + h * step;
      if (i >= per_row) break;
      const int64_t o = base + i;
#define TFHE_MAC(c)                                                           \
  ob[h].c = add_mod(ob[h].c, mul_mod(v[h].c, wb[h].c, pc.q, pc.mu), pc.q);    \
  oa[h].c = add_mod(oa[h].c, mul_mod(v[h].c, wa[h].c, pc.q, pc.mu), pc.q);
      TFHE_MAC(x) TFHE_MAC(y) TFHE_MAC(z) TFHE_MAC(w)
#undef TFHE_MAC
      st4(acc_b + o, ob[h]);
      st4(acc_a + o, oa[h]);
    }
  }
}

// Hoisted HROTATE (ckks.py:276-282): the slice-row MAC of the key switch and
// the addend phi(b) in one pass, phi never materialised:
//   acc_b[r] = phi(x)[r] * kb[key_row[r]] + P_r * phi(base)[r]
//   acc_a[r] = phi(x)[r] * ka[key_row[r]]
// with phi(v)[k] = v[((t (2k+1) mod 2n) - 1) / 2] (kernels.py:77-85) and P_r
// the product of the specials mod q_r, so that ModDown's (acc_b - y) P^-1 is
// phi(b) + ksb bit for bit.  perm_x = 0: x already holds phi(x).
__global__ void ks_mac_rot_kernel(const uint32_t* __restrict__ x, const uint32_t* __restrict__ base,
                                  const uint32_t* __restrict__ kb, const uint32_t* __restrict__ ka,
                                  uint32_t* __restrict__ acc_b, uint32_t* __restrict__ acc_a,
                                  const PrimeConst* __restrict__ pcs,
                                  const __grid_constant__ MacArgs ma, int batch, int log_n,
                                  uint32_t t, int perm_x) {
  const int row = blockIdx.y;
  const PrimeConst pc = pcs[ma.prime[row]];
  const int n = 1 << log_n;
  const int64_t per_row = (int64_t)batch * n;
  const int64_t rbase = (int64_t)row * per_row;
  const uint32_t* kbr = kb + ma.key_off[row];
  const uint32_t* kar = ka + ma.key_off[row];
  const uint32_t pm = ma.pmod[row], pms = ma.pmod_shoup[row];
  const uint32_t mask = (uint32_t)n - 1, half = (t - 1) >> 1;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4; i < per_row;
       i += (int64_t)gridDim.x * blockDim.x * 4) {
    const int64_t o = rbase + i;
    const int coef = (int)(i & mask);
    const int64_t mrow = o - coef;   // this member's row start
    uint32_t src[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) src[e] = (t * (uint32_t)(coef + e) + half) & mask;
    const uint4 wb = ld4(kbr + coef), wa = ld4(kar + coef);
    uint4 v, bv;
    if (perm_x) {
      v = make_uint4(__ldg(x + mrow + src[0]), __ldg(x + mrow + src[1]), __ldg(x + mrow + src[2]),
                     __ldg(x + mrow + src[3]));
    } else {
      v = ld4(x + o);
    }
    bv = make_uint4(__ldg(base + mrow + src[0]), __ldg(base + mrow + src[1]),
                    __ldg(base + mrow + src[2]), __ldg(base + mrow + src[3]));
    uint4 ob, oa;
#define TFHE_MACR(c)                                                               \
  ob.c = add_mod(mul_mod(v.c, wb.c, pc.q, pc.mu), mul_shoup(bv.c, pm, pms, pc.q), pc.q); \
  oa.c = mul_mod(v.c, wa.c, pc.q, pc.mu);
    TFHE_MACR(x) TFHE_MACR(y) TFHE_MACR(z) TFHE_MACR(w)
#undef TFHE_MACR
    st4(acc_b + o, ob);
    st4(acc_a + o, oa);
  }
}

// fused ModDown + rescale preparation (poly_ops.h: MdRsArgs)
__global__ void md_rescale_prep_kernel(uint32_t* __restrict__ acc, const uint32_t* __restrict__ base,
                                       const uint32_t* conv, const uint32_t* __restrict__ t,
                                       uint32_t* w, const PrimeConst* __restrict__ pcs,
                                       const __grid_constant__ MdRsArgs ar, int64_t per_row) {
  const int row = blockIdx.y;
  const PrimeConst pc = pcs[ar.prime[row]];
  const uint32_t pi = ar.pinv[row], pis = ar.pinv_shoup[row];
  uint32_t* xr = acc + ar.acc_row[row] * per_row;
  const uint32_t* br = ar.base_row[row] >= 0 ? base + ar.base_row[row] * per_row : nullptr;
  const uint32_t* cr = conv + ar.conv_row[row] * per_row;
  const uint32_t* tr = t + ar.t_row[row] * per_row;
  uint32_t* wr = w + ar.w_row[row] * per_row;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4; i < per_row;
       i += (int64_t)gridDim.x * blockDim.x * 4) {
    uint4 x = ld4(xr + i), cv = ld4(cr + i), tv = ld4(tr + i);
    uint4 b = br ? ld4(br + i) : make_uint4(0, 0, 0, 0);
    uint4 wv;
#define TFHE_MDRS(c)                                                                   \
  x.c = add_mod(mul_shoup(x.c, pi, pis, pc.q), b.c, pc.q);                             \
  wv.c = add_mod(mul_shoup(cv.c, pi, pis, pc.q), reduce64(tv.c, pc.q, pc.mu), pc.q);
    TFHE_MDRS(x) TFHE_MDRS(y) TFHE_MDRS(z) TFHE_MDRS(w)
#undef TFHE_MDRS
    st4(xr + i, x);
    st4(wr + i, wv);
  }
}

// NTT domain: out[k] = in[((t (2k+1) mod 2n) - 1) / 2]   (kernels.py:77-96)
__global__ void automorph_ntt_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                     uint32_t t, int log_n, int64_t rows) {
  const uint32_t n = 1u << log_n, mask2n = 2 * n - 1;
  const int64_t total = rows << log_n;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4; i < total;
       i += (int64_t)gridDim.x * blockDim.x * 4) {
    const int64_t rbase = i & ~(int64_t)(n - 1);
    const uint32_t k = (uint32_t)(i & (n - 1));
    uint4 r;
    r.x = __ldg(in + rbase + (((t * (2 * k + 1)) & mask2n) >> 1));
    r.y = __ldg(in + rbase + (((t * (2 * k + 3)) & mask2n) >> 1));
    r.z = __ldg(in + rbase + (((t * (2 * k + 5)) & mask2n) >> 1));
    r.w = __ldg(in + rbase + (((t * (2 * k + 7)) & mask2n) >> 1));
    st4(out + i, r);
  }
}

// NTT domain, small multiplier (t mod n <= kAutSmallT, e.g. rotation by 1:
// t = 5): out[k] = in[(t k + c) mod n], c = (t - 1) / 2.  A source window
// [j0, j0 + W) of one polynomial row feeds at most t + 1 runs of consecutive
// outputs, k in [(j0 - c + m n) / t, (j0 + W - c + m n) / t) for m <= t, so the
// block stages the window in shared memory (coalesced 16-byte loads) and
// writes the t runs with coalesced stores -- instead of the stride-t gather,
// whose partially used sectors cost ~50% extra DRAM reads.
constexpr int kAutWin = 4096;
constexpr uint32_t kAutSmallT = 64;
__global__ void __launch_bounds__(256)
    automorph_ntt_window_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                uint32_t t, int log_n) {
  __shared__ __align__(16) uint32_t win[kAutWin];
  const uint32_t n = 1u << log_n, mask = n - 1;
  const uint32_t tt = t & mask;                       // multiplier of k (mod n)
  const uint32_t c = ((t - 1) >> 1) & mask;           // (t(2k+1) mod 2n - 1) / 2 = t k + c mod n
  const int wins = (int)(n / kAutWin);
  const int64_t row = blockIdx.x / wins;
  const uint32_t j0 = (uint32_t)(blockIdx.x % wins) * kAutWin;
  const uint32_t* src = in + (row << log_n) + j0;
  for (int i = threadIdx.x * 4; i < kAutWin; i += blockDim.x * 4)
    *reinterpret_cast<uint4*>(win + i) = __ldg(reinterpret_cast<const uint4*>(src + i));
  __syncthreads();
  uint32_t* dst = out + (row << log_n);
  for (uint32_t m = 0; m <= tt; ++m) {   // t k + c < (tt + 1) n
    // k range of run m: t k + c - m n in [j0, j0 + W)
    const int64_t base = (int64_t)m * n - c;
    const int64_t lo = (int64_t)j0 + base, hi = lo + kAutWin;
    const int64_t k_lo = lo <= 0 ? 0 : (lo + tt - 1) / tt;
    const int64_t k_hi = min((int64_t)n, (hi + tt - 1) / tt);
    for (int64_t k = k_lo + threadIdx.x; k < k_hi; k += blockDim.x)
      dst[k] = win[(uint32_t)(tt * k - base) - j0];
  }
}

// coefficient domain: x^i -> +-x^{t i mod n}  (kernels.py:97-107)
__global__ void automorph_coeff_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                       const PrimeConst* __restrict__ pcs,
                                       const __grid_constant__ RowPrimes rp, uint32_t t, int log_n,
                                       int batch) {
  const uint32_t n = 1u << log_n;
  const int row = blockIdx.y;
  const uint32_t q = pcs[rp.prime[row]].q;
  const int64_t per_row = (int64_t)batch << log_n;
  const int64_t base = (int64_t)row * per_row;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < per_row;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pbase = base + (i & ~(int64_t)(n - 1));
    const uint32_t c = (uint32_t)(i & (n - 1));
    const uint32_t e = (uint32_t)(((uint64_t)t * c) & (2 * n - 1));
    uint32_t v = __ldg(in + base + i);
    if (e >= n) v = v ? q - v : 0;
    out[pbase + (e & (n - 1))] = v;
  }
}

int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

dim3 grid_rows(int64_t per_row, int rows, int threads) {
  // enough blocks per row to cover it with 4-wide threads, capped so the
  // whole grid is a few waves of the SM count
  int64_t need = (per_row / 4 + threads - 1) / threads;
  int64_t cap = std::max<int64_t>(1, (int64_t)sm_count() * 8 / std::max(rows, 1));
  return dim3((unsigned)std::max<int64_t>(1, std::min(need, cap)), rows);
}

int check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return 3;
  }
  return 0;
}

}  // namespace

int launch_binary(const Ctx& c, int op, const uint32_t* a, const uint32_t* b, uint32_t* out,
                  const int16_t* row_prime, int rows, int64_t per_row, cudaStream_t st) {
  if (rows <= 0 || per_row <= 0) return 0;
  RowPrimes rp;
  memcpy(rp.prime, row_prime, sizeof(int16_t) * rows);
  dim3 g = grid_rows(per_row, rows, 256);
  switch (op) {
    case OP_ADD: binary_kernel<OP_ADD><<<g, 256, 0, st>>>(a, b, out, c.d_pc, rp, per_row); break;
    case OP_SUB: binary_kernel<OP_SUB><<<g, 256, 0, st>>>(a, b, out, c.d_pc, rp, per_row); break;
    case OP_MUL: binary_kernel<OP_MUL><<<g, 256, 0, st>>>(a, b, out, c.d_pc, rp, per_row); break;
    default: set_error("bad binary op"); return 2;
  }
  return check("binary kernel");
}

int launch_unary(const Ctx& c, int op, const uint32_t* a, uint32_t* out, const int16_t* row_prime,
                 const uint32_t* scalars, int rows, int64_t per_row, cudaStream_t st) {
  if (rows <= 0 || per_row <= 0) return 0;
  ScalarArgs sa;
  for (int r = 0; r < rows; ++r) {
    sa.prime[r] = row_prime[r];
    const uint32_t q = c.h_pc[row_prime[r]].q;
    sa.s[r] = scalars ? scalars[r] % q : 0;
    sa.s_shoup[r] = (uint32_t)(((uint64_t)sa.s[r] << 32) / q);
  }
  dim3 g = grid_rows(per_row, rows, 256);
  if (op == OP_NEG) unary_kernel<OP_NEG><<<g, 256, 0, st>>>(a, out, c.d_pc, sa, per_row);
  else if (op == OP_SCALAR) unary_kernel<OP_SCALAR><<<g, 256, 0, st>>>(a, out, c.d_pc, sa, per_row);
  else { set_error("bad unary op"); return 2; }
  return check("unary kernel");
}

int launch_tensor(const Ctx& c, const uint32_t* b0, const uint32_t* a0, const uint32_t* b1,
                  const uint32_t* a1, uint32_t* d0, uint32_t* d1, uint32_t* d2,
                  const int16_t* row_prime, int rows, int64_t per_row, cudaStream_t st,
                  const TensorMac* mac) {
  if (rows <= 0 || per_row <= 0) return 0;
  RowPrimes rp;
  memcpy(rp.prime, row_prime, sizeof(int16_t) * rows);
  TensorMac none;
  memset(&none, 0, sizeof(none));
  dim3 g = grid_rows(per_row, rows, 256);
  tensor_kernel<<<g, 256, 0, st>>>(b0, a0, b1, a1, d0, d1, d2, c.d_pc, rp, per_row,
                                   mac ? *mac : none);
  return check("tensor kernel");
}

int launch_ks_mac(const Ctx& c, const uint32_t* x, const uint32_t* kb, const uint32_t* ka,
                  uint32_t* acc_b, uint32_t* acc_a, const int16_t* row_prime,
                  const int64_t* key_off, int rows, int batch, int first, cudaStream_t st) {
  if (rows <= 0) return 0;
  MacArgs ma;
  for (int r = 0; r < rows; ++r) {
    ma.prime[r] = row_prime[r];
    ma.key_off[r] = key_off[r];
  }
  dim3 g = grid_rows((int64_t)batch * c.n, rows, 256);
  ks_mac_kernel<<<g, 256, 0, st>>>(x, kb, ka, acc_b, acc_a, c.d_pc, ma, batch, c.n, first);
  return check("ks mac kernel");
}

int launch_ks_mac_rot(const Ctx& c, const uint32_t* x, const uint32_t* base, const uint32_t* kb,
                      const uint32_t* ka, uint32_t* acc_b, uint32_t* acc_a,
                      const int16_t* row_prime, const int64_t* key_off, const uint32_t* pmod,
                      int rows, int batch, uint32_t t, int perm_x, cudaStream_t st) {
  if (rows <= 0) return 0;
  if (rows > kMaxRows || (t & 1) == 0) {
    set_error("ks_mac_rot: too many rows or even galois element");
    return 2;
  }
  MacArgs ma;
  for (int r = 0; r < rows; ++r) {
    ma.prime[r] = row_prime[r];
    ma.key_off[r] = key_off[r];
    const uint32_t q = c.primes[row_prime[r]];
    ma.pmod[r] = pmod[r] % q;
    ma.pmod_shoup[r] = (uint32_t)(((uint64_t)ma.pmod[r] << 32) / q);
  }
  dim3 g = grid_rows((int64_t)batch * c.n, rows, 256);
  ks_mac_rot_kernel<<<g, 256, 0, st>>>(x, base, kb, ka, acc_b, acc_a, c.d_pc, ma, batch, c.log_n,
                                       t & (2u * c.n - 1), perm_x);
  return check("ks mac rot kernel");
}

int launch_md_rescale_prep(const Ctx& c, uint32_t* acc, const uint32_t* base, const uint32_t* conv,
                           const uint32_t* t, uint32_t* w, const MdRsArgs& ar, int rows,
                           int64_t per_row, cudaStream_t st) {
  if (rows <= 0) return 0;
  if (rows > kMaxRows || per_row % 4) {
    set_error("md_rescale_prep: too many rows or unaligned rows");
    return 2;
  }
  dim3 g = grid_rows(per_row, rows, 256);
  md_rescale_prep_kernel<<<g, 256, 0, st>>>(acc, base, conv, t, w, c.d_pc, ar, per_row);
  return check("md_rescale_prep kernel");
}

int launch_automorph(const Ctx& c, const uint32_t* in, uint32_t* out, uint32_t t, int ntt_domain,
                     const int16_t* row_prime, int rows, int batch, cudaStream_t st) {
  if (rows <= 0 || batch <= 0) return 0;
  t &= (uint32_t)(2 * c.n - 1);
  if (ntt_domain && c.n >= kAutWin && (t & (uint32_t)(c.n - 1)) <= kAutSmallT &&
      (t & (uint32_t)(c.n - 1)) >= 1) {
    const int64_t blocks = (int64_t)rows * batch * (c.n / kAutWin);
    automorph_ntt_window_kernel<<<(unsigned)blocks, 256, 0, st>>>(in, out, t, c.log_n);
  } else if (ntt_domain) {
    int64_t total = (int64_t)rows * batch * c.n;
    int64_t blocks = std::min<int64_t>((total / 4 + 255) / 256, (int64_t)sm_count() * 16);
    automorph_ntt_kernel<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, st>>>(
        in, out, t, c.log_n, (int64_t)rows * batch);
  } else {
    RowPrimes rp;
    memcpy(rp.prime, row_prime, sizeof(int16_t) * rows);
    dim3 g = grid_rows((int64_t)batch * c.n * 4, rows, 256);
    automorph_coeff_kernel<<<g, 256, 0, st>>>(in, out, c.d_pc, rp, t, c.log_n, batch);
  }
  return check("automorphism kernel");
}

}  // namespace tfhe
