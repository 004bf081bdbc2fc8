// C ABI (include/tfhe_b200.h): context lifetime, argument validation and the
// native orchestration of the CKKS operators (key switch = ModUp / inner
// product / ModDown, hmult, rescale, hrotate) on top of the kernels in
// ntt_tc.cu and poly_ops.cu.  Everything is stream-ordered; no host syncs.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/tfhe_b200.h"
#include "poly_ops.h"
#include "tfhe_internal.h"

struct TfheCtx {
  tfhe::Ctx c;
  int n_chain = 0, n_special = 0;
  // host-streaming transform (tfhe_ntt_host): copy streams + per-slot events,
  // created on first use
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev_start = nullptr, ev_in[3] = {}, ev_done[3] = {}, ev_out[3] = {};
  // pinned host bounce slots [in 3 | out 3] for pageable host buffers
  uint8_t* h_bounce = nullptr;
  size_t h_bounce_chunk = 0;
  // crt_compose constants per basis (device), built on first use
  std::vector<std::pair<std::vector<int16_t>, std::pair<uint32_t*, int>>> crt_cache;
  std::mutex crt_mu;
};

namespace tfhe {

thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

namespace {

uint32_t powmod(uint64_t b, uint64_t e, uint32_t q) {
  uint64_t r = 1 % q, x = b % q;
  while (e) {
    if (e & 1) r = r * x % q;
    x = x * x % q;
    e >>= 1;
  }
  return (uint32_t)r;
}
uint32_t invmod(uint64_t a, uint32_t q) { return powmod(a % q, q - 2, q); }
uint32_t shoup(uint32_t w, uint32_t q) { return (uint32_t)(((uint64_t)w << 32) / q); }
bool getenv_flag(const char* name) {
  const char* e = getenv(name);
  return e && *e && *e != '0';
}

// bump allocator over the caller's workspace
struct Carve {
  uint8_t* p;
  size_t left;
  bool ok = true;
  template <class T>
  T* take(size_t bytes) {
    size_t b = (bytes + 255) & ~(size_t)255;
    if (b > left) {
      ok = false;
      return nullptr;
    }
    T* r = reinterpret_cast<T*>(p);
    p += b;
    left -= b;
    return r;
  }
};

// Key-switch geometry.  Targets are the extended-basis rows a call produces:
// the local chain rows [r0, r0 + nr) then the K special rows (T = nr + K).
// The unpartitioned key switch has r0 = 0, nr = level + 1 (T = E); the
// limb-partitioned one gives each rank its own chain rows and
// every rank the specials.
struct CkksGeom {
  int Lc, K, alpha, l1, E;
  int r0, nr, T;
  bool need_conv;
  int nslices;   // non-empty GKS slices at this level
  int S;         // slices per fused key-switch group (TS path), 1 otherwise
};

CkksGeom geom(const TfheCtx* h, int level, int dnum, int r0 = 0, int nr = -1) {
  CkksGeom g;
  g.Lc = h->n_chain;
  g.K = h->n_special;
  g.alpha = dnum > 0 ? g.Lc / dnum : 1;
  g.l1 = level + 1;
  g.E = g.l1 + g.K;
  g.r0 = r0;
  g.nr = nr < 0 ? g.l1 : nr;
  g.T = g.nr + g.K;
  g.need_conv = g.alpha > 1 || g.K > 1;
  g.nslices = (g.l1 + g.alpha - 1) / g.alpha;
  g.S = 1;
  return g;
}

// slices per key-switch group: bounded by the launch limb map and by a cap on
// the (S * T, batch, n) stage-1 workspace (default 24 GiB of the 180 GB HBM,
// TFHE_KS_WS_GIB overrides): every group after the first re-reads and
// re-writes the (2, T, batch, n) accumulator, so fewer, larger groups save
// HBM traffic (P-Default at B = 128: S = 11, 5 groups, instead of S = 5, 9)
void set_group(CkksGeom& g, const Ctx& c, int batch) {
  if (!c.use_ts) {
    g.S = 1;
    return;
  }
  const size_t row_bytes = (size_t)batch * c.n * 4;
  static const size_t cap_gib = getenv("TFHE_KS_WS_GIB") ? (size_t)atoi(getenv("TFHE_KS_WS_GIB"))
                                                        : (size_t)24;
  const size_t cap = std::max<size_t>(cap_gib, 1) << 30;
  int s_mem = (int)std::max<size_t>(1, cap / (row_bytes * g.T));
  g.S = std::max(1, std::min({g.nslices, kMaxLimbs / g.T, s_mem}));
  // balanced groups: the same number of groups, no small trailing group
  // (45 slices at S <= 11: 5 x 9 rather than 4 x 11 + 1)
  {
    const int ng = (g.nslices + g.S - 1) / g.S;
    g.S = (g.nslices + ng - 1) / ng;
  }
  // test knob: TFHE_KS_MAX_S caps the group size so small goldens also run the
  // multi-group path (every group after the first re-reads the accumulator)
  if (const char* e = getenv("TFHE_KS_MAX_S")) {
    const int cap_s = atoi(e);
    if (cap_s > 0) g.S = std::min(g.S, cap_s);
  }
}

// prime index of target t (local chain rows, then specials)
inline int tprime(const CkksGeom& g, int t) { return t < g.nr ? g.r0 + t : g.Lc + (t - g.nr); }

int ks_ntt_rows(const CkksGeom& g) {
  return std::max({g.S * g.T, g.T, g.l1, 2 * g.nr, 2 * g.K});
}
int ks_conv_rows(const CkksGeom& g) { return std::max({g.S * g.T, g.T, 2 * g.nr}); }

size_t ks_bytes(const CkksGeom& g, int batch, int n) {
  const size_t U = (size_t)batch * n * 4;
  size_t rows = g.l1 /*y*/ + 2 * g.T /*acc*/ + ks_ntt_rows(g) /*ntt ws*/ + 2 * g.K /*ysp*/ +
                (g.need_conv ? ks_conv_rows(g) : 0);
  return rows * U + 16 * 256;
}

int fill_bconv(const Ctx& c, const std::vector<int>& src, const std::vector<int>& dst,
               BconvArgs& ba) {
  if ((int)src.size() > kMaxBconvSrc || (int)dst.size() > kMaxBconvDst) {
    set_error("base conversion too wide");
    return TFHE_EINVAL;
  }
  memset(&ba, 0, sizeof(ba));
  ba.n_src = (int)src.size();
  ba.n_dst = (int)dst.size();
  for (size_t s = 0; s < src.size(); ++s) {
    const uint32_t qs = c.primes[src[s]];
    uint64_t prod = 1;
    for (size_t o = 0; o < src.size(); ++o)
      if (o != s) prod = prod * (c.primes[src[o]] % qs) % qs;
    ba.src_prime[s] = (int16_t)src[s];
    ba.qhat_inv[s] = invmod(prod, qs);
    ba.qhat_inv_shoup[s] = shoup(ba.qhat_inv[s], qs);
  }
  for (size_t t = 0; t < dst.size(); ++t) {
    const uint32_t pt = c.primes[dst[t]];
    ba.dst_prime[t] = (int16_t)dst[t];
    ba.copy_from[t] = -1;
    for (size_t s = 0; s < src.size(); ++s)
      if (c.primes[src[s]] == pt) ba.copy_from[t] = (int16_t)s;
    for (size_t s = 0; s < src.size(); ++s) {
      uint64_t prod = 1;
      for (size_t o = 0; o < src.size(); ++o)
        if (o != s) prod = prod * (c.primes[src[o]] % pt) % pt;
      ba.factor[s * kMaxBconvDst + t] = (uint32_t)prod;
    }
  }
  return 0;
}

// ModDown fused with the rescale that follows it (tfhe_hmult_rescale).  With
// top = level, P = prod of the specials, conv_i the base-converted special
// rows (coefficient domain) and X_i = acc_i P^-1 + base_i:
//   ModDown_i  = X_i - NTT_i(conv_i) P^-1                     (ckks.py:367-381)
//   rescale_i  = (ModDown_i - NTT_i(T)) q_top^-1,  T = INTT_top(ModDown_top)
//                                                             (ckks.py:291-311)
//              = (X_i - NTT_i(conv_i P^-1 + T)) q_top^-1        (NTT_i is linear mod q_i)
// so one forward NTT per output row replaces ModDown's and the rescale's
// (2 level fewer limb-NTTs), bit-identical to rescale(hmult(.)).
int moddown_rescale(const Ctx& c, const CkksGeom& g, uint32_t* acc, const uint32_t* md_in,
                    uint32_t* wbuf, uint32_t* top, uint32_t* tcoef, const uint32_t* base,
                    const int16_t* base_rows, uint32_t* out, int batch, uint32_t* ntt_ws,
                    size_t ntt_ws_bytes, cudaStream_t st) {
  const int lv = g.l1 - 1;   // the prime rescale drops
  const int64_t U = (int64_t)batch * c.n;
  auto p_inv = [&](int i) {
    const uint32_t q = c.primes[i];
    uint64_t pm = 1;
    for (int k = 0; k < g.K; ++k) pm = pm * (c.primes[g.Lc + k] % q) % q;
    return invmod(pm, q);
  };
  auto md_row = [&](int cmp, int i) { return (int16_t)(g.K > 1 ? cmp * g.nr + i : cmp); };
  int rc;
  // 1. ModDown of the top row alone (as the unfused path computes it)
  LimbMap mt;
  EpiArgs et;
  memset(&et, 0, sizeof(et));
  et.mode = EPI_SUB_SCALE;
  et.x = acc;
  et.base = base;
  mt.n = 2;
  for (int cmp = 0; cmp < 2; ++cmp) {
    mt.prime[cmp] = (int16_t)lv;
    mt.in_row[cmp] = md_row(cmp, lv);
    mt.out_row[cmp] = (int16_t)cmp;
    et.x_row[cmp] = (int16_t)(cmp * g.T + lv);
    et.base_row[cmp] = base ? base_rows[cmp * g.nr + lv] : (int16_t)-1;
    et.s[cmp] = p_inv(lv);
    et.s_shoup[cmp] = shoup(et.s[cmp], c.primes[lv]);
  }
  if ((rc = launch_ntt(c, md_in, top, mt, batch, 0, &et, ntt_ws, ntt_ws_bytes, st))) return rc;
  // 2. T = INTT_top(top)
  LimbMap mi;
  mi.n = 2;
  for (int cmp = 0; cmp < 2; ++cmp) {
    mi.prime[cmp] = (int16_t)lv;
    mi.in_row[cmp] = mi.out_row[cmp] = (int16_t)cmp;
  }
  if ((rc = launch_ntt(c, top, tcoef, mi, batch, 1, nullptr, ntt_ws, ntt_ws_bytes, st))) return rc;
  if (lv == 0) return 0;
  // 3. X_i (in place in acc) and W_i = conv_i P^-1 + T mod q_i (row cmp * nr + i of wbuf,
  //    in place over conv_i when K > 1)
  MdRsArgs ar;
  LimbMap mr;
  EpiArgs er;
  memset(&er, 0, sizeof(er));
  er.mode = EPI_SUB_SCALE;
  er.x = acc;
  mr.n = 2 * lv;
  const uint32_t q_top = c.primes[lv];
  for (int cmp = 0; cmp < 2; ++cmp)
    for (int i = 0; i < lv; ++i) {
      const int l = cmp * lv + i;
      ar.prime[l] = (int16_t)i;
      ar.acc_row[l] = (int16_t)(cmp * g.T + i);
      ar.base_row[l] = base ? base_rows[cmp * g.nr + i] : (int16_t)-1;
      ar.conv_row[l] = md_row(cmp, i);
      ar.w_row[l] = (int16_t)(cmp * g.nr + i);
      ar.t_row[l] = (int16_t)cmp;
      ar.pinv[l] = p_inv(i);
      ar.pinv_shoup[l] = shoup(ar.pinv[l], c.primes[i]);
      // 4. out_i = (X_i - NTT_i(W_i)) q_top^-1
      mr.prime[l] = (int16_t)i;
      mr.in_row[l] = (int16_t)(cmp * g.nr + i);
      mr.out_row[l] = (int16_t)l;
      er.x_row[l] = (int16_t)(cmp * g.T + i);
      er.base_row[l] = -1;
      er.s[l] = invmod(q_top, c.primes[i]);
      er.s_shoup[l] = shoup(er.s[l], c.primes[i]);
    }
  if ((rc = launch_md_rescale_prep(c, acc, base, md_in, tcoef, wbuf, ar, 2 * lv, U, st))) return rc;
  return launch_ntt(c, wbuf, out, mr, batch, 0, &er, ntt_ws, ntt_ws_bytes, st);
}

// key switch of the local rows d (nr, B, n; chain rows [r0, r0+nr), NTT
// domain) -> out (2, nr, B, n) [+ add rows base_rows[]].  y_full is the
// coefficient-domain d over ALL level+1 chain rows (the all-gathered INTT of
// the limb-partitioned key switch); NULL = compute it here from d, which then
// must hold every chain row (r0 = 0, nr = level + 1).
//
// rs_scratch != NULL fuses the rescale that follows (tfhe_hmult_rescale): out is
// then (2, level, B, n) = rescale(ModDown(.)) bit for bit, and rs_scratch (>= 2
// rows, dead after ModUp) holds the top row's coefficient form.
//
// rot != NULL is the hoisted HROTATE (ckks.py:276-282): d is the
// UNrotated a (or phi(a) when rot->d_is_phi) and rot->b the unrotated b; phi_t
// is never materialised.  INTT(phi(a)) = phi_coeff(INTT(a)) is the INTT's own
// output scatter, the slice rows' MAC gathers phi(a) and folds P phi(b) into
// acc_b, so ModDown's (acc_b - y) P^-1 = phi(b) + ksb with no addend pass.
// HMULT's tensor product launched by keyswitch_impl itself, so that it can
// also write the slice-row MACs of d2 straight into the freshly carved
// accumulator (TensorMac) instead of a separate ks_mac pass over d2
struct TensorIn {
  const uint32_t* ct0;
  const uint32_t* ct1;
  uint32_t* dd;   // d0 | d1 | d2, P elements each
};

struct RotHoist {
  uint32_t t;
  const uint32_t* b;
  int d_is_phi;   // 1: d already holds phi(a) (planes without the output scatter)
};

int keyswitch_impl(TfheCtx* h, const uint32_t* d, const uint32_t* y_full, int level, int batch,
                   const uint32_t* key, int dnum, int r0, int nr, uint32_t* out,
                   const uint32_t* base, const int16_t* base_rows, Carve& cv, cudaStream_t st,
                   uint32_t* rs_scratch = nullptr, const RotHoist* rot = nullptr,
                   const TensorIn* tin = nullptr) {
  const Ctx& c = h->c;
  CkksGeom g = geom(h, level, dnum, r0, nr);
  set_group(g, c, batch);
  const size_t U = (size_t)batch * c.n;  // elements per limb row
  uint32_t* y = y_full ? nullptr : cv.take<uint32_t>(g.l1 * U * 4);
  uint32_t* acc = cv.take<uint32_t>(2 * g.T * U * 4);
  const size_t ntt_ws_bytes = ks_ntt_rows(g) * U * 4;
  uint32_t* ntt_ws = cv.take<uint32_t>(ntt_ws_bytes);
  uint32_t* ysp = cv.take<uint32_t>(2 * g.K * U * 4);
  // (the fused rescale builds its NTT input W in the conversion rows)
  uint32_t* conv =
      g.need_conv || rs_scratch ? cv.take<uint32_t>(ks_conv_rows(g) * U * 4) : nullptr;
  if (rs_scratch && (y_full || r0 != 0 || g.nr != g.l1 || level < 1)) {
    set_error("fused rescale needs the unpartitioned key switch at level >= 1");
    return TFHE_EINVAL;
  }
  if (!cv.ok) {
    set_error("ckks workspace too small");
    return TFHE_EINVAL;
  }
  const size_t key_pair = (size_t)2 * (g.Lc + g.K) * c.n;  // elements per (b_j, a_j)
  int rc;
  if (rot && (!c.use_ts || y_full || rs_scratch || base || (!rot->d_is_phi && !c.use_p3))) {
    set_error("hoisted rotation: unsupported key-switch configuration");
    return TFHE_EINVAL;
  }

  // 0. (HMULT) the tensor product, with the slice-row MACs of d2 fused: every
  //    row on the grouped path (they all start the accumulator), slice 0's
  //    rows on the per-slice path (its MACs overwrite; later slices add)
  int fused_rows = 0;
  if (tin) {
    if (r0 != 0 || g.nr != g.l1 || rot) {
      set_error("fused tensor product needs the unpartitioned, unrotated key switch");
      return TFHE_EINVAL;
    }
    TensorMac tm;
    memset(&tm, 0, sizeof(tm));
    tm.kb = key;
    tm.ka = key + key_pair / 2;
    tm.acc_b = acc;
    tm.acc_a = acc + g.T * U;
    tm.log_n = c.log_n;
    fused_rows = c.use_ts ? g.nr : std::min(g.alpha, g.l1);
    for (int r = 0; r < fused_rows; ++r)
      tm.key_off[r] = (int64_t)(r / g.alpha) * key_pair + (int64_t)r * c.n;
    tm.rows = fused_rows;
    int16_t rp[kMaxRows];
    for (int i = 0; i < g.l1; ++i) rp[i] = (int16_t)i;
    const size_t P = (size_t)g.l1 * U;
    if ((rc = launch_tensor(c, tin->ct0, tin->ct0 + P, tin->ct1, tin->ct1 + P, tin->dd,
                            tin->dd + P, tin->dd + 2 * P, rp, g.l1, (int64_t)U, st, &tm)))
      return rc;
  }

  // 1. y = INTT(d), every limb of the level  (ModUp's to_coeff, ckks.py:362)
  if (!y_full) {
    if (r0 != 0 || nr != g.l1) {
      set_error("key switch of a limb subset needs the gathered coefficient rows");
      return TFHE_EINVAL;
    }
    LimbMap m;
    m.n = g.l1;
    for (int r = 0; r < g.l1; ++r) m.prime[r] = m.in_row[r] = m.out_row[r] = (int16_t)r;
    EpiArgs es;   // hoisted rotation: y = phi_coeff(INTT(a)) by the INTT's output scatter
    memset(&es, 0, sizeof(es));
    es.mode = EPI_STORE;
    es.scatter_t = rot && !rot->d_is_phi ? rot->t : 0u;
    if ((rc = launch_ntt(c, d, y, m, batch, 1, es.scatter_t ? &es : nullptr, ntt_ws, ntt_ws_bytes,
                         st)))
      return rc;
    y_full = y;
  }

  // 2. ModUp + inner product  (ckks.py:337-351)
  int16_t row_prime[kMaxRows];
  for (int t = 0; t < g.nr; ++t) row_prime[t] = (int16_t)(g.r0 + t);
  if (c.use_ts) {
    // 2a. slice rows are reused unchanged (ckks.py:361-364): acc[r] = d_r * k_{slice(r)}[r]
    int64_t key_off[kMaxRows];
    for (int t = 0; t < g.nr; ++t) {
      const int r = g.r0 + t;
      key_off[t] = (int64_t)(r / g.alpha) * key_pair + (int64_t)r * c.n;
    }
    if (rot) {
      // acc_b = phi(a) k_b + P phi(b), acc_a = phi(a) k_a (phi gathered in the MAC)
      uint32_t pmod[kMaxRows];
      for (int t = 0; t < g.nr; ++t) {
        const uint32_t q = c.primes[g.r0 + t];
        uint64_t pm = 1;
        for (int k = 0; k < g.K; ++k) pm = pm * (c.primes[g.Lc + k] % q) % q;
        pmod[t] = (uint32_t)pm;
      }
      if ((rc = launch_ks_mac_rot(c, d, rot->b, key, key + key_pair / 2, acc, acc + g.T * U,
                                  row_prime, key_off, pmod, g.nr, batch, rot->t, !rot->d_is_phi,
                                  st)))
        return rc;
    } else if (fused_rows < g.nr &&
               (rc = launch_ks_mac(c, d, key, key + key_pair / 2, acc, acc + g.T * U, row_prime,
                                   key_off, g.nr, batch, 1, st))) {
      return rc;
    }
    // 2b. groups of S slices: stage 1 for every (slice, target) pair, stage 2
    // accumulates the S slices of each target on chip (EPI_KS_ACC).  A
    // slice's own rows are skipped in the sum (they were reused in 2a).
    LimbMap tmap;
    tmap.n = g.T;
    EpiArgs ek;
    memset(&ek, 0, sizeof(ek));
    ek.mode = EPI_KS_ACC;
    ek.key = key;
    ek.key_pair = (long long)key_pair;
    ek.acc_b = acc;
    ek.acc_a = acc + g.T * U;
    for (int t = 0; t < g.T; ++t) {
      tmap.prime[t] = (int16_t)tprime(g, t);
      tmap.in_row[t] = (int16_t)t;
      tmap.out_row[t] = (int16_t)t;
      ek.key_row[t] = (int16_t)tprime(g, t);  // key rows are over the full ext basis
      ek.js[t] = (int16_t)(t < g.nr ? (g.r0 + t) / g.alpha : -1);
      ek.init_acc[t] = (int16_t)(t < g.nr);  // specials start from zero
    }
    for (int j0 = 0; j0 < g.nslices; j0 += g.S) {
      const int S = std::min(g.S, g.nslices - j0);
      LimbMap s1;
      s1.n = S * g.T;
      // one input pointer per launch: if any slice of the group needs a base
      // conversion, every slice goes through conv (a 1-limb slice's
      // conversion is the identity reduced mod each target, bit-identical to
      // the NTT reading its raw row)
      bool group_conv = false;
      for (int sl = 0; sl < S; ++sl)
        group_conv |= std::min((j0 + sl) * g.alpha + g.alpha, g.l1) - (j0 + sl) * g.alpha > 1;
      const uint32_t* ntt_in = group_conv ? conv : y_full;
      for (int sl = 0; sl < S; ++sl) {
        const int j = j0 + sl, lo = j * g.alpha, hi = std::min(lo + g.alpha, g.l1);
        int cidx[kMaxRows];   // conv row of target t within the slice (-1: own row)
        if (group_conv) {
          // fast_basis_conv of the slice to the targets it raises, compacted
          // into conv rows [sl*T, sl*T + T - own): the slice's own rows
          // (copies in rns.py:140-142) are never read -- the inner product
          // reuses them unchanged -- so they are not converted at all
          std::vector<int> src, dst;
          for (int q = lo; q < hi; ++q) src.push_back(q);
          for (int t = 0; t < g.T; ++t) {
            if (t < g.nr && (g.r0 + t) / g.alpha == j) {
              cidx[t] = -1;
              continue;
            }
            cidx[t] = (int)dst.size();
            dst.push_back(tprime(g, t));
          }
          BconvArgs ba;
          if ((rc = fill_bconv(c, src, dst, ba))) return rc;
          if ((rc = launch_bconv(c, y_full + (size_t)lo * U, conv + (size_t)sl * g.T * U, ba,
                                 batch, st, /*exact_copies=*/false)))
            return rc;
        }
        for (int t = 0; t < g.T; ++t) {
          const int l = sl * g.T + t;
          s1.prime[l] = (int16_t)tprime(g, t);
          // alpha = 1: fast_basis_conv is the identity on the slice's
          // coefficients (Q = q_lo, Q/q = 1): the NTT reads y's row directly
          // and reduces it mod each target prime inside the byte-sliced GEMM.
          // An own target's limb (never used) reads any valid row.
          s1.in_row[l] =
              (int16_t)(group_conv ? sl * g.T + (cidx[t] >= 0 ? cidx[t] : 0) : lo);
          s1.out_row[l] = (int16_t)l;
        }
      }
      ek.j0 = j0;
      if ((rc = launch_ntt_ts_ks_group(c, ntt_in, ntt_ws, s1, tmap, S, batch, ek, st))) return rc;
      for (int t = 0; t < g.T; ++t) ek.init_acc[t] = 1;
    }
  } else {
    int first = 1;
    for (int j = 0; j < dnum; ++j) {
      const int lo = j * g.alpha;
      if (lo > level) break;
      const int hi = std::min((j + 1) * g.alpha, g.l1);
      LimbMap mu;
      mu.n = 0;
      std::vector<int> src, dst;
      for (int s = lo; s < hi; ++s) src.push_back(s);
      for (int t = 0; t < g.T; ++t) {
        if (t < g.nr && g.r0 + t >= lo && g.r0 + t < hi) continue;
        mu.prime[mu.n] = (int16_t)tprime(g, t);
        mu.out_row[mu.n] = (int16_t)t;
        mu.in_row[mu.n] = (int16_t)(hi - lo == 1 ? lo : mu.n);
        dst.push_back(tprime(g, t));
        ++mu.n;
      }
      const uint32_t* ntt_in = y_full;
      if (hi - lo > 1) {
        BconvArgs ba;
        if ((rc = fill_bconv(c, src, dst, ba))) return rc;
        if ((rc = launch_bconv(c, y_full + (size_t)lo * U, conv, ba, batch, st))) return rc;
        ntt_in = conv;
      }
      // alpha = 1: fast_basis_conv is the identity on the slice's coefficients
      // (Q = q_lo, Q/q = 1), so the NTT reads y's row directly and reduces it
      // mod each target prime inside the byte-sliced GEMM.  The inner product
      // acc += raised * key_j (ckks.py:345-351) is fused into the NTT's output
      // epilogue: the raised limbs never touch HBM.
      const uint32_t* kb = key + (size_t)j * key_pair;
      const uint32_t* ka = kb + (size_t)(g.Lc + g.K) * c.n;
      EpiArgs ek;
      memset(&ek, 0, sizeof(ek));
      ek.mode = EPI_KS_MAC;
      ek.kb = kb;
      ek.ka = ka;
      ek.acc_b = acc;
      ek.acc_a = acc + g.T * U;
      ek.first = first;
      for (int l = 0; l < mu.n; ++l) ek.key_row[l] = mu.prime[l];
      if (mu.n &&
          (rc = launch_ntt(c, ntt_in, nullptr, mu, batch, 0, &ek, ntt_ws, ntt_ws_bytes, st)))
        return rc;
      // slice rows are reused unchanged (ckks.py:361-364): MAC the local ones straight from d
      const int a0 = std::max(lo, g.r0), a1 = std::min(hi, g.r0 + g.nr);
      if (a1 > a0 && !(j == 0 && fused_rows > 0)) {   // slice 0's rows: done by the tensor product
        int64_t key_off[kMaxRows];
        for (int r = a0; r < a1; ++r) key_off[r - a0] = (int64_t)r * c.n;
        const size_t t0 = (size_t)(a0 - g.r0);
        if ((rc = launch_ks_mac(c, d + t0 * U, kb, ka, acc + t0 * U, acc + (g.T + t0) * U,
                                row_prime + t0, key_off, a1 - a0, batch, first, st)))
          return rc;
      }
      first = 0;
    }
  }

  // 3. ModDown of acc_b and acc_a  (ckks.py:367-381)
  LimbMap ms;
  ms.n = 2 * g.K;
  for (int cmp = 0; cmp < 2; ++cmp)
    for (int k = 0; k < g.K; ++k) {
      const int l = cmp * g.K + k;
      ms.prime[l] = (int16_t)(g.Lc + k);
      ms.in_row[l] = (int16_t)(cmp * g.T + g.nr + k);
      ms.out_row[l] = (int16_t)l;
    }
  if ((rc = launch_ntt(c, acc, ysp, ms, batch, 1, nullptr, ntt_ws, ntt_ws_bytes, st))) return rc;

  const uint32_t* md_in = ysp;
  if (g.K > 1) {
    std::vector<int> src, dst;
    for (int k = 0; k < g.K; ++k) src.push_back(g.Lc + k);
    for (int t = 0; t < g.nr; ++t) dst.push_back(g.r0 + t);
    BconvArgs ba;
    if ((rc = fill_bconv(c, src, dst, ba))) return rc;
    // both components in one call (one launch on the element-wise path)
    if ((rc = launch_bconv(c, ysp, conv, ba, batch, st, true, 2, (int64_t)g.K * U,
                           (int64_t)g.nr * U)))
      return rc;
    md_in = conv;
  }
  if (rs_scratch) return moddown_rescale(c, g, acc, md_in, conv, y, rs_scratch, base, base_rows,
                                         out, batch, ntt_ws, ntt_ws_bytes, st);
  LimbMap md;
  EpiArgs ep;
  memset(&ep, 0, sizeof(ep));
  ep.mode = EPI_SUB_SCALE;
  ep.x = acc;
  ep.base = base;
  md.n = 2 * g.nr;
  for (int t = 0; t < g.nr; ++t) {
    const int i = g.r0 + t;
    const uint32_t q = c.primes[i];
    uint64_t pm = 1;
    for (int k = 0; k < g.K; ++k) pm = pm * (c.primes[g.Lc + k] % q) % q;
    for (int cmp = 0; cmp < 2; ++cmp) {
      const int l = cmp * g.nr + t;
      md.prime[l] = (int16_t)i;
      md.in_row[l] = (int16_t)(g.K > 1 ? cmp * g.nr + t : cmp);
      md.out_row[l] = (int16_t)l;
      ep.x_row[l] = (int16_t)(cmp * g.T + t);
      ep.base_row[l] = base ? base_rows[l] : (int16_t)-1;
      ep.s[l] = invmod(pm, q);
      ep.s_shoup[l] = shoup(ep.s[l], q);
    }
  }
  return launch_ntt(c, md_in, out, md, batch, 0, &ep, ntt_ws, ntt_ws_bytes, st);
}

int check_ctx(const TfheCtx* h) {
  if (!h) {
    set_error("null context");
    return TFHE_EINVAL;
  }
  return 0;
}

int check_limbs(const TfheCtx* h, const int32_t* primes, int n) {
  if (n < 0 || n > kMaxLimbs) {
    set_error("limb count out of range (max " + std::to_string(kMaxLimbs) + ")");
    return TFHE_EINVAL;
  }
  for (int i = 0; i < n; ++i)
    if (primes[i] < 0 || primes[i] >= h->c.n_primes) {
      set_error("prime index out of range");
      return TFHE_EINVAL;
    }
  return 0;
}

int check_level(const TfheCtx* h, int level, int batch, int dnum) {
  if (level < 0 || level >= h->n_chain || batch <= 0) {
    set_error("bad level or batch");
    return TFHE_EINVAL;
  }
  if (dnum != 0 && (dnum < 0 || h->n_chain % dnum != 0)) {
    set_error("dnum must divide L+1");
    return TFHE_EINVAL;
  }
  if (h->n_special <= 0 && dnum != 0) {
    set_error("context has no special primes");
    return TFHE_EINVAL;
  }
  if (2 * (level + 1) > kMaxLimbs || level + 1 + h->n_special > kMaxLimbs) {
    set_error("too many limbs for one launch");
    return TFHE_EINVAL;
  }
  return 0;
}

}  // namespace
}  // namespace tfhe

using namespace tfhe;

extern "C" {

int tfhe_abi_version(void) { return TFHE_ABI_VERSION; }
const char* tfhe_last_error(void) { return g_last_error.c_str(); }

int tfhe_ctx_create(int device, int log_n, const uint32_t* primes, const uint32_t* psis,
                    int n_chain, int n_special, TfheCtx** out) {
  if (!out || !primes || !psis || log_n < 4 || log_n > 17 || n_chain < 1 || n_special < 0 ||
      n_chain + n_special > 200) {
    set_error("tfhe_ctx_create: bad arguments");
    return TFHE_EINVAL;
  }
  const uint32_t n = 1u << log_n;
  for (int i = 0; i < n_chain + n_special; ++i) {
    const uint32_t q = primes[i];
    if (q >= (1u << 31) || q % (2 * n) != 1) {
      set_error("prime " + std::to_string(q) + " is not 1 mod 2n or >= 2^31");
      return TFHE_EINVAL;
    }
    if (powmod(psis[i], n, q) != q - 1) {
      set_error("psi is not a negacyclic root for prime " + std::to_string(q));
      return TFHE_EINVAL;
    }
  }
  if (cudaSetDevice(device) != cudaSuccess) {
    set_error("cudaSetDevice failed");
    return TFHE_ECUDA;
  }
  TfheCtx* h = new TfheCtx();
  Ctx& c = h->c;
  c.dev = device;
  c.log_n = log_n;
  c.n = (int)n;
  c.n1 = 1 << (log_n / 2);  // params.build_ntt_plan (MAX_N1 never binds for n <= 2^17)
  c.n2 = c.n / c.n1;
  c.n_primes = n_chain + n_special;
  c.primes.assign(primes, primes + c.n_primes);
  c.psis.assign(psis, psis + c.n_primes);
  h->n_chain = n_chain;
  h->n_special = n_special;
  int rc = build_ntt_tables(c);
  if (rc) {
    tfhe_ctx_destroy(h);
    return rc;
  }
  *out = h;
  return 0;
}

void tfhe_ctx_destroy(TfheCtx* h) {
  if (!h) return;
  Ctx& c = h->c;
  for (auto& e : h->crt_cache) cudaFree(e.second.first);
  if (h->h_bounce) cudaFreeHost(h->h_bounce);
  if (h->h2d) {
    cudaStreamDestroy(h->h2d);
    cudaStreamDestroy(h->d2h);
    cudaEventDestroy(h->ev_start);
    for (int i = 0; i < 3; ++i) {
      cudaEventDestroy(h->ev_in[i]);
      cudaEventDestroy(h->ev_done[i]);
      cudaEventDestroy(h->ev_out[i]);
    }
  }
  cudaFree(c.d_pc);
  cudaFree(c.d_fw2_ks);
  cudaFree(c.d_p3t2ks);
  for (int i = 0; i < 2; ++i) {
    for (int s = 0; s < 2; ++s) {
      cudaFree(c.d_tw[i][s]);
      if (i == 0 && s == 0) cudaFree(c.d_tw_ks);
      cudaFree(c.d_twa[i][s]);
      if (i == 0 && s == 0) cudaFree(c.d_twa_ks);
    }
    cudaFree(c.d_w2[i]);
    cudaFree(c.d_w2s[i]);
    cudaFree(c.d_fdft[i]);
    cudaFree(c.d_p3t1[i]);
    cudaFree(c.d_p3hin[i]);
    cudaFree(c.d_p3hout[i]);
    cudaFree(c.d_p3t2[i]);
    cudaFree(c.d_fw2[i]);
    cudaFree(c.d_w2r[i]);
    cudaFree(c.d_w2rs[i]);
  }
  delete h;
}

int tfhe_ctx_plan(const TfheCtx* h, int* n1, int* n2) {
  if (check_ctx(h)) return TFHE_EINVAL;
  if (n1) *n1 = h->c.n1;
  if (n2) *n2 = h->c.n2;
  return 0;
}

int tfhe_ctx_transform_plan(const TfheCtx* h, int* k0, int* k1, int* k2) {
  if (check_ctx(h)) return TFHE_EINVAL;
  const Ctx& c = h->c;
  int f[3] = {c.n1, c.n2, 0};
  if (c.use_p3) {
    f[0] = 32;
    f[1] = 32;
    f[2] = 64;
  }
  if (k0) *k0 = f[0];
  if (k1) *k1 = f[1];
  if (k2) *k2 = f[2];
  return 0;
}

size_t tfhe_ntt_workspace_bytes(const TfheCtx* h, int n_limbs, int batch) {
  return h ? ntt_workspace_bytes(h->c, n_limbs, batch) : 0;
}

int tfhe_ntt(TfheCtx* h, const uint32_t* in, uint32_t* out, const int32_t* limb_prime,
             const int32_t* in_rows, const int32_t* out_rows, int n_limbs, int batch, int inverse,
             void* ws, size_t ws_bytes, void* stream) {
  int rc;
  if ((rc = check_ctx(h)) || (rc = check_limbs(h, limb_prime, n_limbs))) return rc;
  if (batch < 0 || (n_limbs && (!in || !out || !ws))) {
    set_error("tfhe_ntt: bad arguments");
    return TFHE_EINVAL;
  }
  LimbMap m;
  m.n = n_limbs;
  for (int l = 0; l < n_limbs; ++l) {
    m.prime[l] = (int16_t)limb_prime[l];
    m.in_row[l] = (int16_t)(in_rows ? in_rows[l] : l);
    m.out_row[l] = (int16_t)(out_rows ? out_rows[l] : l);
  }
  return launch_ntt(h->c, in, out, m, batch, inverse != 0, nullptr, ws, ws_bytes,
                    (cudaStream_t)stream);
}

int tfhe_eltwise(TfheCtx* h, int op, const uint32_t* a, const uint32_t* b, uint32_t* out,
                 const int32_t* row_prime, int rows, int64_t per_row, const uint32_t* scalars,
                 void* stream) {
  int rc;
  if ((rc = check_ctx(h))) return rc;
  if (rows < 0 || rows > kMaxRows || per_row % 4 || (rows && (!a || !out))) {
    set_error("tfhe_eltwise: bad shape (rows <= 256, per_row % 4 == 0)");
    return TFHE_EINVAL;
  }
  int16_t rp[kMaxRows];
  for (int r = 0; r < rows; ++r) {
    if (row_prime[r] < 0 || row_prime[r] >= h->c.n_primes) {
      set_error("prime index out of range");
      return TFHE_EINVAL;
    }
    rp[r] = (int16_t)row_prime[r];
  }
  cudaStream_t st = (cudaStream_t)stream;
  switch (op) {
    case TFHE_OP_ADD:
    case TFHE_OP_SUB:
    case TFHE_OP_MUL:
      if (!b) {
        set_error("binary op needs b");
        return TFHE_EINVAL;
      }
      return launch_binary(h->c, op, a, b, out, rp, rows, per_row, st);
    case TFHE_OP_NEG: return launch_unary(h->c, OP_NEG, a, out, rp, nullptr, rows, per_row, st);
    case TFHE_OP_SCALAR:
      if (!scalars) {
        set_error("scalar op needs scalars");
        return TFHE_EINVAL;
      }
      return launch_unary(h->c, OP_SCALAR, a, out, rp, scalars, rows, per_row, st);
  }
  set_error("unknown op");
  return TFHE_EINVAL;
}

int tfhe_automorphism(TfheCtx* h, const uint32_t* in, uint32_t* out, uint32_t galois_t,
                      int ntt_domain, const int32_t* row_prime, int rows, int batch,
                      void* stream) {
  int rc;
  if ((rc = check_ctx(h))) return rc;
  if ((galois_t & 1) == 0 || rows < 0 || rows > kMaxRows || in == out) {
    set_error("tfhe_automorphism: bad arguments (odd t, out != in)");
    return TFHE_EINVAL;
  }
  int16_t rp[kMaxRows];
  for (int r = 0; r < rows; ++r) rp[r] = (int16_t)(row_prime ? row_prime[r] : 0);
  return launch_automorph(h->c, in, out, galois_t, ntt_domain, rp, rows, batch,
                          (cudaStream_t)stream);
}

int tfhe_bconv(TfheCtx* h, const uint32_t* in, uint32_t* out, const int32_t* src_prime,
               int n_src, const int32_t* dst_prime, int n_dst, int batch, void* stream) {
  int rc;
  if ((rc = check_ctx(h)) || (rc = check_limbs(h, src_prime, n_src)) ||
      (rc = check_limbs(h, dst_prime, n_dst)))
    return rc;
  std::vector<int> s(src_prime, src_prime + n_src), d(dst_prime, dst_prime + n_dst);
  BconvArgs ba;
  if ((rc = fill_bconv(h->c, s, d, ba))) return rc;
  return launch_bconv(h->c, in, out, ba, batch, (cudaStream_t)stream);
}

size_t tfhe_ckks_workspace_bytes(const TfheCtx* h, int level, int batch) {
  if (!h) return 0;
  // worst case over dnum: general base conversion buffers included
  // worst case over dnum: alpha = 1 maximises the key-switch group size,
  // general base-conversion buffers included
  CkksGeom g = geom(h, level, h->n_chain);
  set_group(g, h->c, batch);
  g.need_conv = true;
  const size_t U = (size_t)batch * h->c.n * 4;
  return ks_bytes(g, batch, h->c.n) + 3 * (size_t)g.l1 * U + 256;
}

int tfhe_keyswitch(TfheCtx* h, const uint32_t* d, int level, int batch, const uint32_t* key,
                   int dnum, uint32_t* out, const uint32_t* add, void* ws, size_t ws_bytes,
                   void* stream) {
  int rc;
  if ((rc = check_ctx(h)) || (rc = check_level(h, level, batch, dnum ? dnum : -1))) return rc;
  Carve cv{static_cast<uint8_t*>(ws), ws_bytes};
  int16_t rows[kMaxLimbs];
  for (int l = 0; l < 2 * (level + 1); ++l) rows[l] = (int16_t)l;
  return keyswitch_impl(h, d, nullptr, level, batch, key, dnum, 0, level + 1, out, add, rows, cv,
                        (cudaStream_t)stream);
}

int tfhe_hmult(TfheCtx* h, const uint32_t* ct0, const uint32_t* ct1, int level, int batch,
               const uint32_t* rlk, int dnum, uint32_t* out, void* ws, size_t ws_bytes,
               void* stream) {
  int rc;
  if ((rc = check_ctx(h)) || (rc = check_level(h, level, batch, dnum ? dnum : -1))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const int l1 = level + 1;
  const size_t P = (size_t)l1 * batch * h->c.n;  // elements per component
  Carve cv{static_cast<uint8_t*>(ws), ws_bytes};
  uint32_t* dd = cv.take<uint32_t>(3 * P * 4);  // d0 | d1 | d2
  if (!cv.ok) {
    set_error("ckks workspace too small");
    return TFHE_EINVAL;
  }
  int16_t rows[kMaxLimbs];
  for (int l = 0; l < 2 * l1; ++l) rows[l] = (int16_t)l;  // (d0, d1) added to (ksb, ksa)
  const TensorIn tin{ct0, ct1, dd};   // the tensor product runs inside, MACs fused
  return keyswitch_impl(h, dd + 2 * P, nullptr, level, batch, rlk, dnum, 0, l1, out, dd, rows, cv,
                        st, nullptr, nullptr, &tin);
}

int tfhe_hmult_rescale(TfheCtx* h, const uint32_t* ct0, const uint32_t* ct1, int level,
                       int batch, const uint32_t* rlk, int dnum, uint32_t* out, void* ws,
                       size_t ws_bytes, void* stream) {
  int rc;
  if ((rc = check_ctx(h)) || (rc = check_level(h, level, batch, dnum ? dnum : -1))) return rc;
  if (level < 1) {
    set_error("no levels left to rescale");
    return TFHE_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int l1 = level + 1;
  const size_t P = (size_t)l1 * batch * h->c.n;  // elements per component
  Carve cv{static_cast<uint8_t*>(ws), ws_bytes};
  uint32_t* dd = cv.take<uint32_t>(3 * P * 4);  // d0 | d1 | d2
  if (!cv.ok) {
    set_error("ckks workspace too small");
    return TFHE_EINVAL;
  }
  int16_t rows[kMaxLimbs];
  for (int l = 0; l < 2 * l1; ++l) rows[l] = (int16_t)l;
  // d2 (the key-switch input) is dead after ModUp: its first rows hold the top
  // row's coefficient form for the fused rescale
  const TensorIn tin{ct0, ct1, dd};   // the tensor product runs inside, MACs fused
  return keyswitch_impl(h, dd + 2 * P, nullptr, level, batch, rlk, dnum, 0, l1, out, dd, rows, cv,
                        st, dd + 2 * P, nullptr, &tin);
}

int tfhe_rescale(TfheCtx* h, const uint32_t* ct, int level, int batch, uint32_t* out, void* ws,
                 size_t ws_bytes, void* stream) {
  int rc;
  if ((rc = check_ctx(h)) || (rc = check_level(h, level, batch, 0))) return rc;
  if (level < 1) {
    set_error("no levels left to rescale");
    return TFHE_EINVAL;
  }
  const Ctx& c = h->c;
  cudaStream_t st = (cudaStream_t)stream;
  const int l1 = level + 1;
  const size_t U = (size_t)batch * c.n;
  Carve cv{static_cast<uint8_t*>(ws), ws_bytes};
  uint32_t* t = cv.take<uint32_t>(2 * U * 4);
  const size_t nws = (size_t)2 * level * U * 4;
  uint32_t* nw = cv.take<uint32_t>(nws);
  if (!cv.ok) {
    set_error("ckks workspace too small");
    return TFHE_EINVAL;
  }
  // t = INTT_{q_top}(c_top) for b and a
  LimbMap m;
  m.n = 2;
  for (int cmp = 0; cmp < 2; ++cmp) {
    m.prime[cmp] = (int16_t)level;
    m.in_row[cmp] = (int16_t)(cmp * l1 + level);
    m.out_row[cmp] = (int16_t)cmp;
  }
  if ((rc = launch_ntt(c, ct, t, m, batch, 1, nullptr, nw, nws, st))) return rc;
  // out_i = (c_i - NTT_{q_i}(t)) * q_top^-1 : the NTT-domain form of
  // _rescale_poly (ckks.py:301-311), bit-identical by linearity of the NTT
  LimbMap mr;
  EpiArgs ep;
  memset(&ep, 0, sizeof(ep));
  ep.mode = EPI_SUB_SCALE;
  ep.x = ct;
  mr.n = 2 * level;
  const uint32_t q_top = c.primes[level];
  for (int cmp = 0; cmp < 2; ++cmp)
    for (int i = 0; i < level; ++i) {
      const int l = cmp * level + i;
      mr.prime[l] = (int16_t)i;
      mr.in_row[l] = (int16_t)cmp;
      mr.out_row[l] = (int16_t)l;
      ep.x_row[l] = (int16_t)(cmp * l1 + i);
      ep.base_row[l] = -1;
      ep.s[l] = invmod(q_top, c.primes[i]);
      ep.s_shoup[l] = shoup(ep.s[l], c.primes[i]);
    }
  return launch_ntt(c, t, out, mr, batch, 0, &ep, nw, nws, st);
}

int tfhe_hrotate(TfheCtx* h, const uint32_t* ct, int level, int batch, uint32_t galois_t,
                 const uint32_t* key, int dnum, uint32_t* out, void* ws, size_t ws_bytes,
                 void* stream) {
  int rc;
  if ((rc = check_ctx(h)) || (rc = check_level(h, level, batch, dnum ? dnum : -1))) return rc;
  if ((galois_t & 1) == 0) {
    set_error("galois element must be odd");
    return TFHE_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int l1 = level + 1;
  const size_t P = (size_t)l1 * batch * h->c.n;
  Carve cv{static_cast<uint8_t*>(ws), ws_bytes};
  int16_t rp[kMaxRows];
  for (int i = 0; i < 2 * l1; ++i) rp[i] = (int16_t)(i % l1);
  const Ctx& c = h->c;
  if (c.use_ts && !getenv_flag("TFHE_NO_HOIST")) {
    // hoisted automorphism: phi(b) folds into the key switch's
    // slice MAC; phi(a) is the INTT's output scatter on the p3 plan, a gather
    // of a alone on the TS plans (2^14, 2^15)
    RotHoist rot{galois_t, ct, 0};
    const uint32_t* d = ct + P;
    if (!c.use_p3) {
      uint32_t* phia = cv.take<uint32_t>(P * 4);
      if (!cv.ok) {
        set_error("ckks workspace too small");
        return TFHE_EINVAL;
      }
      if ((rc = launch_automorph(c, ct + P, phia, galois_t, 1, rp, l1, batch, st))) return rc;
      d = phia;
      rot.d_is_phi = 1;
    }
    return keyswitch_impl(h, d, nullptr, level, batch, key, dnum, 0, l1, out, nullptr, nullptr, cv,
                          st, nullptr, &rot);
  }
  uint32_t* phi = cv.take<uint32_t>(2 * P * 4);
  if (!cv.ok) {
    set_error("ckks workspace too small");
    return TFHE_EINVAL;
  }
  if ((rc = launch_automorph(h->c, ct, phi, galois_t, 1, rp, 2 * l1, batch, st))) return rc;
  int16_t rows[kMaxLimbs];
  for (int i = 0; i < l1; ++i) {
    rows[i] = (int16_t)i;   // b' = phi(b) + ksb
    rows[l1 + i] = -1;      // a' = ksa
  }
  return keyswitch_impl(h, phi + P, nullptr, level, batch, key, dnum, 0, l1, out, phi, rows, cv,
                        st);
}

}  // extern "C"

/* ---- limb-partitioned evaluation ----------------------------- */
extern "C" {

int tfhe_tensor_product(TfheCtx* h, const uint32_t* ct0, const uint32_t* ct1, int row_lo,
                        int n_rows, int batch, uint32_t* out, void* stream) {
  int rc;
  if ((rc = check_ctx(h))) return rc;
  if (row_lo < 0 || n_rows < 0 || n_rows > kMaxRows || row_lo + n_rows > h->n_chain ||
      batch <= 0 || (n_rows && (!ct0 || !ct1 || !out))) {
    set_error("tfhe_tensor_product: bad arguments");
    return TFHE_EINVAL;
  }
  if (!n_rows) return 0;
  const size_t P = (size_t)n_rows * batch * h->c.n;
  int16_t rp[kMaxRows];
  for (int i = 0; i < n_rows; ++i) rp[i] = (int16_t)(row_lo + i);
  return launch_tensor(h->c, ct0, ct0 + P, ct1, ct1 + P, out, out + P, out + 2 * P, rp, n_rows,
                       (int64_t)batch * h->c.n, (cudaStream_t)stream);
}

int tfhe_keyswitch_part(TfheCtx* h, const uint32_t* d_local, const uint32_t* y_full, int level,
                        int batch, const uint32_t* key, int dnum, int row_lo, int n_rows,
                        uint32_t* out, const uint32_t* add, int add_components, void* ws,
                        size_t ws_bytes, void* stream) {
  int rc;
  if ((rc = check_ctx(h)) || (rc = check_level(h, level, batch, dnum ? dnum : -1))) return rc;
  if (!y_full || !key || !out || row_lo < 0 || n_rows < 1 || row_lo + n_rows > level + 1 ||
      !d_local || add_components < 0 || add_components > 2) {
    set_error("tfhe_keyswitch_part: bad arguments");
    return TFHE_EINVAL;
  }
  Carve cv{static_cast<uint8_t*>(ws), ws_bytes};
  int16_t rows[kMaxLimbs];
  for (int l = 0; l < 2 * n_rows; ++l) rows[l] = (int16_t)(l < add_components * n_rows ? l : -1);
  return keyswitch_impl(h, d_local, y_full, level, batch, key, dnum, row_lo, n_rows, out, add,
                        rows, cv, (cudaStream_t)stream);
}

int tfhe_rescale_part(TfheCtx* h, const uint32_t* ct_local, const uint32_t* top_coeff, int level,
                      int batch, int row_lo, int n_rows, uint32_t* out, void* ws, size_t ws_bytes,
                      void* stream) {
  int rc;
  if ((rc = check_ctx(h)) || (rc = check_level(h, level, batch, 0))) return rc;
  if (level < 1 || !top_coeff || row_lo < 0 || n_rows < 0 || row_lo + n_rows > level + 1 ||
      (n_rows && (!ct_local || !out))) {
    set_error("tfhe_rescale_part: bad arguments");
    return TFHE_EINVAL;
  }
  const Ctx& c = h->c;
  const int nout = std::max(0, std::min(row_lo + n_rows, level) - row_lo);  // rows kept
  if (!nout) return 0;
  const size_t U = (size_t)batch * c.n;
  Carve cv{static_cast<uint8_t*>(ws), ws_bytes};
  const size_t nws = (size_t)2 * nout * U * 4;
  uint32_t* nw = cv.take<uint32_t>(nws);
  if (!cv.ok) {
    set_error("ckks workspace too small");
    return TFHE_EINVAL;
  }
  // out_i = (c_i - NTT_{q_i}(t_top)) * q_top^-1 for the local rows i < level
  LimbMap mr;
  EpiArgs ep;
  memset(&ep, 0, sizeof(ep));
  ep.mode = EPI_SUB_SCALE;
  ep.x = ct_local;
  mr.n = 2 * nout;
  const uint32_t q_top = c.primes[level];
  for (int cmp = 0; cmp < 2; ++cmp)
    for (int t = 0; t < nout; ++t) {
      const int l = cmp * nout + t, i = row_lo + t;
      mr.prime[l] = (int16_t)i;
      mr.in_row[l] = (int16_t)cmp;
      mr.out_row[l] = (int16_t)l;
      ep.x_row[l] = (int16_t)(cmp * n_rows + t);
      ep.base_row[l] = -1;
      ep.s[l] = invmod(q_top, c.primes[i]);
      ep.s_shoup[l] = shoup(ep.s[l], c.primes[i]);
    }
  return launch_ntt(c, top_coeff, out, mr, batch, 0, &ep, nw, nws, (cudaStream_t)stream);
}

}  // extern "C"

/* ---- diagnostics --------------------------------------------------------- */
extern "C" int tfhe_debug_corrupt_twiddle(TfheCtx* h, int prime) {
  if (check_ctx(h)) return TFHE_EINVAL;
  Ctx& c = h->c;
  if (prime < 0 || prime >= c.n_primes) {
    set_error("prime index out of range");
    return TFHE_EINVAL;
  }
  // byte offsets (in each forward stage table) of this prime's first twiddle
  // plane byte: small-n tiles [prime][tile...] and TS planes [prime][half][row][plane][K]
  auto flip = [](void* dev_byte) {
    uint8_t v = 0;
    if (cudaMemcpy(&v, dev_byte, 1, cudaMemcpyDeviceToHost) != cudaSuccess) return false;
    v ^= 0x01;
    return cudaMemcpy(dev_byte, &v, 1, cudaMemcpyHostToDevice) == cudaSuccess;
  };
  bool ok = true;
  for (int s = 0; s < 2; ++s)
    if (c.d_tw[0][s]) ok &= flip(c.d_tw[0][s] + (size_t)prime * c.tw_stride[s]);
  if (c.d_fdft[0]) ok &= flip(c.d_fdft[0] + (size_t)prime * 65536);
  if (c.d_p3t1[0]) ok &= flip(c.d_p3t1[0] + (size_t)prime * 16384);
  for (int s = 0; s < 2; ++s) {
    if (!c.d_twa[0][s]) continue;
    const size_t ntw = s == 0 ? c.n1 : c.n2;      // rows (= K) of this stage
    ok &= flip(reinterpret_cast<uint8_t*>(c.d_twa[0][s]) + (size_t)prime * ntw * ntw * 4);
  }
  if (!ok) {
    set_error("twiddle fault injection: device copy failed");
    return TFHE_ECUDA;
  }
  return 0;
}

/* ---- host-streaming transform (e2e path of batched_apply / transform_rows) -- */
namespace {
constexpr int kHostSlots = 3;
constexpr size_t kHostChunkBytes = (size_t)48 << 20;

int host_chunk_rows(const TfheCtx* h, int n_limbs, int batch) {
  const size_t row = (size_t)batch * h->c.n * 4;
  return (int)std::max<size_t>(1, std::min<size_t>((size_t)n_limbs, kHostChunkBytes / row));
}

bool is_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// host memcpy split over the host cores (pageable <-> pinned bounce slots)
void par_memcpy(void* dst, const void* src, size_t bytes) {
  const size_t blk = (size_t)1 << 20;
  const long long nb = (long long)((bytes + blk - 1) / blk);
#pragma omp parallel for schedule(static)
  for (long long b = 0; b < nb; ++b) {
    const size_t off = (size_t)b * blk;
    memcpy(static_cast<uint8_t*>(dst) + off, static_cast<const uint8_t*>(src) + off,
           std::min(blk, bytes - off));
  }
}
}  // namespace

extern "C" {

size_t tfhe_ntt_host_staging_bytes(const TfheCtx* h, int n_limbs, int batch) {
  if (!h || n_limbs <= 0 || batch <= 0) return 0;
  const int rc = host_chunk_rows(h, n_limbs, batch);
  const size_t chunk = ((size_t)rc * batch * h->c.n * 4 + 255) & ~(size_t)255;
  return (2 * kHostSlots) * chunk + ((ntt_workspace_bytes(h->c, rc, batch) + 255) & ~(size_t)255);
}

int tfhe_ntt_host(TfheCtx* h, const uint32_t* host_in, uint32_t* host_out,
                  const int32_t* limb_prime, int n_limbs, int batch, int inverse, void* staging,
                  size_t staging_bytes, void* stream) {
  int rc;
  if ((rc = check_ctx(h)) || (rc = check_limbs(h, limb_prime, n_limbs))) return rc;
  if (batch <= 0 || (n_limbs && (!host_in || !host_out || !staging)) ||
      staging_bytes < tfhe_ntt_host_staging_bytes(h, n_limbs, batch)) {
    set_error("tfhe_ntt_host: bad arguments or staging too small");
    return TFHE_EINVAL;
  }
  if (!n_limbs) return 0;
  if (!h->h2d) {
    if (cudaStreamCreateWithFlags(&h->h2d, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&h->d2h, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_start, cudaEventDisableTiming) != cudaSuccess) {
      set_error("tfhe_ntt_host: stream creation failed");
      return TFHE_ECUDA;
    }
    for (int i = 0; i < kHostSlots; ++i)
      if (cudaEventCreateWithFlags(&h->ev_in[i], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&h->ev_done[i], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&h->ev_out[i], cudaEventDisableTiming) != cudaSuccess) {
        set_error("tfhe_ntt_host: event creation failed");
        return TFHE_ECUDA;
      }
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int rows = host_chunk_rows(h, n_limbs, batch);
  const size_t row_elems = (size_t)batch * h->c.n;
  const size_t chunk = (rows * row_elems * 4 + 255) & ~(size_t)255;
  uint8_t* base = static_cast<uint8_t*>(staging);
  void* ws = base + 2 * kHostSlots * chunk;
  const size_t ws_bytes = staging_bytes - 2 * kHostSlots * chunk;
  // pageable host buffers go through pinned bounce slots, filled / drained
  // by a parallel host memcpy (a pageable cudaMemcpyAsync is synchronous and
  // serialises the copy engines); this makes the call host-blocking
  const bool stage_in = !is_pinned(host_in), stage_out = !is_pinned(host_out);
  if ((stage_in || stage_out) && h->h_bounce_chunk < chunk) {
    if (h->h_bounce) cudaFreeHost(h->h_bounce);
    h->h_bounce = nullptr;
    h->h_bounce_chunk = 0;
    if (cudaHostAlloc(&h->h_bounce, 2 * kHostSlots * chunk, cudaHostAllocDefault) != cudaSuccess) {
      set_error("tfhe_ntt_host: pinned bounce allocation failed");
      return TFHE_ECUDA;
    }
    h->h_bounce_chunk = chunk;
  }
  auto bounce = [&](int slot, int out) {
    return h->h_bounce + (size_t)(out * kHostSlots + slot) * h->h_bounce_chunk;
  };
  auto drain_out = [&](int i) {
    const int k = i % kHostSlots, r0 = i * rows, nr = std::min(rows, n_limbs - r0);
    cudaEventSynchronize(h->ev_out[k]);
    par_memcpy(host_out + r0 * row_elems, bounce(k, 1), nr * row_elems * 4);
  };
  // staging may still be in use by earlier work on the caller's stream
  cudaEventRecord(h->ev_start, st);
  cudaStreamWaitEvent(h->h2d, h->ev_start, 0);
  cudaStreamWaitEvent(h->d2h, h->ev_start, 0);
  const int n_chunks = (n_limbs + rows - 1) / rows;
  for (int i = 0; i < n_chunks; ++i) {
    const int k = i % kHostSlots, r0 = i * rows, nr = std::min(rows, n_limbs - r0);
    uint32_t* din = reinterpret_cast<uint32_t*>(base + (2 * k) * chunk);
    uint32_t* dout = reinterpret_cast<uint32_t*>(base + (2 * k + 1) * chunk);
    const size_t bytes = nr * row_elems * 4;
    const uint32_t* src = host_in + r0 * row_elems;
    if (stage_in) {
      // bounce slot k is free once chunk i-3's H2D has completed
      if (i >= kHostSlots) cudaEventSynchronize(h->ev_in[k]);
      par_memcpy(bounce(k, 0), src, bytes);
      src = reinterpret_cast<const uint32_t*>(bounce(k, 0));
    }
    // H2D into slot k once chunk i-3 has been transformed (din free)
    if (i >= kHostSlots) cudaStreamWaitEvent(h->h2d, h->ev_done[k], 0);
    cudaMemcpyAsync(din, src, bytes, cudaMemcpyHostToDevice, h->h2d);
    cudaEventRecord(h->ev_in[k], h->h2d);
    // transform on the caller's stream once the data is in and dout is drained
    cudaStreamWaitEvent(st, h->ev_in[k], 0);
    if (i >= kHostSlots) cudaStreamWaitEvent(st, h->ev_out[k], 0);
    LimbMap m;
    m.n = nr;
    for (int l = 0; l < nr; ++l) {
      m.prime[l] = (int16_t)limb_prime[r0 + l];
      m.in_row[l] = m.out_row[l] = (int16_t)l;
    }
    if ((rc = launch_ntt(h->c, din, dout, m, batch, inverse != 0, nullptr, ws, ws_bytes, st)))
      return rc;
    cudaEventRecord(h->ev_done[k], st);
    // D2H of the result (into the bounce slot first for a pageable output,
    // whose previous chunk is copied out before the slot is reused)
    cudaStreamWaitEvent(h->d2h, h->ev_done[k], 0);
    if (stage_out) {
      if (i >= kHostSlots) drain_out(i - kHostSlots);
      cudaMemcpyAsync(bounce(k, 1), dout, bytes, cudaMemcpyDeviceToHost, h->d2h);
    } else {
      cudaMemcpyAsync(host_out + r0 * row_elems, dout, bytes, cudaMemcpyDeviceToHost, h->d2h);
    }
    cudaEventRecord(h->ev_out[k], h->d2h);
  }
  if (stage_out)
    for (int i = std::max(0, n_chunks - kHostSlots); i < n_chunks; ++i) drain_out(i);
  // the caller's stream completes after the last copy back
  for (int k = 0; k < std::min(n_chunks, kHostSlots); ++k) cudaStreamWaitEvent(st, h->ev_out[k], 0);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("tfhe_ntt_host: ") + cudaGetErrorString(e));
    return TFHE_ECUDA;
  }
  return 0;
}

}  // extern "C"

// ============================================================ per-kernel timing
namespace tfhe {
namespace {
struct ProfRec {
  const char* name;
  cudaEvent_t a, b;
};
std::atomic<bool> g_prof{false};
std::mutex g_prof_mu;
std::vector<ProfRec> g_prof_recs;
std::vector<cudaEvent_t> g_prof_pool;
thread_local ProfRec t_open = {nullptr, nullptr, nullptr};
cudaEvent_t prof_event() {
  if (!g_prof_pool.empty()) {
    cudaEvent_t e = g_prof_pool.back();
    g_prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

void prof_begin(const char* name, cudaStream_t st) {
  if (!g_prof.load(std::memory_order_relaxed)) return;
  std::lock_guard<std::mutex> g(g_prof_mu);
  t_open.name = name;
  t_open.a = prof_event();
  t_open.b = prof_event();
  cudaEventRecord(t_open.a, st);
}
void prof_end(cudaStream_t st) {
  if (!t_open.name) return;
  std::lock_guard<std::mutex> g(g_prof_mu);
  cudaEventRecord(t_open.b, st);
  g_prof_recs.push_back(t_open);
  t_open = {nullptr, nullptr, nullptr};
}
}  // namespace tfhe

extern "C" {

int tfhe_profile_enable(int enable) {
  tfhe::g_prof.store(enable != 0);
  return 0;
}

int tfhe_profile_read(char* buf, size_t len) {
  using namespace tfhe;
  std::lock_guard<std::mutex> g(g_prof_mu);
  std::vector<std::string> names;
  std::vector<std::pair<int, double>> acc;
  for (const ProfRec& r : g_prof_recs) {
    if (cudaEventSynchronize(r.b) != cudaSuccess) {
      set_error("tfhe_profile_read: event synchronisation failed");
      return -TFHE_ECUDA;
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    size_t k = 0;
    while (k < names.size() && names[k] != r.name) ++k;
    if (k == names.size()) {
      names.push_back(r.name);
      acc.push_back({0, 0.0});
    }
    acc[k].first += 1;
    acc[k].second += ms;
    g_prof_pool.push_back(r.a);
    g_prof_pool.push_back(r.b);
  }
  g_prof_recs.clear();
  std::string out;
  for (size_t k = 0; k < names.size(); ++k) {
    char line[256];
    snprintf(line, sizeof(line), "%s\t%d\t%.6f\n", names[k].c_str(), acc[k].first, acc[k].second);
    out += line;
  }
  if (buf && len) {
    const size_t n = std::min(len - 1, out.size());
    memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return (int)names.size();
}

}  // extern "C"

// ============================================================ client-side CRT
extern "C" {

static int crt_rows(const TfheCtx* h, const int32_t* limb_prime, int n_limbs, tfhe::CrtRows& r) {
  using namespace tfhe;
  if (!h || !limb_prime || n_limbs < 1 || n_limbs > kMaxCrtRows) {
    set_error("crt: 1..128 limbs over the context's primes");
    return TFHE_EINVAL;
  }
  r.n = n_limbs;
  for (int l = 0; l < n_limbs; ++l) {
    if (limb_prime[l] < 0 || limb_prime[l] >= h->c.n_primes) {
      set_error("crt: prime index out of range");
      return TFHE_EINVAL;
    }
    r.prime[l] = (int16_t)limb_prime[l];
  }
  return 0;
}

int tfhe_crt_decompose(TfheCtx* h, const void* coeffs, int kind, int64_t n,
                       const int32_t* limb_prime, int n_limbs, uint32_t* out, void* stream) {
  using namespace tfhe;
  CrtRows r;
  int rc = crt_rows(h, limb_prime, n_limbs, r);
  if (rc) return rc;
  if (kind != 0 && kind != 1) {
    set_error("crt_decompose: kind must be 0 (int64) or 1 (float64, rint)");
    return TFHE_EINVAL;
  }
  if (n < 0 || (n > 0 && (!coeffs || !out))) {
    set_error("crt_decompose: bad buffers");
    return TFHE_EINVAL;
  }
  return launch_crt_decompose(h->c, coeffs, kind, n, r, out, (cudaStream_t)stream);
}

int tfhe_crt_words(const TfheCtx* h, const int32_t* limb_prime, int n_limbs) {
  using namespace tfhe;
  CrtRows r;
  int rc = crt_rows(h, limb_prime, n_limbs, r);
  if (rc) return -rc;
  return crt_compose_words(h->c, r.prime, r.n);
}

int tfhe_crt_compose(TfheCtx* h, const uint32_t* rows, const int32_t* limb_prime, int n_limbs,
                     int64_t n, double* out_f64, uint32_t* out_words, int n_words, void* stream) {
  using namespace tfhe;
  CrtRows r;
  int rc = crt_rows(h, limb_prime, n_limbs, r);
  if (rc) return rc;
  if (n < 0 || (n > 0 && !rows) || (out_words && n_words < 1)) {
    set_error("crt_compose: bad buffers");
    return TFHE_EINVAL;
  }
  std::vector<int16_t> key(r.prime, r.prime + r.n);
  uint32_t* d_cst = nullptr;
  int W = 0;
  std::lock_guard<std::mutex> guard(h->crt_mu);
  for (auto& e : h->crt_cache)
    if (e.first == key) {
      d_cst = e.second.first;
      W = e.second.second;
    }
  if (!d_cst) {
    std::vector<uint32_t> cst;
    W = crt_compose_constants(h->c, r.prime, r.n, cst);
    if (cudaMalloc(&d_cst, cst.size() * 4) != cudaSuccess ||
        cudaMemcpy(d_cst, cst.data(), cst.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
      set_error("crt_compose: constant upload failed");
      return TFHE_ECUDA;
    }
    h->crt_cache.push_back({key, {d_cst, W}});
  }
  return launch_crt_compose(h->c, rows, n, d_cst, W, r, out_f64, out_words,
                            out_words ? n_words : 0, (cudaStream_t)stream);
}

}  // extern "C"
