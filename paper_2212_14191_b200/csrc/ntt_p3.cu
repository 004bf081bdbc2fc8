// Three-factor tensor-core NTT / INTT for n = 2^16 ("p3" plan): two HBM passes,
// a quarter of the int8 tensor work of the 256 x 256 plan.
//
// The reference's 4-step identity (ntt.py:212-222, params.py:198-228) with
// n = n1 n2, n1 = 1024, n2 = 64, A[i1][i2] = a[64 i1 + i2]:
//   forward  out[1024 k2 + k1] = sum_i2 w^(k2 i2) psi^((2k1+1) i2) S[k1][i2],
//            S[k1][i2] = sum_i1 psi^(64 (2k1+1) i1) A[i1][i2]         (w = psi^2048)
//   inverse  out[1024 k2 + k1] = n^-1 sum_i2 psi^(-1024 (2 i2 + 1) k2) psi^(-(2 i2 + 1) k1) S'[k1][i2],
//            S'[k1][i2] = sum_i1 psi^(-128 k1 i1) A[i1][i2]
// and the 1024-point column transform S is itself split 32 x 32 on chip
// (i1 = 32 a1 + a2, k1 = b1 + 32 b2), the same way ntt_fused.cu splits n = 4096:
//   stage A  SA[b1][a2] = sum_a1 T[b1][a1] x[32 a1 + a2]     T = twisted 32-point DFT
//   inner    Q = SA .* H'                                    (inner Hadamard, twist divided out)
//   stage B  S[b1 + 32 b2] = sum_a2 T[b2][a2] Q[b1][a2]
// so every contraction is a K = 32 (column pass) or K = 64 (row pass) int8
// GEMM on the byte planes -- 32 N (32 + 32 + 64) int8 ops per limb-transform
// instead of 32 N (256 + 256).  All of it is exact modular arithmetic (every
// table carries R = 2^32 for one Montgomery fold), so the output equals the
// reference's bit for bit.
//
// Pass 1 (ntt_col_kernel): unit = 8 columns i2 of one member of one limb; the
//   32 KB tile [i1][8] arrives by TMA, producers byte-split it into the
//   MN-major operand of stage A (m = 8 a2 + t is contiguous for fixed a1: two
//   M = 128 tiles), stage A / inner Hadamard / stage B run on chip (stage B's
//   operand is written by the stage-A epilogue, rows m' = 32 t + b1), and the
//   stage-B epilogue applies the outer Hadamard and stores P^T[i2][k1]
//   (coalesced along k1).
// Pass 2 (ntt_row_kernel): unit = 128 rows k1 of one member; the tile
//   P^T[64][128] arrives by TMA (MN-major again: k1 contiguous for fixed i2),
//   one K = 64 contraction (N = 256: four accumulators x 64 outputs k2), and the
//   epilogue writes out[1024 k2 + k1] (coalesced along k1) through the same
//   fused modes as the other transforms (plain, ModDown/rescale, key-switch MAC).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <cuda.h>

#include "common.cuh"
#include "tfhe_internal.h"

namespace tfhe {

namespace {

constexpr int kPN = 1 << 16, kPn1 = 1024, kPn2 = 64;
constexpr int kPSbo = 144;                       // padded m-group stride (bank-conflict free)
constexpr int kPTile = 4 * 4 * 8 * kPSbo;        // one M = 128 x K = 32 operand, 4 planes (18 KB)
constexpr int kPRaw = 8192 * 4;                  // one unit's raw u32 tile (32 KB)
constexpr int kPThreads = 512;                   // column pass: 16 warps
constexpr int kRowThreads = 384;                 // row pass: 12 warps (3 producers, MMA, 8 epilogue)
constexpr int kPProdWarps = 3, kPMmaWarp = 3;
constexpr int kPItems = 22;                      // ceil(64 warp items / 3 producer warps)


// ---- pass 1 shared memory: T 16 KB | H block | raw 32 KB | A1 2 x (2 tiles) | A2 kA2Bufs x (2 tiles)
// H block words: beta[i2][b2] (column part of the outer Hadamard) | its Shoup |
// H'T[a2][36] (inner Hadamard, transposed) | its Shoup | c[i2][36] (row part of
// the outer Hadamard) [| its Shoup].  The stage-A epilogue reads H'T and c as
// 16-byte vectors (4 outputs b1 per load); the 36-word rows put the 4 (H'T) or
// 8 (c) rows one warp reads on disjoint banks.
//   TFHE_P3_CSHOUP = 1: c as a Shoup operand (3 fewer IMAD-pipe cycles per
//   output than Montgomery) -- its table only fits with one stage-B buffer.
#ifndef TFHE_P3_CSHOUP
#define TFHE_P3_CSHOUP 1
#endif
constexpr int kA2Bufs = TFHE_P3_CSHOUP ? 1 : 2;
constexpr int kHBeta = 0, kHBetaS = 64 * 32, kHIn = 2 * 64 * 32, kHInS = kHIn + 32 * 36,
              kHC = kHInS + 32 * 36, kHCS = kHC + 64 * 36,
              kHWords = kHC + (TFHE_P3_CSHOUP ? 2 : 1) * 64 * 36;
constexpr int kC1T = 16384, kC1H = kHWords * 4;
constexpr int kC1A = 2 * kPTile + 16;            // two M tiles (+16 B: tile 1 on other banks)
constexpr int kC1Smem = kC1T + kC1H + kPRaw + 2 * kC1A + kA2Bufs * kC1A + 32 * 8;
// ---- pass 2 shared memory: T2 64 KB | raw kRawSlots x 32 KB | A 2 x (2 K-steps)
#ifndef TFHE_P3_RAWSLOTS
#define TFHE_P3_RAWSLOTS 2
#endif
constexpr int kRawSlots = TFHE_P3_RAWSLOTS;
constexpr int kC2T = 65536;
// grouped key-switch row pass: warpgroup 0 (producers + MMA) gives registers to
// the two epilogue warpgroups (128 * 128 + 256 * 184 <= 384 * 168)
constexpr int kRowRegsLow = 128, kRowRegsEpi = 184;
constexpr int kC2A = 2 * kPTile;                 // K = 64: two K-steps of one M tile
#ifndef TFHE_P3_ABUFS
#define TFHE_P3_ABUFS 2
#endif
constexpr int kABufs = TFHE_P3_ABUFS;            // MMA operand buffers (1: room for a 3rd raw slot)
constexpr int kC2Smem = kC2T + kRawSlots * kPRaw + kABufs * kC2A + 64 * 8;

struct ColArgs {
  const uint8_t* tab;      // [prime] 16 KB: T (B operand, 4 planes x 128 rows x 32 K)
  const uint32_t* hin;     // unused
  const uint32_t* hout;    // [prime] H block (kHWords): beta, c R, H' and Shoup companions
  uint32_t* P;             // P^T workspace: [limb][member][i2][k1]
  const PrimeConst* pc;
  int batch, units;
  LimbMap map;
  unsigned long long* trace;   // TFHE_P3_TRACE builds only
  CUtensorMap tmap;        // input viewed as [rows * batch][1024 i1][64 i2], box {8, 256, 1}
};

struct RowArgs {
  const uint8_t* tab;      // [prime] 64 KB: T2 (B operand, 2 K-steps x 4 planes x 256 rows)
  uint32_t* out;
  const PrimeConst* pc;
  int batch, units;
  int S;                   // EPI_KS_ACC: slices per (target, member, row block) group, else 1;
                           // the P^T row of (slice s, limb l) is s * map.n + l
  int strided;             // group g of CTA c: c + k * gridDim.x (limb-synchronous CTAs)
  LimbMap map;             // in_row = P^T workspace row
  EpiArgs epi;
  CUtensorMap tmap;        // P^T viewed as [rows * batch * 64 i2][1024 k1], box {128, 64}
};

TFHE_DEV uint32_t fold4_m(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, const PrimeConst& pc) {
  const uint64_t v = (uint64_t)(c0 + (c1 << 8)) + ((uint64_t)(c2 + (c3 << 8)) << 16);
  const uint32_t m = (uint32_t)v * pc.qneg_inv;
  return (uint32_t)((v + (uint64_t)m * pc.q) >> 32);
}
TFHE_DEV uint32_t mont_l(uint32_t a, uint32_t b, const PrimeConst& pc) {
  const uint64_t v = (uint64_t)a * b;
  const uint32_t m = (uint32_t)v * pc.qneg_inv;
  return (uint32_t)((v + (uint64_t)m * pc.q) >> 32);
}
TFHE_DEV uint32_t corr_q(uint32_t t, uint32_t q) { return t >= q ? t - q : t; }
TFHE_DEV void planes4p(uint32_t v0, uint32_t v1, uint32_t v2, uint32_t v3, uint32_t (&w)[4]) {
  const uint32_t lo01 = __byte_perm(v0, v1, 0x5140), hi01 = __byte_perm(v0, v1, 0x7362);
  const uint32_t lo23 = __byte_perm(v2, v3, 0x5140), hi23 = __byte_perm(v2, v3, 0x7362);
  w[0] = __byte_perm(lo01, lo23, 0x5410);
  w[1] = __byte_perm(lo01, lo23, 0x7632);
  w[2] = __byte_perm(hi01, hi23, 0x5410);
  w[3] = __byte_perm(hi01, hi23, 0x7632);
}
// MN-major operand, M = 128 rows, K-step kc (32 k each), plane j, padded SBO:
// core matrices 16 m x 8 k, LBO (k groups) = 8 SBO, SBO (m groups)
TFHE_DEV uint32_t p_off(int kc, int j, int m, int k) {
  return (uint32_t)((kc * 4 + j) * (4 * 8 * kPSbo) + (k >> 3) * (8 * kPSbo) + (m >> 4) * kPSbo +
                    (k & 7) * 16 + (m & 15));
}

// timeline probes of the column pass (-DTFHE_P3_TRACE): per-unit event clocks
// of CTA 0, lane 0 of the first warp of each role; compiled out otherwise
#ifdef TFHE_P3_TRACE
constexpr int kPTraceN = 128;
#define PTRACE(ev, i)                                                                \
  do {                                                                               \
    if (blockIdx.x == 0 && lane == 0 && (i) < kPTraceN &&                            \
        (warp == 0 || warp == 3 || warp == 4 || warp == 12))                         \
      a.trace[(ev) * kPTraceN + (i)] = clock64();                                    \
  } while (0)
#else
#define PTRACE(ev, i) do { } while (0)
#endif

// ============================================================================ pass 1
template <bool INV>
__global__ void __launch_bounds__(kPThreads, 1) ntt_col_kernel(const __grid_constant__ ColArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sT = smem;
  uint32_t* sH = reinterpret_cast<uint32_t*>(smem + kC1T);
  uint8_t* sRaw = smem + kC1T + kC1H;
  uint8_t* sA1 = sRaw + kPRaw;                  // [2] buffers of two M tiles
  uint8_t* sA2 = sA1 + 2 * kC1A;                // [kA2Bufs] buffers (stage B operand)
  uint64_t* bar = reinterpret_cast<uint64_t*>(sA2 + kA2Bufs * kC1A);
  uint64_t* raw_full = bar + 0;
  uint64_t* raw_empty = bar + 1;
  uint64_t* a1_full = bar + 2;     // [2]
  uint64_t* a1_empty = bar + 4;    // [2]
  uint64_t* accA_full = bar + 6;
  uint64_t* accA_empty = bar + 7;
  uint64_t* accB_full = bar + 10;
  uint64_t* accB_empty = bar + 11;
  uint64_t* tw_full = bar + 12;
  uint64_t* tw_empty = bar + 13;
  uint64_t* epiA_done = bar + 14;
  uint64_t* epiB_done = bar + 15;
  uint64_t* a2_full = bar + 16;    // [2]
  uint64_t* a2_empty = bar + 18;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 20);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int u0 = (int)((long long)a.units * blockIdx.x / gridDim.x);
  const int cnt = (int)((long long)a.units * (blockIdx.x + 1) / gridDim.x) - u0;
  if (tid == 0) {
    mbar_init(raw_full, 1);
    mbar_init(raw_empty, 32 * kPProdWarps);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&a1_full[s], 32 * kPProdWarps);
      mbar_init(&a1_empty[s], 1);
    }
    mbar_init(accA_full, 1);
    mbar_init(accA_empty, 256);
    for (int s2 = 0; s2 < 2; ++s2) {
      mbar_init(&a2_full[s2], 256);
      mbar_init(&a2_empty[s2], 1);
    }
    mbar_init(accB_full, 1);
    mbar_init(accB_empty, 128);
    mbar_init(tw_full, 1);
    mbar_init(tw_empty, 1);
    mbar_init(epiA_done, 256);
    mbar_init(epiB_done, 128);
    fence_mbar_init();
  }
  if (warp == kPMmaWarp) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // unit = (limb, member, column block cb of 8): limb-major, then member, cb
  struct UPos {
    int limb, b, cb;
  };
  const int upl = a.batch * 8;
  const UPos p0 = {u0 / upl, (u0 % upl) >> 3, u0 & 7};
  auto adv = [&](UPos& p) {
    if (++p.cb == 8) {
      p.cb = 0;
      if (++p.b == a.batch) {
        p.b = 0;
        ++p.limb;
      }
    }
  };
  auto last_of_limb = [&](const UPos& p, int it) {
    return it + 1 == cnt || (p.cb == 7 && p.b + 1 == a.batch);
  };

  if (warp < kPProdWarps) {
    // -------------------------------------------------------------- producers
    auto issue_raw = [&](const UPos& p) {
      mbar_arrive_expect_tx(raw_full, kPRaw);
      const int row = a.map.in_row[p.limb] * a.batch + p.b;
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4)
        tma_load_3d(sRaw + c4 * 8192, &a.tmap, 8 * p.cb, 256 * c4, row, raw_full);
    };
    UPos pos = p0, ahead = p0;
    if (tid == 0 && cnt > 0) issue_raw(ahead);
    adv(ahead);
    // raw word (k = a1, m = 8 a2 + t) sits at 256 k + m.  64 warp items per
    // unit: (4 k rows, 32 m); lane -> (r = lane / 8, c = lane % 8)
    const int r = lane >> 3, c = lane & 7;
    int prev_limb = -1;
    uint32_t tw_ph = 0;
    for (int it = 0; it < cnt; ++it, adv(pos)) {
      const int limb = pos.limb;
      mbar_wait(raw_full, it & 1);
      PTRACE(0, it);
      uint4 x[kPItems];
#pragma unroll
      for (int k = 0; k < kPItems; ++k) {
        const int item = min(warp + kPProdWarps * k, 63);
        const int ib = item >> 3, jb = item & 7;
        x[k] = *reinterpret_cast<const uint4*>(sRaw + ((4 * ib + r) * 256 + 32 * jb + 4 * c) * 4);
      }
      fence_proxy_async_smem();   // raw reads before the next TMA write (see the row pass)
      mbar_arrive(raw_empty);
      if (tid == 0 && it + 1 < cnt) {
        mbar_wait(raw_empty, it & 1);
        issue_raw(ahead);
      }
      adv(ahead);
      if (limb != prev_limb) {
        if (tid == 0) {
          if (prev_limb >= 0) {
            mbar_wait(tw_empty, tw_ph);
            mbar_wait(epiA_done, tw_ph);
            mbar_wait(epiB_done, tw_ph);
          }
          const int pr = a.map.prime[limb];
          mbar_arrive_expect_tx(tw_full, kC1T + kC1H);
          bulk_g2s(sT, a.tab + (size_t)pr * kC1T, kC1T, tw_full);
          bulk_g2s(sH, a.hout + (size_t)pr * kHWords, kC1H, tw_full);
        }
        if (prev_limb >= 0) tw_ph ^= 1;
        prev_limb = limb;
      }
      const int buf = it & 1;
      if (it >= 2) mbar_wait(&a1_empty[buf], ((it >> 1) - 1) & 1);
      PTRACE(1, it);
      uint8_t* dst = sA1 + buf * kC1A;
#pragma unroll
      for (int k = 0; k < kPItems; ++k) {
        const int item = warp + kPProdWarps * k;
        if (item >= 64) break;
        const int ib = item >> 3, jb = item & 7;
        const int kk = 4 * ib + r, m = 32 * jb + 4 * c;
        uint32_t w[4];
        planes4p(x[k].x, x[k].y, x[k].z, x[k].w, w);
        uint8_t* t = dst + (m >> 7) * (kPTile + 16);
#pragma unroll
        for (int j = 0; j < 4; ++j) *reinterpret_cast<uint32_t*>(t + p_off(0, j, m & 127, kk)) = w[j];
      }
      fence_proxy_async_smem();
      mbar_arrive(&a1_full[buf]);
      PTRACE(2, it);
    }
  } else if (warp == kPMmaWarp) {
    // -------------------------------------------------------------- MMA issuer
    // per M tile and plane j one MMA, N = 128 = the four output-byte tiles of T
    // (rows 32 i + c) landing in accumulators C_0..C_3 (TMEM columns 32 i + c)
    constexpr uint32_t idesc = idesc_i8(128, 128) | (1u << 15);   // A MN-major
    const uint32_t sT_u = smem_u32(sT);
    auto issue = [&](uint32_t a_base, uint32_t d) {
#pragma unroll
      for (int tile = 0; tile < 2; ++tile)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint64_t ad = smem_desc_kmajor(a_base + tile * (kPTile + 16) + j * (4 * 8 * kPSbo),
                                               8 * kPSbo, kPSbo);
          const uint64_t bd = smem_desc_kmajor(sT_u + j * 4096, 2048, 128);
          mma_i8_ss(d + tile * 128, ad, bd, idesc, j != 0);
        }
    };
    UPos pos2 = p0;
    auto stageB = [&](int v) {
      const int b2f = v % kA2Bufs;
      mbar_wait(&a2_full[b2f], (v / kA2Bufs) & 1);
      PTRACE(4, v);
      if (v >= 1) mbar_wait(accB_empty, (v - 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        issue(smem_u32(sA2 + b2f * kC1A), tmem + 256);
        PTRACE(5, v);
        mma_commit(&a2_empty[b2f]);
        mma_commit(accB_full);
        if (last_of_limb(pos2, v)) mma_commit(tw_empty);
      }
      __syncwarp();
      adv(pos2);
    };
    int prev_limb = -1;
    uint32_t tw_ph = 0;
    int sB = 0;
    UPos pos = p0;
    for (int it = 0; it < cnt; ++it, adv(pos)) {
      if (pos.limb != prev_limb) {
        while (sB < it) stageB(sB++);
        if (prev_limb >= 0) tw_ph ^= 1;
        mbar_wait(tw_full, tw_ph);
        prev_limb = pos.limb;
      }
      const int buf = it & 1;
      mbar_wait(&a1_full[buf], (it >> 1) & 1);
      if (it >= 1) mbar_wait(accA_empty, (it - 1) & 1);
      PTRACE(11, it);
      tc_fence_after();
      if (elect_one()) {
        issue(smem_u32(sA1 + buf * kC1A), tmem);
        PTRACE(3, it);
        mma_commit(&a1_empty[buf]);
        mma_commit(accA_full);
      }
      __syncwarp();
      while (sB < it) stageB(sB++);
    }
    while (sB < cnt) stageB(sB++);
  } else if (warp < 12) {
    // -------------------------------------------------------------- stage-A epilogue
    // warp -> (lane quarter q, M tile tau): row m = 128 tau + 32 q + lane
    // = (a2 = m / 8, column t = m % 8); its 32 outputs b1 fold, take the inner
    // Hadamard and land in stage B's operand (rows m' = 32 t + b1, k = a2)
    const int q = warp & 3, tau = (warp - 4) >> 2;
    const int m = 128 * tau + 32 * q + lane, a2 = m >> 3, t = m & 7;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    uint8_t* a2t0 = sA2 + (t >> 2) * (kPTile + 16);  // stage-B tile of this column (buffer 0)
    const int mb = 32 * (t & 3);                      // its rows m' = mb + b1
    int prev_limb = -1;
    uint32_t tw_ph = 0;
    UPos pos = p0;
    for (int it = 0; it < cnt; ++it, adv(pos)) {
      if (pos.limb != prev_limb) {
        if (prev_limb >= 0) tw_ph ^= 1;
        mbar_wait(tw_full, tw_ph);   // this limb's tables (the column twist for epi B)
        prev_limb = pos.limb;
      }
      const int pr = a.map.prime[pos.limb];
      const PrimeConst pc = a.pc[pr];
      // the inner Hadamard H'[b1][a2] and the row part c[i2 = 8 cb + t][b1] of
      // the outer Hadamard, 4 consecutive b1 per vector load
      const uint32_t* hrow = sH + kHIn + a2 * 36;
      const uint32_t* hrows = sH + kHInS + a2 * 36;
      const uint32_t* crow = sH + kHC + (8 * pos.cb + t) * 36;
      const uint32_t* crows = sH + kHCS + (8 * pos.cb + t) * 36;
      (void)crows;
      mbar_wait(accA_full, it & 1);
      PTRACE(6, it);
      tc_fence_after();
#pragma unroll 1
      for (int g = 0; g < 2; ++g) {
        uint32_t acc[4][16];
#pragma unroll
        for (int i = 0; i < 4; ++i) tmem_ld16(tmem + lane_off + tau * 128 + i * 32 + 16 * g, acc[i]);
        tmem_ld_wait();
        if (g == 1) {
          tc_fence_before();
          mbar_arrive(accA_empty);
        }
        uint32_t p[16];
#pragma unroll
        for (int e4 = 0; e4 < 4; ++e4) {
          const int b1 = 16 * g + 4 * e4;
          const uint4 hv = *reinterpret_cast<const uint4*>(hrow + b1);
          const uint4 hs = *reinterpret_cast<const uint4*>(hrows + b1);
          const uint4 cv = *reinterpret_cast<const uint4*>(crow + b1);
          const uint32_t hva[4] = {hv.x, hv.y, hv.z, hv.w}, hsa[4] = {hs.x, hs.y, hs.z, hs.w};
          const uint32_t cva[4] = {cv.x, cv.y, cv.z, cv.w};
#if TFHE_P3_CSHOUP
          const uint4 cs = *reinterpret_cast<const uint4*>(crows + b1);
          const uint32_t csa[4] = {cs.x, cs.y, cs.z, cs.w};
#endif
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int e = 4 * e4 + u;
            const uint32_t s = fold4_m(acc[0][e], acc[1][e], acc[2][e], acc[3][e], pc);
            const uint32_t sh = mul_shoup_lazy(s, hva[u], hsa[u], pc.q);   // S H', [0, 2q)
#if TFHE_P3_CSHOUP
            p[e] = mul_shoup_lazy(sh, cva[u], csa[u], pc.q);               // c: Shoup
#else
            p[e] = mont_l(sh, cva[u], pc);                                 // c: Montgomery (c R)
#endif
          }
        }
        uint32_t pl[4][4];
#pragma unroll
        for (int e4 = 0; e4 < 4; ++e4) {
          uint32_t w[4];
          planes4p(p[4 * e4], p[4 * e4 + 1], p[4 * e4 + 2], p[4 * e4 + 3], w);
#pragma unroll
          for (int j = 0; j < 4; ++j) pl[j][e4] = w[j];
        }
        if (g == 0 && it >= kA2Bufs) mbar_wait(&a2_empty[it % kA2Bufs], ((it / kA2Bufs) - 1) & 1);
        if (g == 0) PTRACE(7, it);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          *reinterpret_cast<uint4*>(a2t0 + (it % kA2Bufs) * kC1A + p_off(0, j, mb + 16 * g, a2)) =
              make_uint4(pl[j][0], pl[j][1], pl[j][2], pl[j][3]);
      }
      fence_proxy_async_smem();
      mbar_arrive(&a2_full[it % kA2Bufs]);
      PTRACE(8, it);
      if (last_of_limb(pos, it)) mbar_arrive(epiA_done);
    }
  } else {
    // -------------------------------------------------------------- stage-B epilogue
    // warp -> lane quarter q; in M tile tau' its row m' = 32 q + lane is
    // (column t = 4 tau' + q, b1 = lane); outputs k1 = b1 + 32 b2 take the
    // column part beta[i2][b2] of the outer Hadamard (broadcast shared-memory
    // reads; the row part rode in with the inner Hadamard) and go to
    // P^T[i2 = 8 cb + t][k1] (coalesced along b1)
    const int q = warp & 3;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    int prev_limb = -1;
    uint32_t tw_ph = 0;
    UPos pos = p0;
    for (int it = 0; it < cnt; ++it, adv(pos)) {
      if (pos.limb != prev_limb) {
        if (prev_limb >= 0) tw_ph ^= 1;
        mbar_wait(tw_full, tw_ph);   // this limb's beta
        prev_limb = pos.limb;
      }
      const int pr = a.map.prime[pos.limb];
      const PrimeConst pc = a.pc[pr];
      mbar_wait(accB_full, it & 1);
      PTRACE(9, it);
      tc_fence_after();
      uint32_t y[2][32];
#pragma unroll
      for (int tile = 0; tile < 2; ++tile)
#pragma unroll
        for (int cc = 0; cc < 32; cc += 8) {
          uint32_t acc[4][8];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            tmem_ld8(tmem + 256 + lane_off + tile * 128 + i * 32 + cc, acc[i]);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 8; ++e)
            y[tile][cc + e] = fold4_m(acc[0][e], acc[1][e], acc[2][e], acc[3][e], pc);
        }
      tc_fence_before();
      mbar_arrive(accB_empty);
#pragma unroll
      for (int tile = 0; tile < 2; ++tile) {
        const int i2 = 8 * pos.cb + 4 * tile + q;
        const uint32_t* bt = sH + kHBeta + i2 * 32;
        const uint32_t* bts = sH + kHBetaS + i2 * 32;
        uint32_t* o = a.P + (((size_t)a.map.out_row[pos.limb] * a.batch + pos.b) * kPn2 + i2) * kPn1 +
                      lane;
#pragma unroll
        for (int b4 = 0; b4 < 8; ++b4) {
          // lazy Shoup products: P^T in [0, 2q) (the row pass only byte-splits it)
          const uint4 bv = *reinterpret_cast<const uint4*>(bt + 4 * b4);
          const uint4 bs = *reinterpret_cast<const uint4*>(bts + 4 * b4);
          o[32 * (4 * b4)] = mul_shoup_lazy(y[tile][4 * b4], bv.x, bs.x, pc.q);
          o[32 * (4 * b4 + 1)] = mul_shoup_lazy(y[tile][4 * b4 + 1], bv.y, bs.y, pc.q);
          o[32 * (4 * b4 + 2)] = mul_shoup_lazy(y[tile][4 * b4 + 2], bv.z, bs.z, pc.q);
          o[32 * (4 * b4 + 3)] = mul_shoup_lazy(y[tile][4 * b4 + 3], bv.w, bs.w, pc.q);
        }
      }
      PTRACE(10, it);
      if (last_of_limb(pos, it)) mbar_arrive(epiB_done);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kPMmaWarp) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ============================================================================ pass 2
template <int MODE>
__global__ void __launch_bounds__(kRowThreads, 1) ntt_row_kernel(const __grid_constant__ RowArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sT = smem;
  uint8_t* sRaw = smem + kC2T;                  // [kRawSlots] raw tiles (TMA ring)
  uint8_t* sA = sRaw + kRawSlots * kPRaw;        // [kABufs] buffers of two K-steps
  uint64_t* bar = reinterpret_cast<uint64_t*>(sA + kABufs * kC2A);
  uint64_t* a_full = bar + 2;      // [kABufs]
  uint64_t* a_empty = bar + 4;     // [kABufs]
  uint64_t* acc_full = bar + 6;    // [2]
  uint64_t* acc_empty = bar + 8;   // [2]
  uint64_t* tw_full = bar + 10;
  uint64_t* tw_empty = bar + 11;
  uint64_t* raw_full = bar + 12;              // [kRawSlots]
  uint64_t* raw_empty = raw_full + kRawSlots;  // [kRawSlots]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(raw_empty + kRawSlots);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // a.units counts slice groups (S units each); whole groups per CTA, either a
  // contiguous range or (a.strided) groups blockIdx.x + k * gridDim.x, so that
  // all CTAs work on the same limb at a time and its per-limb epilogue operand
  // (the switching-key rows, shared by every member) stays L2-resident
  const int gstep = a.strided ? (int)gridDim.x : 1;
  const int gb = a.strided ? (int)blockIdx.x : (int)((long long)a.units * blockIdx.x / gridDim.x);
  const int ng = a.strided ? (a.units - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x
                           : (int)((long long)a.units * (blockIdx.x + 1) / gridDim.x) - gb;
  const int cnt = ng * a.S;
  if (tid == 0) {
    for (int s = 0; s < kRawSlots; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&raw_empty[s], 32 * kPProdWarps);
    }
    for (int s = 0; s < 2; ++s) {
      if (s < kABufs) {
        mbar_init(&a_full[s], 32 * kPProdWarps);
        mbar_init(&a_empty[s], 1);
      }
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 256);
    }
    mbar_init(tw_full, 1);
    mbar_init(tw_empty, 1);
    fence_mbar_init();
  }
  if (warp == kPMmaWarp) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // unit = (limb, member, row block kb of 128 k1, slice sl): sl fastest (S = 1
  // unless the grouped key-switch epilogue sums S slices per output)
  struct UPos {
    int limb, b, kb, sl, g;
  };
  const int S = a.S;
  const int upl = a.batch * 8;
  const UPos p0 = {gb / upl, (gb % upl) >> 3, gb & 7, 0, gb};
  auto adv = [&](UPos& p) {
    if (++p.sl < S) return;
    p.sl = 0;
    p.g += gstep;
    p.limb = p.g / upl;
    p.b = (p.g % upl) >> 3;
    p.kb = p.g & 7;
  };
  auto last_of_limb = [&](const UPos& p, int it) {
    return it + 1 == cnt || (p.sl + 1 == S && (p.g + gstep) / upl != p.limb);
  };

  if (warp < kPProdWarps) {
    if (MODE == EPI_KS_ACC) reg_dealloc<kRowRegsLow>();
    // -------------------------------------------------------------- producers
    auto issue_raw = [&](const UPos& p, int slot) {
      mbar_arrive_expect_tx(&raw_full[slot], kPRaw);
      const int prow = MODE == EPI_KS_ACC ? p.sl * a.map.n + p.limb : a.map.in_row[p.limb];
      const int row = (prow * a.batch + p.b) * kPn2;
      tma_load_2d(sRaw + slot * kPRaw, &a.tmap, 128 * p.kb, row, &raw_full[slot]);
    };
    UPos pos = p0, ahead = p0;   // kRawSlots raw tiles in flight: ahead = unit it + kRawSlots
    for (int s = 0; s < kRawSlots; ++s) {
      if (tid == 0 && s < cnt) issue_raw(ahead, s);
      adv(ahead);
    }
    // raw word (k = i2, m = k1 local) at 128 k + m; 64 warp items (4 k rows, 32 m)
    const int r = lane >> 3, c = lane & 7;
    int prev_limb = -1;
    uint32_t tw_ph = 0;
    for (int it = 0; it < cnt; ++it, adv(pos)) {
      const int limb = pos.limb;
      const int slot = it % kRawSlots;
      mbar_wait(&raw_full[slot], (it / kRawSlots) & 1);
      uint4 x[kPItems];
      const uint8_t* raw = sRaw + slot * kPRaw;
#pragma unroll
      for (int k = 0; k < kPItems; ++k) {
        const int item = min(warp + kPProdWarps * k, 63);
        const int ib = item >> 2, jb = item & 3;
        x[k] = *reinterpret_cast<const uint4*>(raw + ((4 * ib + r) * 128 + 32 * jb + 4 * c) * 4);
      }
      // the generic-proxy reads of the raw tile must be ordered before the
      // next TMA (async-proxy) write into it: without this fence the refill
      // was observed to land under still-pending reads
      fence_proxy_async_smem();
      mbar_arrive(&raw_empty[slot]);
      if (tid == 0 && it + kRawSlots < cnt) {
        mbar_wait(&raw_empty[slot], (it / kRawSlots) & 1);
        issue_raw(ahead, slot);
      }
      adv(ahead);
      if (limb != prev_limb) {
        if (tid == 0) {
          if (prev_limb >= 0) mbar_wait(tw_empty, tw_ph);
          mbar_arrive_expect_tx(tw_full, kC2T);
          bulk_g2s(sT, a.tab + (size_t)a.map.prime[limb] * kC2T, kC2T, tw_full);
        }
        if (prev_limb >= 0) tw_ph ^= 1;
        prev_limb = limb;
      }
      const int abuf = it % kABufs;
      if (it >= kABufs) mbar_wait(&a_empty[abuf], ((it / kABufs) - 1) & 1);
      uint8_t* dst = sA + abuf * kC2A;
#pragma unroll
      for (int k = 0; k < kPItems; ++k) {
        const int item = warp + kPProdWarps * k;
        if (item >= 64) break;
        const int ib = item >> 2, jb = item & 3;
        const int kk = 4 * ib + r, m = 32 * jb + 4 * c;
        uint32_t w[4];
        planes4p(x[k].x, x[k].y, x[k].z, x[k].w, w);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          *reinterpret_cast<uint32_t*>(dst + p_off(kk >> 5, j, m, kk & 31)) = w[j];
      }
      fence_proxy_async_smem();
      mbar_arrive(&a_full[abuf]);
    }
  } else if (warp == kPMmaWarp) {
    if (MODE == EPI_KS_ACC) reg_dealloc<kRowRegsLow>();
    // -------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = idesc_i8(128, 256) | (1u << 15);   // A MN-major
    const uint32_t sT_u = smem_u32(sT);
    int prev_limb = -1;
    uint32_t tw_ph = 0;
    UPos pos = p0;
    for (int it = 0; it < cnt; ++it, adv(pos)) {
      if (pos.limb != prev_limb) {
        if (prev_limb >= 0) tw_ph ^= 1;
        mbar_wait(tw_full, tw_ph);
        prev_limb = pos.limb;
      }
      const int buf = it & 1, abuf = it % kABufs;
      mbar_wait(&a_full[abuf], (it / kABufs) & 1);
      if (it >= 2) mbar_wait(&acc_empty[buf], ((it >> 1) - 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t ab = smem_u32(sA + abuf * kC2A);
#pragma unroll
        for (int kc = 0; kc < 2; ++kc)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint64_t ad = smem_desc_kmajor(ab + (kc * 4 + j) * (4 * 8 * kPSbo), 8 * kPSbo, kPSbo);
            const uint64_t bd = smem_desc_kmajor(sT_u + (kc * 4 + j) * 8192, 4096, 128);
            mma_i8_ss(tmem + buf * 256, ad, bd, idesc, (kc | j) != 0);
          }
        mma_commit(&a_empty[abuf]);
        mma_commit(&acc_full[buf]);
        if (last_of_limb(pos, it)) mma_commit(tw_empty);
      }
      __syncwarp();
    }
  } else if (MODE == EPI_KS_ACC && warp < 12) {
    reg_alloc<kRowRegsEpi>();
    // -------------------------------------------------- grouped key-switch epilogue
    // warp -> (lane quarter q, column half h) as below.  y arrives as y R (the
    // table carries R^2); the S slices of a (target, member, row block) sum in
    // registers (lazy in [0, 2q) for q < 2^30), the accumulator row is read at
    // the group's start (init_acc, L2-prefetched one group ahead) and written
    // once at its end; a slice's own target row is skipped (reused unchanged,
    // ckks.py:361-364).  Fold and MAC run per 8-column chunk while the TMEM
    // buffer is held, so the key rows stream through a 3-chunk register ring
    // two chunks ahead -- across unit boundaries -- and their L2 latency hides
    // behind two chunks of fold / MAC work.
    const int q = warp & 3, h = (warp - 4) >> 2;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const size_t half = (size_t)a.epi.key_pair / 2;
    auto key_ptr = [&](const UPos& p) -> const uint32_t* {
      if (a.epi.j0 + p.sl == a.epi.js[p.limb]) return nullptr;
      const size_t p0_ = (size_t)32 * h * kPn1 + 128 * p.kb + 32 * q + lane;
      return a.epi.key + (size_t)(a.epi.j0 + p.sl) * a.epi.key_pair +
             (size_t)a.epi.key_row[p.limb] * kPN + p0_;
    };
    auto acc_row = [&](const UPos& p) -> size_t {
      return ((size_t)a.map.out_row[p.limb] * a.batch + p.b) * kPN + (size_t)32 * h * kPn1 +
             128 * p.kb + 32 * q + lane;
    };
    uint32_t sb[32], sa[32];
    // key ring: chunk ch of a unit lives in buffer ch % kKR; after its MAC the
    // buffer is refilled with chunk ch + kKR (this unit's, else the next
    // unit's) -- kKR chunks of lookahead, static register indices (the ring
    // period divides the chunks per unit, so no register rotation is needed)
    constexpr int kKC = 8, kKR = 4, kCPU = 32 / kKC;
    static_assert(kCPU % kKR == 0, "ring period must divide the chunks per unit");
    uint32_t kb[kKR][kKC], ka[kKR][kKC];
    auto load_keys = [&](const uint32_t* kp, int ch, uint32_t (&b)[kKC], uint32_t (&c)[kKC]) {
      if (kp) {
#pragma unroll
        for (int e = 0; e < kKC; ++e) {
          b[e] = __ldg(kp + (kKC * ch + e) * kPn1);
          c[e] = __ldg(kp + half + (kKC * ch + e) * kPn1);
        }
      }
    };
    UPos pos = p0;
    const uint32_t* kp_cur = cnt > 0 ? key_ptr(p0) : nullptr;
    const uint32_t* kp_nxt = nullptr;
#pragma unroll
    for (int r = 0; r < kKR; ++r) load_keys(kp_cur, r, kb[r], ka[r]);
    for (int it = 0; it < cnt; ++it, adv(pos)) {
      const int limb = pos.limb;
      const PrimeConst pc = a.pc[a.map.prime[limb]];
      const int buf = it & 1;
      const size_t arow = acc_row(pos);
      if (pos.sl == 0) {
        if (a.epi.init_acc[limb]) {
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            sb[e] = a.epi.acc_b[arow + (size_t)e * kPn1];
            sa[e] = a.epi.acc_a[arow + (size_t)e * kPn1];
          }
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) sb[e] = sa[e] = 0;
        }
        // the next group's accumulator rows: HBM -> L2 while this group runs
        if (it + S < cnt) {
          UPos ng = pos;
          for (int k = 0; k < S; ++k) adv(ng);
          if (a.epi.init_acc[ng.limb]) {
            const size_t nrow = acc_row(ng);
#pragma unroll 4
            for (int e = 0; e < 32; ++e) {
              prefetch_l2(a.epi.acc_b + nrow + (size_t)e * kPn1);
              prefetch_l2(a.epi.acc_a + nrow + (size_t)e * kPn1);
            }
          }
        }
      }
      kp_nxt = nullptr;
      if (it + 1 < cnt) {
        UPos nx = pos;
        adv(nx);
        kp_nxt = key_ptr(nx);
      }
      const bool lazy = pc.q < (1u << 30);   // warp-uniform: one prime per unit
      const uint32_t q2 = 2 * pc.q;
      mbar_wait(&acc_full[buf], (it >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int ch = 0; ch < kCPU; ++ch) {
        const int rb = ch % kKR;
        uint32_t y[kKC];
#pragma unroll
        for (int hf = 0; hf < kKC / 4; ++hf) {
          uint32_t acc[4][4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            tmem_ld4(tmem + buf * 256 + lane_off + i * 64 + 32 * h + kKC * ch + 4 * hf, acc[i]);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 4; ++e)
            y[4 * hf + e] = fold4_m(acc[0][e], acc[1][e], acc[2][e], acc[3][e], pc);
        }
        if (ch == kCPU - 1) {
          tc_fence_before();
          mbar_arrive(&acc_empty[buf]);
        }
        if (kp_cur) {
          if (lazy) {
#pragma unroll
            for (int e = 0; e < kKC; ++e) {
              const uint32_t tb = sb[kKC * ch + e] + mont_l(y[e], kb[rb][e], pc);
              const uint32_t ta = sa[kKC * ch + e] + mont_l(y[e], ka[rb][e], pc);
              sb[kKC * ch + e] = min(tb, tb - q2);
              sa[kKC * ch + e] = min(ta, ta - q2);
            }
          } else {
#pragma unroll
            for (int e = 0; e < kKC; ++e) {
              sb[kKC * ch + e] =
                  add_mod(sb[kKC * ch + e], corr_q(mont_l(y[e], kb[rb][e], pc), pc.q), pc.q);
              sa[kKC * ch + e] =
                  add_mod(sa[kKC * ch + e], corr_q(mont_l(y[e], ka[rb][e], pc), pc.q), pc.q);
            }
          }
        }
        // refill: chunk ch + kKR of this unit, or chunk ch + kKR - kCPU of the next
        if (ch + kKR < kCPU) load_keys(kp_cur, ch + kKR, kb[rb], ka[rb]);
        else load_keys(kp_nxt, ch + kKR - kCPU, kb[rb], ka[rb]);
      }
      if (pos.sl + 1 == S) {
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          a.epi.acc_b[arow + (size_t)e * kPn1] = corr_q(sb[e], pc.q);   // [0, 2q) -> [0, q)
          a.epi.acc_a[arow + (size_t)e * kPn1] = corr_q(sa[e], pc.q);
        }
      }
      kp_cur = kp_nxt;
    }
  } else if (MODE != EPI_KS_ACC && warp < 12) {
    // -------------------------------------------------------------- epilogue
    // warp -> (lane quarter q, column half h): row k1 = 128 kb + 32 q + lane,
    // columns k2 in [32 h, 32 h + 32); fold all 32 first, release the
    // accumulator buffer, then the epilogue mode; out[1024 k2 + k1]
    const int q = warp & 3, h = (warp - 4) >> 2;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    uint32_t sb[MODE == EPI_KS_ACC ? 32 : 1], sa[MODE == EPI_KS_ACC ? 32 : 1];   // group sums
    UPos pos = p0;
    for (int it = 0; it < cnt; ++it, adv(pos)) {
      const int limb = pos.limb;
      const PrimeConst pc = a.pc[a.map.prime[limb]];
      const int buf = it & 1;
      const int k1 = 128 * pos.kb + 32 * q + lane;
      const size_t pos0 = (size_t)32 * h * kPn1 + k1;   // the warp's first output position
      const size_t orow = ((size_t)a.map.out_row[limb] * a.batch + pos.b) * kPN + pos0;
      if (MODE == EPI_SUB_SCALE && it + 1 < cnt) {
        // the next unit's x / base rows (HBM) -> L2 while this unit runs
        UPos nx = pos;
        adv(nx);
        const size_t np0 = (size_t)32 * h * kPn1 + 128 * nx.kb + 32 * q + lane;
        const uint32_t* nxs = a.epi.x + ((size_t)a.epi.x_row[nx.limb] * a.batch + nx.b) * kPN + np0;
        const int nbr = a.epi.base_row[nx.limb];
        const uint32_t* nbs =
            nbr >= 0 ? a.epi.base + ((size_t)nbr * a.batch + nx.b) * kPN + np0 : nullptr;
#pragma unroll 4
        for (int e = 0; e < 32; ++e) {
          prefetch_l2(nxs + (size_t)e * kPn1);
          if (nbs) prefetch_l2(nbs + (size_t)e * kPn1);
        }
      }
      // EPI_KS_ACC: this slice's key rows (none for the slice's own target row);
      // the first 8 columns are requested before the accumulator wait and each
      // later chunk one chunk ahead, so the L2 latency overlaps the fold / MAC
      const bool use_key = MODE == EPI_KS_ACC && a.epi.j0 + pos.sl != a.epi.js[limb];
      const uint32_t* kbp = nullptr;
      uint32_t kbv[2][8], kav[2][8];
      if (use_key) {
        kbp = a.epi.key + (size_t)(a.epi.j0 + pos.sl) * a.epi.key_pair +
              (size_t)a.epi.key_row[limb] * kPN + pos0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          kbv[0][e] = __ldg(kbp + e * kPn1);
          kav[0][e] = __ldg(kbp + a.epi.key_pair / 2 + e * kPn1);
        }
      }
      if (MODE == EPI_KS_ACC && pos.sl == 0) {
        // a group's first slice: its accumulator rows (or zero), requested before
        // the accumulator wait too (the previous group's sums are already stored)
        if (a.epi.init_acc[limb]) {
          const size_t arow = ((size_t)a.map.out_row[limb] * a.batch + pos.b) * kPN + pos0;
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            sb[e] = a.epi.acc_b[arow + (size_t)e * kPn1];
            sa[e] = a.epi.acc_a[arow + (size_t)e * kPn1];
          }
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) sb[e] = sa[e] = 0;
        }
      }
      mbar_wait(&acc_full[buf], (it >> 1) & 1);
      tc_fence_after();
      uint32_t y[32];
#pragma unroll
      for (int cc = 0; cc < 32; cc += 8) {
        uint32_t acc[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          tmem_ld8(tmem + buf * 256 + lane_off + i * 64 + 32 * h + cc, acc[i]);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 8; ++e)
          y[cc + e] = MODE == EPI_KS_ACC   // the grouped key switch takes y lazy in [0, 2q)
                          ? fold4_m(acc[0][e], acc[1][e], acc[2][e], acc[3][e], pc)
                          : corr_q(fold4_m(acc[0][e], acc[1][e], acc[2][e], acc[3][e], pc), pc.q);
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[buf]);
      if (MODE == EPI_STORE) {
        if (a.epi.scatter_t) {
          // hoisted HROTATE: the INTT output lands permuted by x -> x^t
          // (kernels.py:97-107); coefficient i goes to t i mod 2n, negated past n
          uint32_t* o = a.out + ((size_t)a.map.out_row[limb] * a.batch + pos.b) * kPN;
          const uint32_t tt = a.epi.scatter_t;
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const uint32_t j = (tt * (uint32_t)(pos0 + (size_t)e * kPn1)) & (2 * kPN - 1);
            o[j & (kPN - 1)] = j >= (uint32_t)kPN ? (y[e] ? pc.q - y[e] : 0u) : y[e];
          }
        } else {
          uint32_t* o = a.out + orow;
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e * kPn1] = y[e];
        }
      } else if (MODE == EPI_SUB_SCALE) {
        const uint32_t* xs = a.epi.x + ((size_t)a.epi.x_row[limb] * a.batch + pos.b) * kPN + pos0;
        const int br = a.epi.base_row[limb];
        const uint32_t* bs =
            br >= 0 ? a.epi.base + ((size_t)br * a.batch + pos.b) * kPN + pos0 : nullptr;
        const uint32_t ss = a.epi.s[limb], ssp = a.epi.s_shoup[limb];
        uint32_t* o = a.out + orow;
#pragma unroll
        for (int cc = 0; cc < 32; cc += 8) {
          uint32_t xv[8], bv[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            xv[e] = xs[(cc + e) * kPn1];
            if (bs) bv[e] = bs[(cc + e) * kPn1];
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            uint32_t t = mul_shoup(sub_mod(xv[e], y[cc + e], pc.q), ss, ssp, pc.q);
            if (bs) t = add_mod(bv[e], t, pc.q);
            o[(cc + e) * kPn1] = t;
          }
        }
      } else if (MODE == EPI_KS_ACC) {
        // y arrives as y R (the table carries R^2); the S slices of this
        // (target, member, row block) sum in registers, the accumulator row is
        // read at the group's start (init_acc) and written once at its end.
        // A slice's own target row is skipped (reused unchanged, ckks.py:361-364).
        const size_t arow = ((size_t)a.map.out_row[limb] * a.batch + pos.b) * kPN + pos0;
        const bool lazy = pc.q < (1u << 30);   // warp-uniform: one prime per unit
        const uint32_t q2 = 2 * pc.q;
        if (use_key) {
          const uint32_t* kap = kbp + a.epi.key_pair / 2;
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            const int cur = ch & 1, cc = 8 * ch;
            if (ch < 3) {
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                kbv[cur ^ 1][e] = __ldg(kbp + (cc + 8 + e) * kPn1);
                kav[cur ^ 1][e] = __ldg(kap + (cc + 8 + e) * kPn1);
              }
            }
            if (lazy) {
              // q < 2^30: the sums stay in [0, 2q) (< 2^31), one unsigned min per add
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const uint32_t tb = sb[cc + e] + mont_l(y[cc + e], kbv[cur][e], pc);
                const uint32_t ta = sa[cc + e] + mont_l(y[cc + e], kav[cur][e], pc);
                sb[cc + e] = min(tb, tb - q2);
                sa[cc + e] = min(ta, ta - q2);
              }
            } else {
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                sb[cc + e] = add_mod(sb[cc + e], corr_q(mont_l(y[cc + e], kbv[cur][e], pc), pc.q), pc.q);
                sa[cc + e] = add_mod(sa[cc + e], corr_q(mont_l(y[cc + e], kav[cur][e], pc), pc.q), pc.q);
              }
            }
          }
        }
        if (pos.sl + 1 == S) {
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            a.epi.acc_b[arow + (size_t)e * kPn1] = corr_q(sb[e], pc.q);   // [0, 2q) -> [0, q)
            a.epi.acc_a[arow + (size_t)e * kPn1] = corr_q(sa[e], pc.q);
          }
        }
      } else {   // EPI_KS_MAC: y arrives as y R (the table carries R^2)
        const size_t kr = (size_t)a.epi.key_row[limb] * kPN + pos0;
        uint32_t* ob = a.epi.acc_b + orow;
        uint32_t* oa = a.epi.acc_a + orow;
        const bool first = a.epi.first != 0;
#pragma unroll
        for (int cc = 0; cc < 32; cc += 8) {
          uint32_t kb[8], ka[8], pb[8], pa[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            kb[e] = __ldg(a.epi.kb + kr + (cc + e) * kPn1);
            ka[e] = __ldg(a.epi.ka + kr + (cc + e) * kPn1);
            if (!first) {
              pb[e] = ob[(cc + e) * kPn1];
              pa[e] = oa[(cc + e) * kPn1];
            }
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const uint32_t tb = corr_q(mont_l(y[cc + e], kb[e], pc), pc.q);
            const uint32_t ta = corr_q(mont_l(y[cc + e], ka[e], pc), pc.q);
            ob[(cc + e) * kPn1] = first ? tb : add_mod(pb[e], tb, pc.q);
            oa[(cc + e) * kPn1] = first ? ta : add_mod(pa[e], ta, pc.q);
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kPMmaWarp) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ============================================================================ host
uint32_t mulmod_p(uint64_t a, uint64_t b, uint32_t q) { return (uint32_t)(a * b % q); }
uint32_t powmod_p(uint64_t b, uint64_t e, uint32_t q) {
  uint64_t r = 1 % q, x = b % q;
  while (e) {
    if (e & 1) r = r * x % q;
    x = x * x % q;
    e >>= 1;
  }
  return (uint32_t)r;
}

typedef CUresult (*EncodeTiledFnP)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFnP encode_p() {
  static EncodeTiledFnP fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) ==
            cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFnP>(p);
  }
  return fn;
}

int max_row(const LimbMap& m) {
  int r = 0;
  for (int l = 0; l < m.n; ++l) r = std::max(r, (int)m.in_row[l]);
  return r + 1;
}

// B-operand byte tiles of an ntw x ntw table T[c][k] (values carry R), K-steps of
// 32, N = 4 ntw rows n = ntw i + c (output byte i of 2^(8j) T):  tile (kc, j)
template <class F>
void pack_tiles(uint8_t* base, int ntw, uint32_t q, F T) {
  const int nrows = 4 * ntw, tile = nrows * 32;
  for (int cc = 0; cc < ntw; ++cc)
    for (int k = 0; k < ntw; ++k) {
      const uint32_t t = T(cc, k);
      const int kc = k / 32, kr = k % 32;
      for (int j = 0; j < 4; ++j) {
        const uint32_t vj = mulmod_p(t, 1ull << (8 * j), q);
        for (int i = 0; i < 4; ++i) {
          const int nr = ntw * i + cc;
          const size_t off = ((size_t)kc * 4 + j) * tile + (kr >> 4) * (nrows * 16) +
                             (nr >> 3) * 128 + (nr & 7) * 16 + (kr & 15);
          base[off] = (uint8_t)(vj >> (8 * i));
        }
      }
    }
}

}  // namespace

int build_p3_tables(Ctx& c) {
  if (c.n != kPN) return 0;
  for (uint32_t q : c.primes)
    if (q <= (1u << 20)) return 0;   // Montgomery folds only
  const int np = c.n_primes;
  std::vector<uint8_t> t1((size_t)np * kC1T), t2((size_t)np * kC2T), t2ks;
  std::vector<uint32_t> hin(1), hout((size_t)np * kHWords);
  for (int inv = 0; inv < 2; ++inv) {
    if (!inv) t2ks.assign(t2.size(), 0);
    for (int p = 0; p < np; ++p) {
      const uint32_t q = c.primes[p];
      const uint32_t R = (uint32_t)(((uint64_t)1 << 32) % q);
      const uint32_t R2 = mulmod_p(R, R, q);
      const uint32_t psi = inv ? powmod_p(c.psis[p], q - 2, q) : c.psis[p];
      const uint32_t n_inv = powmod_p(kPN, q - 2, q);
      std::vector<uint32_t> pw(2 * kPN);   // psi^e (psi^-e for the inverse)
      pw[0] = 1;
      for (int e = 1; e < 2 * kPN; ++e) pw[e] = mulmod_p(pw[e - 1], psi, q);
      auto P = [&](uint64_t e) { return pw[e % (2 * kPN)]; };
      // pass 1 (32 x 32 inner transform of the 1024-point columns): w32 = psi^4096;
      // forward twist t[k] = psi^(2048 k) on the contraction index of stage A,
      // also applied by stage B and divided out of the inner Hadamard
      uint32_t tw[32], twi[32];
      for (int k = 0; k < 32; ++k) {
        tw[k] = inv ? 1u : P(2048ull * k);
        twi[k] = powmod_p(tw[k], q - 2, q);
      }
      pack_tiles(t1.data() + (size_t)p * kC1T, 32, q, [&](int cc, int k) {
        return mulmod_p(mulmod_p(P(4096ull * ((cc * k) & 31)), tw[k], q), R, q);
      });
      // outer Hadamard (forward psi^((2 k1 + 1) i2), inverse psi^-((2 i2 + 1) k1)),
      // k1 = b1 + 32 b2, factored as c[i2][b1] beta[i2][b2]:
      //   forward c = psi^((2 b1 + 1) i2), beta = psi^(64 i2 b2)
      //   inverse c = psi^-((2 i2 + 1) b1), beta = psi^-(32 (2 i2 + 1) b2)
      // c scales the stage-B input row (t, b1), so it rides in the inner
      // Hadamard; beta is applied per output column by the stage-B epilogue
      uint32_t* ht = hout.data() + (size_t)p * kHWords;
      auto shoup_p = [&](uint32_t w) { return (uint32_t)(((uint64_t)w << 32) / q); };
      for (int i2 = 0; i2 < kPn2; ++i2)
        for (int b2 = 0; b2 < 32; ++b2) {
          const uint32_t bv = inv ? P(32ull * (2 * i2 + 1) * b2) : P(64ull * i2 * b2);
          ht[kHBeta + i2 * 32 + b2] = bv;   // Shoup operand: no R
          ht[kHBetaS + i2 * 32 + b2] = shoup_p(bv);
        }
      for (int i2 = 0; i2 < kPn2; ++i2)
        for (int b1 = 0; b1 < 32; ++b1) {
          const uint32_t cv = inv ? P((2ull * i2 + 1) * b1) : P((2ull * b1 + 1) * i2);
#if TFHE_P3_CSHOUP
          ht[kHC + i2 * 36 + b1] = cv;   // Shoup operand: no R
          ht[kHCS + i2 * 36 + b1] = shoup_p(cv);
#else
          ht[kHC + i2 * 36 + b1] = mulmod_p(cv, R, q);   // Montgomery operand
#endif
        }
      for (int b1 = 0; b1 < 32; ++b1)
        for (int a2 = 0; a2 < 32; ++a2) {
          // inner Hadamard: forward psi^(64 (2 b1 + 1) a2), inverse psi^-(128 a2 b1)
          const uint32_t h = mulmod_p(inv ? P(128ull * a2 * b1) : P(64ull * (2 * b1 + 1) * a2),
                                      twi[a2], q);
          ht[kHIn + a2 * 36 + b1] = h;   // Shoup operand (no R), transposed
          ht[kHInS + a2 * 36 + b1] = shoup_p(h);
        }
      // pass 2 (64-point rows): forward psi^(2048 k2 i2), inverse
      // psi^-(1024 (2 i2 + 1) k2) n^-1 (row twist on the output k2)
      auto T2 = [&](int k2, int i2) {
        uint32_t v = inv ? mulmod_p(P(1024ull * (2 * i2 + 1) * k2), n_inv, q) : P(2048ull * k2 * i2);
        return mulmod_p(v, R, q);
      };
      pack_tiles(t2.data() + (size_t)p * kC2T, 64, q, T2);
      if (!inv)   // key-switch MAC: y R out of the fold (Montgomery form)
        pack_tiles(t2ks.data() + (size_t)p * kC2T, 64, q,
                   [&](int k2, int i2) { return mulmod_p(T2(k2, i2), R, q); });
      (void)R2;
    }
    auto up = [&](void** dst, const void* src, size_t bytes) {
      return cudaMalloc(dst, bytes) == cudaSuccess &&
             cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice) == cudaSuccess;
    };
    if (!up(reinterpret_cast<void**>(&c.d_p3t1[inv]), t1.data(), t1.size()) ||
        !up(reinterpret_cast<void**>(&c.d_p3hin[inv]), hin.data(), hin.size() * 4) ||
        !up(reinterpret_cast<void**>(&c.d_p3hout[inv]), hout.data(), hout.size() * 4) ||
        !up(reinterpret_cast<void**>(&c.d_p3t2[inv]), t2.data(), t2.size()) ||
        (!inv && !up(reinterpret_cast<void**>(&c.d_p3t2ks), t2ks.data(), t2ks.size()))) {
      set_error("p3 ntt table upload failed");
      return 3;
    }
  }
  return 0;
}

// pass 1 over `map` into the P^T workspace (rows = limb index of map)
int launch_p3_col(const Ctx& c, const uint32_t* in, uint32_t* P, const LimbMap& map, int batch,
                  int inverse, cudaStream_t st) {
  ColArgs a;
  memset(&a, 0, sizeof(a));
  a.tab = c.d_p3t1[inverse];
  a.hin = c.d_p3hin[inverse];
  a.hout = c.d_p3hout[inverse];
  a.P = P;
  a.pc = c.d_pc;
  a.batch = batch;
  a.map = map;
  const long long units = (long long)map.n * batch * 8;
  if (units >= (1ll << 31)) {
    set_error("p3 column pass: too many units");
    return 2;
  }
  a.units = (int)units;
  EncodeTiledFnP fn = encode_p();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return 3;
  }
  cuuint64_t dims[3] = {64, 1024, (cuuint64_t)max_row(map) * batch};
  cuuint64_t strides[2] = {256, (cuuint64_t)kPN * 4};
  cuuint32_t box[3] = {8, 256, 1};
  cuuint32_t es[3] = {1, 1, 1};
  if (fn(&a.tmap, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<uint32_t*>(in), dims, strides, box,
         es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    set_error("p3 column tensor map encode failed");
    return 3;
  }
  const int grid = (int)std::min<long long>(c.sms, units);
  if (grid <= 0) return 0;
#ifdef TFHE_P3_TRACE
  static unsigned long long* tbuf = nullptr;
  if (!tbuf) cudaMalloc(&tbuf, 16 * kPTraceN * 8);
  cudaMemsetAsync(tbuf, 0, 16 * kPTraceN * 8, st);
  a.trace = tbuf;
#endif
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kC1Smem);
    prof_begin(inverse ? "ntt_col_kernel<inv>" : "ntt_col_kernel<fwd>", st);
    kern<<<grid, kPThreads, kC1Smem, st>>>(a);
    prof_end(st);
  };
  if (inverse) go(ntt_col_kernel<true>);
  else go(ntt_col_kernel<false>);
#ifdef TFHE_P3_TRACE
  {
    std::vector<unsigned long long> hbuf(16 * kPTraceN);
    cudaMemcpy(hbuf.data(), tbuf, hbuf.size() * 8, cudaMemcpyDeviceToHost);
    static int seq = 0;
    char fn[256];
    snprintf(fn, sizeof(fn), "gpurun_out/ptrace_%d.bin", seq++);
    if (FILE* f = fopen(fn, "wb")) {
      fwrite(hbuf.data(), 8, hbuf.size(), f);
      fclose(f);
    }
  }
#endif
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("p3 column pass launch: ") + cudaGetErrorString(e));
    return 3;
  }
  return 0;
}

// pass 2: P^T rows map.in_row[l] -> out rows map.out_row[l] through the epilogue
int launch_p3_row(const Ctx& c, const uint32_t* P, uint32_t* out, const LimbMap& map, int batch,
                  int inverse, const EpiArgs* epi, cudaStream_t st, int S = 1) {
  const int mode = epi ? epi->mode : EPI_STORE;
  if ((mode == EPI_KS_MAC || mode == EPI_KS_ACC) && inverse) {
    set_error("p3 row pass: the key-switch epilogues need a forward transform");
    return 2;
  }
  RowArgs a;
  memset(&a, 0, sizeof(a));
  a.S = mode == EPI_KS_ACC ? S : 1;
  a.tab = (mode == EPI_KS_MAC || mode == EPI_KS_ACC) ? c.d_p3t2ks : c.d_p3t2[inverse];
  a.out = out;
  a.pc = c.d_pc;
  a.batch = batch;
  a.map = map;
  if (epi) a.epi = *epi;
  else a.epi.mode = EPI_STORE;
  const long long units = (long long)map.n * batch * 8 * a.S;
  if (units >= (1ll << 31)) {
    set_error("p3 row pass: too many units");
    return 2;
  }
  a.units = (int)units;
  EncodeTiledFnP fn = encode_p();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return 3;
  }
  const int prow = mode == EPI_KS_ACC ? a.S * map.n : max_row(map);   // P^T rows read
  cuuint64_t dims[2] = {1024, (cuuint64_t)prow * batch * 64};
  cuuint64_t strides[1] = {4096};
  cuuint32_t box[2] = {128, 64};
  cuuint32_t es[2] = {1, 1};
  if (fn(&a.tmap, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint32_t*>(P), dims, strides, box,
         es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    set_error("p3 row tensor map encode failed");
    return 3;
  }
  // whole slice groups per CTA (a group's sums live in one CTA's registers)
  const long long groups = units / a.S;
  const int grid = (int)std::min<long long>(c.sms, groups);
  if (grid <= 0) return 0;
  a.units = (int)groups;   // the kernel splits groups, then expands them by S
  // the key-switch epilogues read per-limb key rows shared by every member:
  // limb-synchronous CTAs keep them in L2 (contiguous ranges put every limb in
  // flight at once -- 1.75x DRAM read amplification at P-Default)
  static const int strided_env = getenv("TFHE_P3_STRIDED") ? atoi(getenv("TFHE_P3_STRIDED")) : -1;
  a.strided = strided_env >= 0 ? strided_env : (mode == EPI_KS_ACC || mode == EPI_KS_MAC);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kC2Smem);
    static const char* const names[] = {"ntt_row_kernel<store>", "ntt_row_kernel<sub_scale>",
                                        "ntt_row_kernel<ks_mac>", "ntt_row_kernel<ks_acc>"};
    prof_begin(mode >= 0 && mode < 4 ? names[mode] : "ntt_row_kernel", st);
    kern<<<grid, kRowThreads, kC2Smem, st>>>(a);
    prof_end(st);
  };
  if (mode == EPI_KS_ACC) go(ntt_row_kernel<EPI_KS_ACC>);
  else if (mode == EPI_SUB_SCALE) go(ntt_row_kernel<EPI_SUB_SCALE>);
  else if (mode == EPI_KS_MAC) go(ntt_row_kernel<EPI_KS_MAC>);
  else go(ntt_row_kernel<EPI_STORE>);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("p3 row pass launch: ") + cudaGetErrorString(e));
    return 3;
  }
  return 0;
}

int launch_ntt_p3_ks_group(const Ctx& c, const uint32_t* in, void* ws, const LimbMap& s1map,
                           const LimbMap& tmap, int S, int batch, const EpiArgs& epi,
                           cudaStream_t st) {
  if (s1map.n != S * tmap.n) {
    set_error("key-switch group: stage-1 map must hold S * T limbs");
    return 2;
  }
  // P^T row l = s * T + t; a slice's own target rows are reused unchanged
  // (ckks.py:361-364) and their sums skipped by the row pass, so the column
  // pass leaves those P^T rows unwritten (don't-care)
  LimbMap m1;
  m1.n = 0;
  for (int l = 0; l < s1map.n; ++l) {
    const int sl = l / tmap.n, t = l % tmap.n;
    if (epi.j0 + sl == epi.js[t]) continue;
    m1.prime[m1.n] = s1map.prime[l];
    m1.in_row[m1.n] = s1map.in_row[l];
    m1.out_row[m1.n] = (int16_t)l;
    ++m1.n;
  }
  int rc = m1.n ? launch_p3_col(c, in, static_cast<uint32_t*>(ws), m1, batch, 0, st) : 0;
  if (rc) return rc;
  EpiArgs e = epi;
  e.mode = EPI_KS_ACC;
  return launch_p3_row(c, static_cast<const uint32_t*>(ws), nullptr, tmap, batch, 0, &e, st, S);
}

int launch_ntt_p3(const Ctx& c, const uint32_t* in, uint32_t* out, const LimbMap& map, int batch,
                  int inverse, const EpiArgs* epi, void* ws, cudaStream_t st) {
  LimbMap m1 = map;   // pass 1 writes P^T row l for limb l
  for (int l = 0; l < m1.n; ++l) m1.out_row[l] = (int16_t)l;
  int rc = launch_p3_col(c, in, static_cast<uint32_t*>(ws), m1, batch, inverse, st);
  if (rc) return rc;
  static const bool dbg = getenv("TFHE_P3_DBG") != nullptr;   // tests: expose P^T
  if (dbg)
    return cudaMemcpyAsync(out, ws, (size_t)map.n * batch * kPN * 4, cudaMemcpyDeviceToDevice, st)
               ? 3 : 0;
  LimbMap m2 = map;
  for (int l = 0; l < m2.n; ++l) m2.in_row[l] = (int16_t)l;
  return launch_p3_row(c, static_cast<const uint32_t*>(ws), out, m2, batch, inverse, epi, st);
}

}  // namespace tfhe
