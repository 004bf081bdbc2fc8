// Fused two-stage tensor-core NTT / INTT for n = 4096 (plan 64 x 64: Set_A,
// `default`, BASELINE configs[0]) -- one persistent launch per call, stage 1's
// P never leaves the SM.
//
// Same exact byte-sliced arithmetic as ntt_tc.cu (SURVEY Appendix B's
// 4-accumulator form, ref ntt.py:212-340): data byte planes X_j times
// pre-multiplied twiddle planes V_{j,i} = bytes i of 2^(8j) T R mod q,
// accumulators C_i = sum_j V_{j,i} X_j in TMEM, folded by one Montgomery step.
//
// One shared twiddle table.  With n1 = n2 = 64 and w = psi^128 (a primitive
// 64th root of unity) the reference's stage matrices (params.py:198-228) are
//   forward:  W1[k1][i1] = w^(k1 i1) psi^(64 i1),   W3[i2][k2] = w^(i2 k2)
//   inverse:  W1[k1][i1] = w^-(k1 i1),              W3[i2][k2] = w^-(i2 k2) psi^(-64 k2) n^-1
// i.e. both stages are the SAME symmetric 64-point DFT matrix D (w or w^-1)
// plus a diagonal twist: forward pre-multiplies input row i1 by psi^(64 i1)
// (in the producers, one Montgomery product per element), inverse
// post-multiplies output column k2 by psi^(-64 k2) n^-1 (in the stage-2
// epilogue).  So one 64 KB byte-plane table serves both stages and the whole
// working set fits in shared memory: D tiles 64 KB | A1 32 KB | A2 32 KB |
// raw ring 2 x 32 KB | W2 16 KB (+ 4 KB of A1 bank-conflict padding).
//
// Work unit = two batch members of one limb (MMA M = 128 rows).
//   stage 1: D1[(b,i2)][k1] = sum_i1 A'_b[i1][i2] D[k1][i1]   A1 = data planes, MN-major
//            (m = (b,i2) contiguous for fixed k = i1, so producers store 4-byte words)
//   epi 1:   P = fold(D1) .* W2, byte-split straight into A2 (MN-major again: the
//            thread of row (b,i2) holds 16 consecutive k1 = 16 contiguous bytes of
//            A2 row k = i2, one 16-byte store per plane)
//   stage 2: D2[(b,k1)][k2] = sum_i2 P_b[k1][i2] D[k2][i2]
//   epi 2:   out[b][k2 n1 + k1] = fold(D2) (x twist) -> fused epilogue modes
// Roles (16 warps, 128 registers each): 0-2 producers (bulk-copy raw members
// in, twist, byte split), 3 MMA issuer + TMEM owner, 4-7 stage-1 epilogue (one
// per TMEM lane quarter, 16-column chunks written to A2 as they fold), 8-15
// stage-2 epilogue (two per lane quarter, 32 columns each).  TMEM: columns [0,256) stage-1 accumulators, [256,512) stage 2.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "tfhe_internal.h"

namespace tfhe {

namespace {

constexpr int kFN = 4096, kFn1 = 64;
constexpr int kFRows = 128;                   // MMA M: two members x 64 rows
constexpr int kFPlane = kFRows * 32;          // one A plane tile (128 rows x 32 K bytes)
constexpr int kFABytes = 2 * 4 * kFPlane;     // KC = 2 K-steps x 4 planes = 32 KB
// A1 pads each 16-row core-matrix group by 16 bytes (SBO 144): the producers'
// 4-byte stores of 8 lanes then hit distinct banks
constexpr int kFSbo1 = 144, kFLbo1 = 8 * kFSbo1, kFPlane1 = 4 * kFLbo1;
constexpr int kFA1Bytes = 2 * 4 * kFPlane1;
constexpr int kFTwBytes = 2 * 4 * 256 * 32;   // (K-step, plane) B tiles of 256 rows x 32 K = 64 KB
constexpr int kFRawBytes = 2 * kFN * 4;       // one unit's raw u32 data (two members)
constexpr int kFW2Bytes = kFN * 4;
constexpr int kFThreads = 512;
constexpr int kFProdWarps = 3;
constexpr int kFMmaWarp = 3;
constexpr int kFEpi1Warp0 = 4, kFEpi2Warp0 = 8;
constexpr int kFSmem = kFTwBytes + kFA1Bytes + kFABytes + 2 * kFRawBytes + kFW2Bytes + 2 * 64 * 4 + 32 * 8;

struct FusedArgs {
  const uint32_t* in;
  uint32_t* out;
  const uint8_t* dft;      // [prime] 64 KB byte-plane tiles of D (direction of the call)
  const uint32_t* w2m;     // [prime][k1][i2] W2 R mod q (Montgomery Hadamard)
  const uint32_t* twist;   // [prime][64]: forward pre-twist (x R or x R^2) / inverse post-twist
  const PrimeConst* pc;
  int batch, upl;          // members; units per limb = ceil(batch / 2)
  int inverse;
  long long units;
  LimbMap map;
  EpiArgs epi;
};

// sum_i 2^(8i) C_i (C_i < 2^24 for K = 64) -> v 2^-32 mod q, lazy in [0, 2q)
TFHE_DEV uint32_t fold4_mont(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                             const PrimeConst& pc) {
  const uint64_t v = (uint64_t)(c0 + (c1 << 8)) + ((uint64_t)(c2 + (c3 << 8)) << 16);
  const uint32_t m = (uint32_t)v * pc.qneg_inv;
  return (uint32_t)((v + (uint64_t)m * pc.q) >> 32);
}
// a b 2^-32 mod q for a b < q 2^32, lazy in [0, 2q)
TFHE_DEV uint32_t mont_lazy(uint32_t a, uint32_t b, const PrimeConst& pc) {
  const uint64_t v = (uint64_t)a * b;
  const uint32_t m = (uint32_t)v * pc.qneg_inv;
  return (uint32_t)((v + (uint64_t)m * pc.q) >> 32);
}
TFHE_DEV uint32_t corr(uint32_t t, uint32_t q) { return t >= q ? t - q : t; }

TFHE_DEV void planes4f(uint32_t v0, uint32_t v1, uint32_t v2, uint32_t v3, uint32_t (&w)[4]) {
  const uint32_t lo01 = __byte_perm(v0, v1, 0x5140), hi01 = __byte_perm(v0, v1, 0x7362);
  const uint32_t lo23 = __byte_perm(v2, v3, 0x5140), hi23 = __byte_perm(v2, v3, 0x7362);
  w[0] = __byte_perm(lo01, lo23, 0x5410);
  w[1] = __byte_perm(lo01, lo23, 0x7632);
  w[2] = __byte_perm(hi01, hi23, 0x5410);
  w[3] = __byte_perm(hi01, hi23, 0x7632);
}

// byte offset of (row m, k) inside an MN-major operand (K-step kc = k / 32,
// plane j): SWIZZLE_NONE core matrices of 16 m x 8 k, LBO (k groups) = 8 SBO,
// SBO (m groups) = 128 (A2) or 144 (A1, padded)
template <int SBO>
TFHE_DEV uint32_t mn_off(int j, int m, int k) {
  return (uint32_t)(((k >> 5) * 4 + j) * (32 * SBO) + ((k & 31) >> 3) * (8 * SBO) +
                    (m >> 4) * SBO + (k & 7) * 16 + (m & 15));
}

__global__ void __launch_bounds__(kFThreads, 1) ntt_fused_kernel(const __grid_constant__ FusedArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sD = smem;
  uint8_t* sA1 = sD + kFTwBytes;
  uint8_t* sA2 = sA1 + kFA1Bytes;
  uint8_t* sRaw = sA2 + kFABytes;
  uint32_t* sW2 = reinterpret_cast<uint32_t*>(sRaw + 2 * kFRawBytes);
  uint32_t* sTw = sW2 + kFN;                   // 64 twist constants
  uint64_t* bar = reinterpret_cast<uint64_t*>(sTw + 2 * 64);
  uint64_t* raw_full = bar + 0;    // [2]
  uint64_t* raw_empty = bar + 2;   // [2]
  uint64_t* a1_full = bar + 4;
  uint64_t* a1_empty = bar + 5;
  uint64_t* acc1_full = bar + 6;
  uint64_t* acc1_empty = bar + 7;
  uint64_t* a2_full = bar + 8;
  uint64_t* a2_empty = bar + 9;
  uint64_t* acc2_full = bar + 10;
  uint64_t* acc2_empty = bar + 11;
  uint64_t* tw_full = bar + 12;
  uint64_t* tw_empty = bar + 13;
  uint64_t* epi1_done = bar + 14;
  uint64_t* epi2_done = bar + 15;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long u0 = a.units * blockIdx.x / gridDim.x;
  const int cnt = (int)(a.units * (blockIdx.x + 1) / gridDim.x - u0);
  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&raw_empty[s], 32 * kFProdWarps);
    }
    mbar_init(a1_full, 32 * kFProdWarps);
    mbar_init(a1_empty, 1);
    mbar_init(acc1_full, 1);
    mbar_init(acc1_empty, 128);
    mbar_init(a2_full, 128);
    mbar_init(a2_empty, 1);
    mbar_init(acc2_full, 1);
    mbar_init(acc2_empty, 256);
    mbar_init(tw_full, 1);
    mbar_init(tw_empty, 1);
    mbar_init(epi1_done, 128);
    mbar_init(epi2_done, 256);
    fence_mbar_init();
  }
  if (warp == kFMmaWarp) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const bool fwd = !a.inverse;
  auto limb_of = [&](int it) { return (int)((u0 + it) / a.upl); };
  auto last_of_limb = [&](int it) { return it + 1 == cnt || limb_of(it + 1) != limb_of(it); };

  if (warp < 4) {
    if (warp < kFProdWarps) {
      // ------------------------------------------------------------ producers
      const int ptid = tid;   // 0..95
      auto issue_raw = [&](int it, int slot) {
        const long long g = u0 + it;
        const int limb = (int)(g / a.upl), pair = (int)(g % a.upl);
        const int b0 = 2 * pair, nb = min(2, a.batch - b0);
        const uint32_t bytes = (uint32_t)nb * kFN * 4;
        mbar_arrive_expect_tx(&raw_full[slot], bytes);
        bulk_g2s(sRaw + slot * kFRawBytes,
                 a.in + ((size_t)a.map.in_row[limb] * a.batch + b0) * kFN, bytes, &raw_full[slot]);
      };
      if (ptid == 0)
        for (int it = 0; it < 2 && it < cnt; ++it) issue_raw(it, it);
      int prev_limb = -1;
      uint32_t tw_ph = 0;
      for (int it = 0; it < cnt; ++it) {
        const int limb = limb_of(it);
        if (limb != prev_limb) {
          if (ptid == 0) {
            if (prev_limb >= 0) {
              // every MMA and epilogue of the previous limb is done with the tables
              mbar_wait(tw_empty, tw_ph);
              mbar_wait(epi1_done, tw_ph);
              mbar_wait(epi2_done, tw_ph);
            }
            const int pr = a.map.prime[limb];
            mbar_arrive_expect_tx(tw_full, kFTwBytes + kFW2Bytes + 64 * 4);
            bulk_g2s(sD, a.dft + (size_t)pr * kFTwBytes, kFTwBytes, tw_full);
            bulk_g2s(sW2, a.w2m + (size_t)pr * kFN, kFW2Bytes, tw_full);
            bulk_g2s(sTw, a.twist + (size_t)pr * 64, 64 * 4, tw_full);
          }
          if (prev_limb >= 0) tw_ph ^= 1;
          mbar_wait(tw_full, tw_ph);   // the pre-twist constants are resident
          prev_limb = limb;
        }
        const PrimeConst pc = a.pc[a.map.prime[limb]];
        const int slot = it & 1;
        mbar_wait(&raw_full[slot], (it >> 1) & 1);
        if (it >= 1) mbar_wait(a1_empty, (it - 1) & 1);   // MMA1(it-1) has read A1
        const uint8_t* raw = sRaw + slot * kFRawBytes;
        // 64 warp items per unit: (member b, 4 rows i1, 32 columns i2); lane ->
        // (r = lane / 8, c = lane % 8): 16-byte raw reads conflict-free per phase
        const int r = lane >> 3, c = lane & 7;
        for (int item = warp; item < 64; item += kFProdWarps) {
          const int b = item >> 5, ib = (item >> 1) & 15, jb = item & 1;
          const int i1 = 4 * ib + r, i2 = 32 * jb + 4 * c;
          uint4 x = *reinterpret_cast<const uint4*>(raw + (size_t)b * kFN * 4 + (i1 * kFn1 + i2) * 4);
          if (fwd) {
            const uint32_t t = sTw[i1];   // psi^(64 i1) R (x R again for the key-switch MAC)
            x.x = mont_lazy(x.x, t, pc);
            x.y = mont_lazy(x.y, t, pc);
            x.z = mont_lazy(x.z, t, pc);
            x.w = mont_lazy(x.w, t, pc);
          }
          uint32_t w[4];
          planes4f(x.x, x.y, x.z, x.w, w);
          const int m = b * 64 + i2;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            *reinterpret_cast<uint32_t*>(sA1 + mn_off<kFSbo1>(j, m, i1)) = w[j];
        }
        fence_proxy_async_smem();
        mbar_arrive(a1_full);
        mbar_arrive(&raw_empty[slot]);
        if (ptid == 0 && it + 2 < cnt) {
          mbar_wait(&raw_empty[slot], (it >> 1) & 1);
          issue_raw(it + 2, slot);
        }
      }
    } else {
      // ------------------------------------------------------------ MMA issuer
      // one MMA per (K-step, data plane): N = 256 = the four output-byte tiles
      // V_{j,0..3} side by side, landing in the four accumulators C_0..C_3
      // (TMEM columns i*64); A MN-major
      constexpr uint32_t idesc = idesc_i8(kFRows, 256) | (1u << 15);
      const uint32_t sD_u = smem_u32(sD);
      auto issue = [&](uint32_t a_base, uint32_t d, uint32_t sbo) {
#pragma unroll
        for (int kc = 0; kc < 2; ++kc)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint64_t ad = smem_desc_kmajor(a_base + (kc * 4 + j) * 32 * sbo, 8 * sbo, sbo);
            const uint64_t bd = smem_desc_kmajor(sD_u + (kc * 4 + j) * 8192, 4096, 128);
            mma_i8_ss(d, ad, bd, idesc, (kc | j) != 0);
          }
      };
      auto stage2 = [&](int v) {
        mbar_wait(a2_full, v & 1);
        if (v >= 1) mbar_wait(acc2_empty, (v - 1) & 1);
        tc_fence_after();
        if (elect_one()) {
          issue(smem_u32(sA2), tmem + 256, 128);
          mma_commit(a2_empty);
          mma_commit(acc2_full);
          if (last_of_limb(v)) mma_commit(tw_empty);
        }
        __syncwarp();
      };
      int prev_limb = -1;
      uint32_t tw_ph = 0;
      int s2_next = 0;   // next unit whose stage 2 is still to issue
      for (int it = 0; it < cnt; ++it) {
        const int limb = limb_of(it);
        if (limb != prev_limb) {
          // the previous limb's stage 2 goes first: its tables are still resident
          while (s2_next < it) stage2(s2_next++);
          if (prev_limb >= 0) tw_ph ^= 1;
          mbar_wait(tw_full, tw_ph);
          prev_limb = limb;
        }
        mbar_wait(a1_full, it & 1);
        if (it >= 1) mbar_wait(acc1_empty, (it - 1) & 1);
        tc_fence_after();
        if (elect_one()) {
          issue(smem_u32(sA1), tmem, kFSbo1);
          mma_commit(a1_empty);
          mma_commit(acc1_full);
        }
        __syncwarp();
        while (s2_next < it) stage2(s2_next++);
      }
      while (s2_next < cnt) stage2(s2_next++);
    }
  } else if (warp < kFEpi2Warp0) {
    // -------------------------------------------------------------- stage-1 epilogue
    // warp -> TMEM lane quarter q (rows 32q..32q+31), all 64 columns k1 in
    // 16-column chunks: fold, Hadamard, byte-split, store into A2
    const int q = warp & 3;
    const int row = q * 32 + lane, b = row >> 6, i2 = row & 63;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    int prev_limb = -1;
    uint32_t tw_ph = 0;
    for (int it = 0; it < cnt; ++it) {
      const int limb = limb_of(it);
      if (limb != prev_limb) {
        if (prev_limb >= 0) tw_ph ^= 1;
        mbar_wait(tw_full, tw_ph);   // this limb's W2
        prev_limb = limb;
      }
      const PrimeConst pc = a.pc[a.map.prime[limb]];
      mbar_wait(acc1_full, it & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < 64; c0 += 16) {
        uint32_t acc[4][16];
#pragma unroll
        for (int i = 0; i < 4; ++i) tmem_ld16(tmem + lane_off + i * 64 + c0, acc[i]);
        tmem_ld_wait();
        if (c0 == 48) {
          tc_fence_before();
          mbar_arrive(acc1_empty);   // buffer drained: MMA1(it+1) may start
        }
        uint32_t p[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          // S = fold (twiddles carry R), P = S W2 (W2 carries R): both lazy [0, 2q)
          const uint32_t s = fold4_mont(acc[0][e], acc[1][e], acc[2][e], acc[3][e], pc);
          p[e] = mont_lazy(s, sW2[(c0 + e) * 64 + i2], pc);
        }
        uint32_t pl[4][4];   // [plane][word]
#pragma unroll
        for (int e4 = 0; e4 < 4; ++e4) {
          uint32_t w[4];
          planes4f(p[4 * e4], p[4 * e4 + 1], p[4 * e4 + 2], p[4 * e4 + 3], w);
#pragma unroll
          for (int j = 0; j < 4; ++j) pl[j][e4] = w[j];
        }
        if (c0 == 0 && it >= 1) mbar_wait(a2_empty, (it - 1) & 1);   // MMA2(it-1) read A2
        const int m = b * 64 + c0;   // A2 row (b, k1) of the chunk's first k1
#pragma unroll
        for (int j = 0; j < 4; ++j)
          *reinterpret_cast<uint4*>(sA2 + mn_off<128>(j, m, i2)) =
              make_uint4(pl[j][0], pl[j][1], pl[j][2], pl[j][3]);
      }
      fence_proxy_async_smem();
      mbar_arrive(a2_full);
      if (last_of_limb(it)) mbar_arrive(epi1_done);
    }
  } else {
    // -------------------------------------------------------------- stage-2 epilogue
    const int q = warp & 3, h = (warp - kFEpi2Warp0) >> 2;
    const int row = q * 32 + lane, b = row >> 6, k1 = row & 63;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const int mode = a.epi.mode;
    int prev_limb = -1;
    uint32_t tw_ph = 0;
    for (int it = 0; it < cnt; ++it) {
      const long long gu = u0 + it;
      const int limb = limb_of(it);
      if (limb != prev_limb) {
        if (prev_limb >= 0) tw_ph ^= 1;
        mbar_wait(tw_full, tw_ph);   // this limb's post-twist (inverse)
        prev_limb = limb;
      }
      const PrimeConst pc = a.pc[a.map.prime[limb]];
      const int bm = 2 * (int)(gu % a.upl) + b;   // batch member of this row
      const bool valid = bm < a.batch;
      const size_t orow = ((size_t)a.map.out_row[limb] * a.batch + bm) * kFN + k1;
      mbar_wait(acc2_full, it & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c0 = 32 * h; c0 < 32 * h + 32; c0 += 8) {
        uint32_t acc[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i) tmem_ld8(tmem + 256 + lane_off + i * 64 + c0, acc[i]);
        // epilogue operands (issued before the TMEM wait so the loads overlap it)
        uint32_t p0[8], p1[8], kb[8], ka[8];
        const uint32_t* s0 = nullptr;
        const uint32_t* s1 = nullptr;
        if (valid) {
          if (mode == EPI_SUB_SCALE) {
            s0 = a.epi.x + ((size_t)a.epi.x_row[limb] * a.batch + bm) * kFN + k1;
            const int br = a.epi.base_row[limb];
            if (br >= 0) s1 = a.epi.base + ((size_t)br * a.batch + bm) * kFN + k1;
          } else if (mode == EPI_KS_MAC && !a.epi.first) {
            s0 = a.epi.acc_b + orow;
            s1 = a.epi.acc_a + orow;
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const size_t pos = (size_t)(c0 + e) * kFn1;
            if (s0) p0[e] = s0[pos];
            if (s1) p1[e] = s1[pos];
          }
          if (mode == EPI_KS_MAC) {
            const size_t kr = (size_t)a.epi.key_row[limb] * kFN + k1;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              kb[e] = __ldg(a.epi.kb + kr + (size_t)(c0 + e) * kFn1);
              ka[e] = __ldg(a.epi.ka + kr + (size_t)(c0 + e) * kFn1);
            }
          }
        }
        tmem_ld_wait();
        if (c0 + 8 == 32 * h + 32) {
          tc_fence_before();
          mbar_arrive(acc2_empty);   // buffer drained: MMA2(it+1) may start
        }
        if (!valid) continue;
        uint32_t y[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          uint32_t t = fold4_mont(acc[0][e], acc[1][e], acc[2][e], acc[3][e], pc);
          if (!fwd) t = mont_lazy(t, sTw[c0 + e], pc);   // psi^(-64 k2) n^-1 (R)
          y[e] = corr(t, pc.q);
        }
        uint32_t* o = a.out + orow + (size_t)c0 * kFn1;
        if (mode == EPI_KS_MAC) {
          // y arrives as y R (the forward pre-twist carries R^2): one Montgomery
          // product per key gives y k
          uint32_t* ob = a.epi.acc_b + orow + (size_t)c0 * kFn1;
          uint32_t* oa = a.epi.acc_a + orow + (size_t)c0 * kFn1;
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const uint32_t tb = corr(mont_lazy(y[e], kb[e], pc), pc.q);
            const uint32_t ta = corr(mont_lazy(y[e], ka[e], pc), pc.q);
            ob[e * kFn1] = a.epi.first ? tb : add_mod(p0[e], tb, pc.q);
            oa[e * kFn1] = a.epi.first ? ta : add_mod(p1[e], ta, pc.q);
          }
          continue;
        }
        if (mode == EPI_SUB_SCALE) {
          const uint32_t s = a.epi.s[limb], ss = a.epi.s_shoup[limb];
#pragma unroll
          for (int e = 0; e < 8; ++e) y[e] = mul_shoup(sub_mod(p0[e], y[e], pc.q), s, ss, pc.q);
          if (s1) {
#pragma unroll
            for (int e = 0; e < 8; ++e) y[e] = add_mod(p1[e], y[e], pc.q);
          }
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e * kFn1] = y[e];
      }
      if (last_of_limb(it)) mbar_arrive(epi2_done);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kFMmaWarp) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

uint32_t mulmod_f(uint64_t a, uint64_t b, uint32_t q) { return (uint32_t)(a * b % q); }
uint32_t powmod_f(uint64_t b, uint64_t e, uint32_t q) {
  uint64_t r = 1 % q, x = b % q;
  while (e) {
    if (e & 1) r = r * x % q;
    x = x * x % q;
    e >>= 1;
  }
  return (uint32_t)r;
}

}  // namespace

bool fused_eligible(const Ctx& c) { return c.d_fdft[0] != nullptr; }

int build_fused_tables(Ctx& c) {
  if (!(c.n == kFN && c.n1 == 64 && c.n2 == 64)) return 0;
  for (uint32_t q : c.primes)
    if (q <= (1u << 20)) return 0;   // the fused epilogues use Montgomery folds only
  const int np = c.n_primes;
  std::vector<uint8_t> tiles((size_t)np * kFTwBytes);
  std::vector<uint32_t> w2((size_t)np * kFN), tw((size_t)np * 64);
  for (int inv = 0; inv < 2; ++inv) {
    for (int p = 0; p < np; ++p) {
      const uint32_t q = c.primes[p];
      const uint32_t psi = inv ? powmod_f(c.psis[p], q - 2, q) : c.psis[p];
      const uint32_t w = powmod_f(psi, 128, q);   // primitive 64th root (inverse: w^-1)
      const uint32_t R = (uint32_t)(((uint64_t)1 << 32) % q);
      uint32_t wp[64];
      wp[0] = 1;
      for (int e = 1; e < 64; ++e) wp[e] = mulmod_f(wp[e - 1], w, q);
      uint8_t* base = tiles.data() + (size_t)p * kFTwBytes;
      for (int cc = 0; cc < 64; ++cc)        // output column (k1 or k2)
        for (int k = 0; k < 64; ++k) {       // contraction index (i1 or i2)
          const uint32_t t = mulmod_f(wp[(cc * k) & 63], R, q);   // D[cc][k] R
          const int kc = k / 32, kr = k % 32;
          for (int j = 0; j < 4; ++j) {
            const uint32_t vj = mulmod_f(t, 1ull << (8 * j), q);
            for (int i = 0; i < 4; ++i) {
              // B operand of the (kc, j) MMA: 256 K-major rows n = 64 i + cc, 32 K bytes
              // (SBO = 128 between 8-row groups, LBO = 4096 between the K halves)
              const int nr = 64 * i + cc;
              const size_t off = ((size_t)kc * 4 + j) * 8192 + (kr >> 4) * 4096 + (nr >> 3) * 128 +
                                 (nr & 7) * 16 + (kr & 15);
              base[off] = (uint8_t)(vj >> (8 * i));
            }
          }
        }
      // W2 R: forward psi^(2 k1 i2 + i2), inverse psi^-(2 k1 i2 + k1) (params.py:198-228)
      std::vector<uint32_t> pw(2 * kFN);
      pw[0] = 1;
      for (int e = 1; e < 2 * kFN; ++e) pw[e] = mulmod_f(pw[e - 1], psi, q);
      for (int k1 = 0; k1 < 64; ++k1)
        for (int i2 = 0; i2 < 64; ++i2) {
          const int e = inv ? (2 * k1 * i2 + k1) : (2 * k1 * i2 + i2);
          w2[(size_t)p * kFN + k1 * 64 + i2] = mulmod_f(pw[e % (2 * kFN)], R, q);
        }
      // twists: forward pre-twist psi^(64 i1) R; inverse post-twist psi^(-64 k2) n^-1 R
      const uint32_t n_inv = powmod_f(kFN, q - 2, q);
      for (int k = 0; k < 64; ++k) {
        uint32_t v = mulmod_f(pw[64 * k], R, q);
        if (inv) v = mulmod_f(v, n_inv, q);
        tw[(size_t)p * 64 + k] = v;
      }
    }
    auto up = [&](void** dst, const void* src, size_t bytes) {
      return cudaMalloc(dst, bytes) == cudaSuccess &&
             cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice) == cudaSuccess;
    };
    if (!up(reinterpret_cast<void**>(&c.d_fdft[inv]), tiles.data(), tiles.size()) ||
        !up(reinterpret_cast<void**>(&c.d_fw2[inv]), w2.data(), w2.size() * 4) ||
        !up(reinterpret_cast<void**>(&c.d_ftw[inv]), tw.data(), tw.size() * 4)) {
      set_error("fused ntt table upload failed");
      return 3;
    }
    if (!inv) {
      // key-switch MAC variant of the forward pre-twist: psi^(64 i1) R^2
      for (int p = 0; p < np; ++p) {
        const uint32_t q = c.primes[p];
        const uint32_t R = (uint32_t)(((uint64_t)1 << 32) % q);
        for (int k = 0; k < 64; ++k) tw[(size_t)p * 64 + k] = mulmod_f(tw[(size_t)p * 64 + k], R, q);
      }
      if (!up(reinterpret_cast<void**>(&c.d_ftw_ks), tw.data(), tw.size() * 4)) {
        set_error("fused ntt table upload failed");
        return 3;
      }
    }
  }
  return 0;
}

// -1: not applicable (the caller runs the two-stage kernels)
int launch_ntt_fused(const Ctx& c, const uint32_t* in, uint32_t* out, const LimbMap& map,
                     int batch, int inverse, const EpiArgs* epi, cudaStream_t st) {
  if (!fused_eligible(c) || getenv("TFHE_NO_FUSED")) return -1;
  const int mode = epi ? epi->mode : EPI_STORE;
  if (mode == EPI_KS_ACC || (mode == EPI_KS_MAC && inverse)) return -1;
  // in-place calls must map every limb onto its own row (a unit reads its
  // members' input before it writes their output, nothing else)
  if (in == out)
    for (int l = 0; l < map.n; ++l)
      if (map.in_row[l] != map.out_row[l]) return -1;
  FusedArgs a;
  memset(&a, 0, sizeof(a));
  a.in = in;
  a.out = out;
  a.dft = c.d_fdft[inverse ? 1 : 0];
  a.w2m = c.d_fw2[inverse ? 1 : 0];
  a.twist = inverse ? c.d_ftw[1] : (mode == EPI_KS_MAC ? c.d_ftw_ks : c.d_ftw[0]);
  a.pc = c.d_pc;
  a.batch = batch;
  a.upl = (batch + 1) / 2;
  a.inverse = inverse ? 1 : 0;
  a.units = (long long)a.upl * map.n;
  a.map = map;
  if (epi) a.epi = *epi;
  else a.epi.mode = EPI_STORE;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(ntt_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFSmem);
    attr = true;
  }
  const int grid = (int)std::min<long long>(c.sms, a.units);
  if (grid <= 0) return 0;
  ntt_fused_kernel<<<grid, kFThreads, kFSmem, st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("fused ntt launch: ") + cudaGetErrorString(e));
    return 3;
  }
  return 0;
}

}  // namespace tfhe
