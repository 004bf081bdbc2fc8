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
// i.e. both stages are the same 64-point DFT matrix D (w or w^-1) up to a
// diagonal twist: forward twists the contraction index (t[k] = psi^(64 k)),
// inverse the output index (u[c] = psi^(-64 c) n^-1).  Both stages therefore
// use ONE table T (forward T[c][k] = w^(ck) t[k], inverse T[c][k] = u[c] w^-(ck))
// and the twist the other stage did not ask for is divided out of the Hadamard
// table for free: forward W2'[k1][i2] = W2 / t[i2] (stage 2 multiplies column
// i2 by t), inverse W2' = W2 / u[k1] (stage 1 multiplies row k1 by u).  No
// per-element twist is computed anywhere, and the whole working set fits in
// shared memory: D tiles 64 KB | A1 2 x 36 KB (padded
// against bank conflicts) | A2 32 KB | raw 32 KB | W2 17 KB.
//
// Work unit = two batch members of one limb (MMA M = 128 rows).
//   stage 1: D1[(b,i2)][k1] = sum_i1 A'_b[i1][i2] D[k1][i1]   A1 = data planes, MN-major
//            (m = (b,i2) contiguous for fixed k = i1, so producers store 4-byte words)
//   epi 1:   P = fold(D1) .* W2, byte-split straight into A2 (MN-major again: the
//            thread of row (b,i2) holds 16 consecutive k1 = 16 contiguous bytes of
//            A2 row k = i2, one 16-byte store per plane)
//   stage 2: D2[(b,k1)][k2] = sum_i2 P_b[k1][i2] D[k2][i2]
//   epi 2:   out[b][k2 n1 + k1] = fold(D2) (x twist) -> fused epilogue modes
// Roles (16 warps, 128 registers each): 0-2 producers (one bulk copy per unit
// lands the two raw members; each thread pulls its <= 22 x 16 bytes into
// registers at once so the slot refills early, then twists / byte-splits into
// the double-buffered A1), 3 MMA issuer + TMEM owner, 4-11 stage-1 epilogue
// (two per TMEM lane quarter, 32 columns each in 16-column chunks written to
// A2 as they fold), 12-15 stage-2 epilogue (one per lane quarter: folds all 64
// columns first and releases the accumulators, then applies the epilogue
// mode and stores).  TMEM: columns [0,256) stage-1 accumulators, [256,512) stage 2.
#include <algorithm>
#include <cstdio>
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
constexpr int kFThreads = 512;               // 16 warps = 4 per SMSP at 128 registers
constexpr int kFProdWarps = 3;
constexpr int kFEpi1Warp0 = 4;
#ifndef TFHE_FUSED_E1_MAC
#define TFHE_FUSED_E1_MAC 1
#endif
#ifndef TFHE_FUSED_E1_SUB
#define TFHE_FUSED_E1_SUB 1
#endif
// epilogue warps per TMEM lane quarter: 12 epilogue warps split 2 + 1 (plain
// transforms: stage 1 has the heavier epilogue) or 1 + 2 (fused epilogue modes:
// stage 2 streams operands); each warp owns 64 / W columns
template <int MODE>
__host__ __device__ constexpr int epi1_per_q() {
  return MODE == EPI_STORE ? 2 : MODE == EPI_KS_MAC ? TFHE_FUSED_E1_MAC : TFHE_FUSED_E1_SUB;
}
constexpr int kFMmaWarp = 3;
constexpr int kFItems = 22;                   // ceil(64 warp items / 3 producer warps)
// W2 R transposed [i2][k1] with a 68-word row pitch: the stage-1 epilogue
// reads its row's 16 consecutive k1 as four conflict-free 16-byte loads
constexpr int kFW2Pitch = 68;
constexpr int kFW2TBytes = 64 * kFW2Pitch * 4;
constexpr int kFSmem = kFTwBytes + 2 * kFA1Bytes + kFABytes + kFRawBytes + kFW2TBytes + 32 * 8;

struct FusedArgs {
  const uint32_t* in;
  uint32_t* out;
  const uint8_t* dft;      // [prime] 64 KB byte-plane tiles of D (direction of the call)
  const uint32_t* w2m;     // [prime][i2][68-word row: k1] W2 R mod q (Montgomery Hadamard)
  const PrimeConst* pc;
  int batch, upl;          // members; units per limb = ceil(batch / 2)
  int inverse;
  long long units;
  LimbMap map;
  EpiArgs epi;
  unsigned long long* trace;   // TFHE_FUSED_TRACE builds only
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

// mbarrier wait that suspends the warp (hint: up to ~1 ms) instead of spinning,
// so waiting roles do not steal issue slots from the working ones
TFHE_DEV void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2;\n\t"
      "@!P bra WAITS_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000)
      : "memory");
}

// timeline probes (-DTFHE_FUSED_TRACE): per-unit event clocks of CTA 0, one
// lane of the first warp of each role; compiled out otherwise
#ifdef TFHE_FUSED_TRACE
constexpr int kFTraceN = 128;
#define FTRACE(ev, i)                                                               \
  do {                                                                              \
    if (blockIdx.x == 0 && lane == 0 && (i) < kFTraceN && (warp == 0 || warp == 3 || \
                                                          warp == 4 || warp == 8))  \
      a.trace[(ev) * kFTraceN + (i)] = clock64();                                   \
  } while (0)
#else
#define FTRACE(ev, i) do { } while (0)
#endif

template <int MODE, bool INV>
__global__ void __launch_bounds__(kFThreads, 1) ntt_fused_kernel(const __grid_constant__ FusedArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sD = smem;
  uint8_t* sA1 = sD + kFTwBytes;                 // [2] buffers
  uint8_t* sA2 = sA1 + 2 * kFA1Bytes;
  uint8_t* sRaw = sA2 + kFABytes;
  uint32_t* sW2 = reinterpret_cast<uint32_t*>(sRaw + kFRawBytes);   // [i2][68]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sW2 + 64 * kFW2Pitch);
  uint64_t* raw_full = bar + 0;
  uint64_t* raw_empty = bar + 1;
  uint64_t* a1_full = bar + 2;     // [2]
  uint64_t* a1_empty = bar + 4;    // [2]
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

  constexpr int kW1 = epi1_per_q<MODE>(), kW2 = 3 - kW1;   // warps per lane quarter
  constexpr int kC1 = 64 / kW1, kC2 = 64 / kW2;             // columns per warp
  constexpr int kFEpi2Warp0 = kFEpi1Warp0 + 4 * kW1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int u0 = (int)(a.units * blockIdx.x / gridDim.x);
  const int cnt = (int)(a.units * (blockIdx.x + 1) / gridDim.x) - u0;
  if (tid == 0) {
    mbar_init(raw_full, 1);
    mbar_init(raw_empty, 32 * kFProdWarps);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&a1_full[s], 32 * kFProdWarps);
      mbar_init(&a1_empty[s], 1);
    }
    mbar_init(acc1_full, 1);
    mbar_init(acc1_empty, 128 * kW1);
    mbar_init(a2_full, 128 * kW1);
    mbar_init(a2_empty, 1);
    mbar_init(acc2_full, 1);
    mbar_init(acc2_empty, 128 * kW2);
    mbar_init(tw_full, 1);
    mbar_init(tw_empty, 1);
    mbar_init(epi1_done, 128 * kW1);
    mbar_init(epi2_done, 128 * kW2);
    fence_mbar_init();
  }
  if (warp == kFMmaWarp) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // unit position (limb, member pair), advanced incrementally by every role
  // (no per-unit integer division)
  struct UPos {
    int limb, pair;
  };
  const UPos p0 = {u0 / a.upl, u0 % a.upl};
  auto adv = [&](UPos& p) {
    if (++p.pair == a.upl) {
      p.pair = 0;
      ++p.limb;
    }
  };
  auto last_of_limb = [&](const UPos& p, int it) { return it + 1 == cnt || p.pair + 1 == a.upl; };

  if (warp < kFProdWarps) {
    // -------------------------------------------------------------- producers
    // (thread 0 = warp 0 lane 0 also owns the bulk copies)
    auto issue_raw = [&](const UPos& p) {
      const int b0 = 2 * p.pair, nb = min(2, a.batch - b0);
      const uint32_t bytes = (uint32_t)nb * kFN * 4;
      mbar_arrive_expect_tx(raw_full, bytes);
      bulk_g2s(sRaw, a.in + ((size_t)a.map.in_row[p.limb] * a.batch + b0) * kFN, bytes, raw_full);
    };
    UPos pos = p0, ahead = p0;
    if (tid == 0 && cnt > 0) issue_raw(ahead);
    adv(ahead);
    // 64 warp items per unit: (member b, 4 rows i1, 32 columns i2); warp w takes
    // items w + 3k.  lane -> (r = lane / 8, c = lane % 8): the 16-byte raw reads
    // are conflict-free per 8-lane phase, the padded A1 stores per warp
    const int r = lane >> 3, c = lane & 7;
    int prev_limb = -1;
    uint32_t tw_ph = 0;
    for (int it = 0; it < cnt; ++it, adv(pos)) {
      const int limb = pos.limb;
      mbar_wait(raw_full, it & 1);
      FTRACE(0, it);
      uint4 x[kFItems];
#pragma unroll
      for (int k = 0; k < kFItems; ++k) {
        const int item = min(warp + kFProdWarps * k, 63);
        const int b = item >> 5, ib = (item >> 1) & 15, jb = item & 1;
        x[k] = *reinterpret_cast<const uint4*>(sRaw + (size_t)b * kFN * 4 +
                                               ((4 * ib + r) * kFn1 + 32 * jb + 4 * c) * 4);
      }
      fence_proxy_async_smem();   // raw reads before the next TMA write into the slot
      mbar_arrive(raw_empty);
      if (tid == 0 && it + 1 < cnt) {
        mbar_wait(raw_empty, it & 1);   // every producer has its values in registers
        issue_raw(ahead);
      }
      adv(ahead);
      if (limb != prev_limb) {
        if (tid == 0) {
          if (prev_limb >= 0) {
            // every MMA and epilogue of the previous limb is done with the tables
            mbar_wait(tw_empty, tw_ph);
            mbar_wait(epi1_done, tw_ph);
            mbar_wait(epi2_done, tw_ph);
          }
          const int pr = a.map.prime[limb];
          mbar_arrive_expect_tx(tw_full, kFTwBytes + kFW2TBytes);
          bulk_g2s(sD, a.dft + (size_t)pr * kFTwBytes, kFTwBytes, tw_full);
          bulk_g2s(sW2, a.w2m + (size_t)pr * (kFW2TBytes / 4), kFW2TBytes, tw_full);
        }
        if (prev_limb >= 0) tw_ph ^= 1;
        prev_limb = limb;
      }
      const int buf = it & 1;
      if (it >= 2) mbar_wait(&a1_empty[buf], ((it >> 1) - 1) & 1);   // MMA1(it-2) read it
      FTRACE(1, it);
      uint8_t* dst = sA1 + buf * kFA1Bytes;
#pragma unroll
      for (int k = 0; k < kFItems; ++k) {
        const int item = warp + kFProdWarps * k;
        if (item >= 64) break;
        const int b = item >> 5, ib = (item >> 1) & 15, jb = item & 1;
        const int i1 = 4 * ib + r, m = b * 64 + 32 * jb + 4 * c;
        const uint4 v = x[k];
        uint32_t w[4];
        planes4f(v.x, v.y, v.z, v.w, w);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          *reinterpret_cast<uint32_t*>(dst + mn_off<kFSbo1>(j, m, i1)) = w[j];
      }
      fence_proxy_async_smem();
      mbar_arrive(&a1_full[buf]);
      FTRACE(2, it);
    }
  } else if (warp == kFMmaWarp) {
    // -------------------------------------------------------------- MMA issuer
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
    UPos pos2 = p0;   // position of the next stage-2 unit
    auto stage2 = [&](int v) {
      mbar_wait(a2_full, v & 1);
      FTRACE(4, v);
      if (v >= 1) mbar_wait(acc2_empty, (v - 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        issue(smem_u32(sA2), tmem + 256, 128);
        FTRACE(5, v);
        mma_commit(a2_empty);
        mma_commit(acc2_full);
        if (last_of_limb(pos2, v)) mma_commit(tw_empty);
      }
      __syncwarp();
      adv(pos2);
    };
    int prev_limb = -1;
    uint32_t tw_ph = 0;
    int s2_next = 0;   // next unit whose stage 2 is still to issue
    UPos pos = p0;
    for (int it = 0; it < cnt; ++it, adv(pos)) {
      const int limb = pos.limb;
      if (limb != prev_limb) {
        // the previous limb's stage 2 goes first: its tables are still resident
        while (s2_next < it) stage2(s2_next++);
        if (prev_limb >= 0) tw_ph ^= 1;
        mbar_wait(tw_full, tw_ph);
        prev_limb = limb;
      }
      const int buf = it & 1;
      mbar_wait(&a1_full[buf], (it >> 1) & 1);
      if (it >= 1) mbar_wait(acc1_empty, (it - 1) & 1);
      FTRACE(11, it);
      tc_fence_after();
      if (elect_one()) {
        issue(smem_u32(sA1 + buf * kFA1Bytes), tmem, kFSbo1);
        FTRACE(3, it);
        mma_commit(&a1_empty[buf]);
        mma_commit(acc1_full);
      }
      __syncwarp();
      while (s2_next < it) stage2(s2_next++);
    }
    while (s2_next < cnt) stage2(s2_next++);
  } else if (warp < kFEpi2Warp0) {
    // -------------------------------------------------------------- stage-1 epilogue
    // warp -> TMEM lane quarter q (rows 32q..32q+31), all 64 columns k1 in
    // 16-column chunks: fold, Hadamard, byte-split, store into A2
    const int q = warp & 3, h = (warp - kFEpi1Warp0) >> 2;   // column slice h of kW1
    const int row = q * 32 + lane, b = row >> 6, i2 = row & 63;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    int prev_limb = -1;
    uint32_t tw_ph = 0;
    UPos pos = p0;
    for (int it = 0; it < cnt; ++it, adv(pos)) {
      const int limb = pos.limb;
      if (limb != prev_limb) {
        if (prev_limb >= 0) tw_ph ^= 1;
        mbar_wait(tw_full, tw_ph);   // this limb's W2
        prev_limb = limb;
      }
      const PrimeConst pc = a.pc[a.map.prime[limb]];
      mbar_wait(acc1_full, it & 1);
      FTRACE(6, it);
      tc_fence_after();
#pragma unroll 1
      for (int c0 = kC1 * h; c0 < kC1 * h + kC1; c0 += 16) {
        uint32_t acc[4][16];
#pragma unroll
        for (int i = 0; i < 4; ++i) tmem_ld16(tmem + lane_off + i * 64 + c0, acc[i]);
        tmem_ld_wait();
        if (c0 == kC1 * h + kC1 - 16) {
          tc_fence_before();
          mbar_arrive(acc1_empty);   // buffer drained: MMA1(it+1) may start
        }
        uint32_t w2[16];
#pragma unroll
        for (int e4 = 0; e4 < 4; ++e4) {
          const uint4 t = *reinterpret_cast<const uint4*>(sW2 + i2 * kFW2Pitch + c0 + 4 * e4);
          w2[4 * e4] = t.x; w2[4 * e4 + 1] = t.y; w2[4 * e4 + 2] = t.z; w2[4 * e4 + 3] = t.w;
        }
        uint32_t p[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          // S = fold (twiddles carry R), P = S W2 (W2 carries R): both lazy [0, 2q)
          const uint32_t s = fold4_mont(acc[0][e], acc[1][e], acc[2][e], acc[3][e], pc);
          p[e] = mont_lazy(s, w2[e], pc);
        }
        uint32_t pl[4][4];   // [plane][word]
#pragma unroll
        for (int e4 = 0; e4 < 4; ++e4) {
          uint32_t w[4];
          planes4f(p[4 * e4], p[4 * e4 + 1], p[4 * e4 + 2], p[4 * e4 + 3], w);
#pragma unroll
          for (int j = 0; j < 4; ++j) pl[j][e4] = w[j];
        }
        if (c0 == kC1 * h && it >= 1) mbar_wait(a2_empty, (it - 1) & 1);   // MMA2(it-1) read A2
        if (c0 == kC1 * h) FTRACE(7, it);
        const int m = b * 64 + c0;   // A2 row (b, k1) of the chunk's first k1
#pragma unroll
        for (int j = 0; j < 4; ++j)
          *reinterpret_cast<uint4*>(sA2 + mn_off<128>(j, m, i2)) =
              make_uint4(pl[j][0], pl[j][1], pl[j][2], pl[j][3]);
      }
      fence_proxy_async_smem();
      mbar_arrive(a2_full);
      FTRACE(8, it);
      if (last_of_limb(pos, it)) mbar_arrive(epi1_done);
    }
  } else {
    // -------------------------------------------------------------- stage-2 epilogue
    // kW2 warps per lane quarter, kC2 columns k2 each: pass 1 folds the
    // warp's columns of the row (b, k1) into registers and releases the
    // accumulators (MMA2 of the next unit may start), pass 2 applies the
    // epilogue mode 8 columns at a time; the row's operands (x / base /
    // accumulators / key rows) are strided by n1
    const int q = warp & 3, h = (warp - kFEpi2Warp0) >> 2;
    const int row = q * 32 + lane, b = row >> 6, k1 = row & 63;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    UPos pos = p0;
    for (int it = 0; it < cnt; ++it, adv(pos)) {
      const int limb = pos.limb;
      const PrimeConst pc = a.pc[a.map.prime[limb]];
      const int bm = 2 * pos.pair + b;   // batch member of this row
      const bool valid = bm < a.batch;
      const size_t cofs = (size_t)kC2 * h * kFn1;   // the warp's first column k2
      const size_t orow = ((size_t)a.map.out_row[limb] * a.batch + bm) * kFN + k1 + cofs;
      if ((MODE == EPI_KS_MAC && !a.epi.first) || MODE == EPI_SUB_SCALE) {
        // the next unit's epilogue operand rows (accumulators / x and base,
        // in HBM) -> L2 while this unit runs: the epilogue reads them column
        // chunk by column chunk
        UPos nx = pos;
        adv(nx);
        const int nbm = 2 * nx.pair + b;
        if (it + 1 < cnt && nbm < a.batch) {
          const uint32_t* p0_;
          const uint32_t* p1_;
          if (MODE == EPI_KS_MAC) {
            const size_t nrow = ((size_t)a.map.out_row[nx.limb] * a.batch + nbm) * kFN + k1 + cofs;
            p0_ = a.epi.acc_b + nrow;
            p1_ = a.epi.acc_a + nrow;
          } else {
            p0_ = a.epi.x + ((size_t)a.epi.x_row[nx.limb] * a.batch + nbm) * kFN + k1 + cofs;
            const int br = a.epi.base_row[nx.limb];
            p1_ = br >= 0 ? a.epi.base + ((size_t)br * a.batch + nbm) * kFN + k1 + cofs : nullptr;
          }
#pragma unroll 4
          for (int e = 0; e < kC2; ++e) {
            prefetch_l2(p0_ + (size_t)e * kFn1);
            if (p1_) prefetch_l2(p1_ + (size_t)e * kFn1);
          }
        }
      }
      mbar_wait(acc2_full, it & 1);
      FTRACE(9, it);
      tc_fence_after();
      uint32_t y[kC2];
#pragma unroll
      for (int cc = 0; cc < kC2; cc += 8) {
        uint32_t acc[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i) tmem_ld8(tmem + 256 + lane_off + i * 64 + kC2 * h + cc, acc[i]);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 8; ++e)
          y[cc + e] = fold4_mont(acc[0][e], acc[1][e], acc[2][e], acc[3][e], pc);   // lazy
      }
      tc_fence_before();
      mbar_arrive(acc2_empty);   // accumulators drained: MMA2(it+1) may start
      if (valid) {
#pragma unroll
        for (int e = 0; e < kC2; ++e) y[e] = corr(y[e], pc.q);
        if (MODE == EPI_STORE) {
          uint32_t* o = a.out + orow;
#pragma unroll
          for (int e = 0; e < kC2; ++e) o[e * kFn1] = y[e];
        } else if (MODE == EPI_SUB_SCALE) {
          const uint32_t* xs = a.epi.x + ((size_t)a.epi.x_row[limb] * a.batch + bm) * kFN + k1 + cofs;
          const int br = a.epi.base_row[limb];
          const uint32_t* bs =
              br >= 0 ? a.epi.base + ((size_t)br * a.batch + bm) * kFN + k1 + cofs : nullptr;
          const uint32_t ss = a.epi.s[limb], ssp = a.epi.s_shoup[limb];
          uint32_t* o = a.out + orow;
#pragma unroll
          for (int cc = 0; cc < kC2; cc += 8) {
            uint32_t xv[8], bv[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              xv[e] = xs[(cc + e) * kFn1];
              if (bs) bv[e] = bs[(cc + e) * kFn1];
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              uint32_t t = mul_shoup(sub_mod(xv[e], y[cc + e], pc.q), ss, ssp, pc.q);
              if (bs) t = add_mod(bv[e], t, pc.q);
              o[(cc + e) * kFn1] = t;
            }
          }
        } else {   // EPI_KS_MAC: y arrives as y R (the pre-twist carries R^2)
          const size_t kr = (size_t)a.epi.key_row[limb] * kFN + k1 + cofs;
          uint32_t* ob = a.epi.acc_b + orow;
          uint32_t* oa = a.epi.acc_a + orow;
          const bool first = a.epi.first != 0;
#pragma unroll
          for (int cc = 0; cc < kC2; cc += 8) {
            uint32_t kb[8], ka[8], pb[8], pa[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              kb[e] = __ldg(a.epi.kb + kr + (cc + e) * kFn1);
              ka[e] = __ldg(a.epi.ka + kr + (cc + e) * kFn1);
              if (!first) {
                pb[e] = ob[(cc + e) * kFn1];
                pa[e] = oa[(cc + e) * kFn1];
              }
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const uint32_t tb = corr(mont_lazy(y[cc + e], kb[e], pc), pc.q);
              const uint32_t ta = corr(mont_lazy(y[cc + e], ka[e], pc), pc.q);
              ob[(cc + e) * kFn1] = first ? tb : add_mod(pb[e], tb, pc.q);
              oa[(cc + e) * kFn1] = first ? ta : add_mod(pa[e], ta, pc.q);
            }
          }
        }
      }
      FTRACE(10, it);
      if (last_of_limb(pos, it)) mbar_arrive(epi2_done);
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
  std::vector<uint32_t> w2((size_t)np * 64 * kFW2Pitch, 0), w2ks;
  for (int inv = 0; inv < 2; ++inv) {
    if (!inv) w2ks.assign(w2.size(), 0);
    for (int p = 0; p < np; ++p) {
      const uint32_t q = c.primes[p];
      const uint32_t psi = inv ? powmod_f(c.psis[p], q - 2, q) : c.psis[p];
      const uint32_t w = powmod_f(psi, 128, q);   // primitive 64th root (inverse: w^-1)
      const uint32_t R = (uint32_t)(((uint64_t)1 << 32) % q);
      const uint32_t n_inv = powmod_f(kFN, q - 2, q);
      std::vector<uint32_t> pw(2 * kFN);
      pw[0] = 1;
      for (int e = 1; e < 2 * kFN; ++e) pw[e] = mulmod_f(pw[e - 1], psi, q);
      uint32_t wp[64], tw[64], tw_inv[64];
      wp[0] = 1;
      for (int e = 1; e < 64; ++e) wp[e] = mulmod_f(wp[e - 1], w, q);
      // the twist: forward column twist t[k] = psi^(64 k) of W1; inverse row
      // twist u[c] = psi^(-64 c) n^-1 of W3 (see the header)
      for (int k = 0; k < 64; ++k) {
        tw[k] = inv ? mulmod_f(pw[64 * k], n_inv, q) : pw[64 * k];
        tw_inv[k] = powmod_f(tw[k], q - 2, q);
      }
      uint8_t* base = tiles.data() + (size_t)p * kFTwBytes;
      for (int cc = 0; cc < 64; ++cc)        // output column (k1 or k2)
        for (int k = 0; k < 64; ++k) {       // contraction index (i1 or i2)
          // T[cc][k] R: forward w^(cc k) t[k], inverse u[cc] w^-(cc k)
          const uint32_t t = mulmod_f(mulmod_f(wp[(cc * k) & 63], tw[inv ? cc : k], q), R, q);
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
      // Hadamard W2 R (forward psi^(2 k1 i2 + i2), inverse psi^-(2 k1 i2 + k1),
      // params.py:198-228), divided by the twist the shared table adds: stage 2
      // multiplies by t[i2] (forward), stage 1 by u[k1] (inverse)
      for (int k1 = 0; k1 < 64; ++k1)
        for (int i2 = 0; i2 < 64; ++i2) {
          const int e = inv ? (2 * k1 * i2 + k1) : (2 * k1 * i2 + i2);
          const uint32_t v = mulmod_f(mulmod_f(pw[e % (2 * kFN)], tw_inv[inv ? k1 : i2], q), R, q);
          w2[((size_t)p * 64 + i2) * kFW2Pitch + k1] = v;
          // key-switch MAC: one more R, so stage 2 yields y R (Montgomery form)
          if (!inv) w2ks[((size_t)p * 64 + i2) * kFW2Pitch + k1] = mulmod_f(v, R, q);
        }
    }
    auto up = [&](void** dst, const void* src, size_t bytes) {
      return cudaMalloc(dst, bytes) == cudaSuccess &&
             cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice) == cudaSuccess;
    };
    if (!up(reinterpret_cast<void**>(&c.d_fdft[inv]), tiles.data(), tiles.size()) ||
        !up(reinterpret_cast<void**>(&c.d_fw2[inv]), w2.data(), w2.size() * 4) ||
        (!inv && !up(reinterpret_cast<void**>(&c.d_fw2_ks), w2ks.data(), w2ks.size() * 4))) {
      set_error("fused ntt table upload failed");
      return 3;
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
  a.w2m = inverse ? c.d_fw2[1] : (mode == EPI_KS_MAC ? c.d_fw2_ks : c.d_fw2[0]);
  a.pc = c.d_pc;
  a.batch = batch;
  a.upl = (batch + 1) / 2;
  a.inverse = inverse ? 1 : 0;
  a.units = (long long)a.upl * map.n;
  if (a.units >= (1ll << 31)) return -1;
  a.map = map;
  if (epi) a.epi = *epi;
  else a.epi.mode = EPI_STORE;
  const int grid = (int)std::min<long long>(c.sms, a.units);
  if (grid <= 0) return 0;
#ifdef TFHE_FUSED_TRACE
  static unsigned long long* tbuf = nullptr;
  if (!tbuf) cudaMalloc(&tbuf, 16 * kFTraceN * 8);
  cudaMemsetAsync(tbuf, 0, 16 * kFTraceN * 8, st);
  a.trace = tbuf;
#endif
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kFSmem);
    prof_begin("ntt_fused_kernel", st);
    kern<<<grid, kFThreads, kFSmem, st>>>(a);
    prof_end(st);
  };
  if (inverse) {
    if (mode == EPI_SUB_SCALE) go(ntt_fused_kernel<EPI_SUB_SCALE, true>);
    else go(ntt_fused_kernel<EPI_STORE, true>);
  } else {
    if (mode == EPI_SUB_SCALE) go(ntt_fused_kernel<EPI_SUB_SCALE, false>);
    else if (mode == EPI_KS_MAC) go(ntt_fused_kernel<EPI_KS_MAC, false>);
    else go(ntt_fused_kernel<EPI_STORE, false>);
  }
#ifdef TFHE_FUSED_TRACE
  {
    std::vector<unsigned long long> h(16 * kFTraceN);
    cudaMemcpy(h.data(), tbuf, h.size() * 8, cudaMemcpyDeviceToHost);
    static int seq = 0;
    char fn[256];
    snprintf(fn, sizeof(fn), "gpurun_out/ftrace_%d.bin", seq++);
    if (FILE* f = fopen(fn, "wb")) {
      fwrite(h.data(), 8, h.size(), f);
      fclose(f);
    }
  }
#endif
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("fused ntt launch: ") + cudaGetErrorString(e));
    return 3;
  }
  return 0;
}

}  // namespace tfhe
