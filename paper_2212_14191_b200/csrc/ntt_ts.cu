// Twiddle-resident tensor-core NTT stages (n1, n2 in {128, 256}; N = 2^14..2^16;
// at N = 2^13 stage 2 only, after the resident small-n stage 1: Ctx::ts_stage2).
//
// Same math as ntt_tc.cu (TensorFHE's byte-sliced GEMM formulation, ref
// ntt.py:212-340), re-tiled so the CONSTANT operand never streams:
//
//   D[r][col] = sum_k T[r][k] * X[k][col]        (mod q)
//     stage 1: r = k1, k = i1, col = (b, i2), T = W1, X = A_b      -> P = D .* W2
//     stage 2: r = k2, k = i2, col = (b, k1), T = W3^T, X = P_b^T  -> out[k2*n1 + k1]
//
// * A operand (twiddle byte planes T_i, i = 0..3) lives in TMEM for the whole
//   lifetime of a (limb, 128-row half) work group: tcgen05.mma ... [a_tmem]
//   ("TS" form).  Nothing twiddle-related is re-read per tile.
// * B operand (data) streams through a 6-stage smem ring: 16 data columns per
//   chunk, split into byte planes X_j by 4 producer warps and laid out as
//   B' = [X_0 | X_1 | X_2 | X_3] along N (N = 64).
// * Byte weights: T X = sum_{s=0..6} 2^(8s) C_s with C_s = sum_{i+j=s} T_i X_j.
//   One MMA (A = T_i, B = B') writes D[:, 16 j + c] = T_i X_j; placing its
//   output at column 16 i makes block 16 (i+j) accumulate exactly C_{i+j}
//   ("shifted window"), so 4 MMAs per K-step produce all 7 accumulators
//   (7 x 16 TMEM columns, double-buffered).  C_s < 4 * 256 * 255^2 < 2^26.
// * Epilogue warps fold sum C_s 2^(8s) (2^(8s) mod q for s >= 4) in 64 bits,
//   Barrett-reduce, apply W2 (stage 1) or the fused output epilogue
//   (stage 2) and store through a smem transpose (full 32-byte sectors).
//
// Roles: warps 0-3 data producers, warps 4-11 epilogue (+ twiddle -> TMEM
// loads; two warps per TMEM lane quarter, 8 columns each), warp 12 TMEM
// allocation + single-thread MMA issue.  Persistent grid
// (one CTA per SM); with two 128-row halves the CTAs run in pairs over the
// same data range so the second read of each data chunk hits L2.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda.h>

#include "common.cuh"
#include "tfhe_internal.h"

namespace tfhe {

namespace {

constexpr int kNC = 16;                  // data columns per chunk
constexpr int kRing = 4;                 // smem operand ring depth (chunks)
// 4 warpgroups: producers (warps 0-3), epilogue (4-11), MMA issuer (warp 12;
// warps 13-15 idle).  Registers are rebalanced with setmaxnreg: each SMSP
// holds one warp of every warpgroup, so 96 + 2 * 176 + 64 <= 512 per lane.
constexpr int kEpiWarps = 8;              // two epilogue warps per TMEM lane quarter
constexpr int kCW = kNC / (kEpiWarps / 4);  // chunk columns per epilogue warp
constexpr int kMmaWarp = 4 + kEpiWarps;
// MMA-issuing warps (chunks round-robin): while one issuer waits on its
// barriers / steps its bookkeeping the other keeps the tensor queue fed
#ifndef TFHE_MMA_ISSUERS
#define TFHE_MMA_ISSUERS 2
#endif
constexpr int kMmaIssuers = TFHE_MMA_ISSUERS;
constexpr int kThreadsTS = 512;
constexpr int kRegsProducer = 96, kRegsEpilogue = 176, kRegsMma = 64;
constexpr uint32_t kAccCol0 = 256, kAccCol1 = 384;
// Performance-experiment knobs (env TFHE_DBG) exist only in builds with
// -DTFHE_TS_DBG; normal builds compile them away.
#ifdef TFHE_TS_DBG
#define kDbg (a.dbg)
#elif defined(TFHE_TS_DBG_VAL)
#define kDbg (TFHE_TS_DBG_VAL)
#else
#define kDbg 0
#endif

struct TsArgs {
  const uint32_t* in;
  uint32_t* out;
  const uint32_t* twa;  // [prime][half][128][4][K/4] words
  const uint32_t* w2;
  const uint32_t* w2s;
  const PrimeConst* pc;
  int n, n1, n2, batch;
  int R;      // data columns per member (stage 1: n2, stage 2: n1)
  int H;      // 128-row twiddle halves
  int C;      // chunks per limb
  int n_limbs;
  int S;      // stage-2 input slices per (limb, chunk) group (EPI_KS_ACC), else 1;
              // the stage-2 input row of (slice s, limb l) is s * n_limbs + l
  unsigned long long* trace;  // TFHE_TS_TRACE builds: per-chunk event clocks of CTA 0
  int dbg;    // perf experiments only (env TFHE_DBG): 1 = producers skip global loads,
              // 2 = epilogue skips math/stores; results are garbage when set
  CUtensorMap tmap;  // TMA view of the input (stage 1: [rows*B][n1][n2]; stage 2:
                     // blocked P [rows*B][n2/16][n1][16], 64-byte swizzle)
  LimbMap map;
  EpiArgs epi;
};

#ifdef TFHE_TS_TRACE
constexpr int kTraceN = 512;
#define TS_TRACE(ev, i)                                                        \
  do {                                                                         \
    if (blockIdx.x == 0 && lane == 0 && (i) < kTraceN)                         \
      a.trace[(ev) * kTraceN + (i)] = clock64();                               \
  } while (0)
#else
#define TS_TRACE(ev, i) do { } while (0)
#endif

template <int K>
__host__ __device__ constexpr int ring_stage_bytes() { return (K / 32) * 2048; }

TFHE_DEV void planes4(uint32_t v0, uint32_t v1, uint32_t v2, uint32_t v3, uint32_t (&w)[4]) {
  uint32_t lo01 = __byte_perm(v0, v1, 0x5140), hi01 = __byte_perm(v0, v1, 0x7362);
  uint32_t lo23 = __byte_perm(v2, v3, 0x5140), hi23 = __byte_perm(v2, v3, 0x7362);
  w[0] = __byte_perm(lo01, lo23, 0x5410);
  w[1] = __byte_perm(lo01, lo23, 0x7632);
  w[2] = __byte_perm(hi01, hi23, 0x5410);
  w[3] = __byte_perm(hi01, hi23, 0x7632);
}

// byte offset of (B' row, k) inside one chunk stage: per K-step kc a 64-row x
// 32-byte K-major SWIZZLE_NONE tile (LBO = 1024, SBO = 128)
TFHE_DEV uint32_t ring_off(int row, int k) {
  const int kc = k >> 5, kk = k & 31;
  return (uint32_t)(kc * 2048 + (kk >> 4) * 1024 + (row >> 3) * 128 + (row & 7) * 16 + (kk & 15));
}

// iteration state shared by the three roles: every role walks the same unit
// sequence (limb, chunk) and the same ring / accumulator phases.  Chunks of a
// limb run member-major (c = b * R / kNC + x0 / kNC): a member's columns are
// contiguous in memory, which measured ~3% faster than grouping the members
// that share a column block -- except for the fused key-switch epilogue
// (EPI_KS_ACC), whose key tiles depend on the column block only: there the
// chunks run column-block-major (c = (x0 / kNC) * batch + b) so consecutive
// units of a CTA reuse the same S key tiles (L2-resident) across the batch
// instead of streaming them once per member.
struct UnitIter {
  int limb, c, b, x0;
  int sl;         // slice within the (limb, chunk) group (EPI_KS_ACC)
  int S;          // slices per group
  int R;          // data columns per member
  int B;          // batch members (column-block-major order), 0 = member-major
  int s;          // ring slot
  uint32_t rph;   // ring phase parity of slot s
  int ab;         // accumulator buffer
  uint32_t aph;   // accumulator phase parity
  TFHE_DEV void init(long long g0, int C, int R_, int S_, int B_ = 0) {
    limb = (int)(g0 / C);
    c = (int)(g0 % C);
    R = R_;
    B = B_;
    if (B) {
      b = c % B;
      x0 = c / B * kNC;
    } else {
      b = c * kNC / R;
      x0 = c * kNC % R;
    }
    sl = 0; S = S_;
    s = 0; rph = 0; ab = 0; aph = 0;
  }
  TFHE_DEV void next(int C) {
    if (++sl == S) {
      sl = 0;
      if (++c == C) { c = 0; ++limb; b = 0; x0 = 0; }
      else if (B) {
        if (++b == B) { b = 0; x0 += kNC; }
      } else if ((x0 += kNC) == R) { x0 = 0; ++b; }
    }
    if (++s == kRing) { s = 0; rph ^= 1; }
    ab ^= 1;
    if (ab == 0) aph ^= 1;
  }
};

// MN-major variant (stage 1): per K-step a tile of 4 planes x 4 K-groups of
// 128-byte core matrices (8 k rows x 16 column bytes); LBO (K) = 128,
// SBO (N, = plane) = 512.  (plane j, column c, k) -> byte offset
TFHE_DEV uint32_t ring_off_mn(int j, int c, int k) {
  const int kc = k >> 5, kk = k & 31;
  return (uint32_t)(kc * 2048 + j * 512 + (kk >> 3) * 128 + (kk & 7) * 16 + c);
}


// Epilogue staging per warp: in[2][T] operand tiles (double-buffered
// prefetch) | out[2] transpose tiles, 1 KB each; T depends on what the
// epilogue reads: W2 (stage 1), nothing (store), x + base (ModDown /
// rescale), key rows + accumulators (fused key switch).
template <int STAGE, int MODE>
__host__ __device__ constexpr int in_tiles() {
  return STAGE == 1 ? 1 : MODE == EPI_STORE ? 0 : MODE == EPI_SUB_SCALE ? 2 : 4;
}
template <int STAGE, int MODE>
__host__ __device__ constexpr int warp_stg_bytes() { return (2 * in_tiles<STAGE, MODE>() + 2) * 1024; }
// TMA raw-data ring depth: whatever shared memory the operand ring and the
// epilogue staging leave (up to 8 chunks in flight hides DRAM latency)
constexpr int kSmemBudget = 226 * 1024;
template <int STAGE, int K, int MODE>
__host__ __device__ constexpr int raw_slots() {
  return (kSmemBudget - kRing * ring_stage_bytes<K>() - kEpiWarps * warp_stg_bytes<STAGE, MODE>()) /
                     (K * 64) > 8
             ? 8
             : (kSmemBudget - kRing * ring_stage_bytes<K>() -
                kEpiWarps * warp_stg_bytes<STAGE, MODE>()) / (K * 64);
}

// 32 rows x 64 B staging, 16-byte chunks XOR-swizzled so both the row-wise
// and the 4-lanes-per-row accesses are bank-conflict free
TFHE_DEV uint32_t stg_off(int row, int q) { return (uint32_t)(row * 64 + 16 * (q ^ ((row >> 1) & 3))); }
// 32 rows x 32 B epilogue tile: row-wise (1 lane per row) and 2-lanes-per-row
// 16-byte accesses are both conflict free
TFHE_DEV uint32_t stg8_off(int row, int q) { return (uint32_t)(row * 32 + 16 * (q ^ ((row >> 2) & 1))); }

TFHE_DEV void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc)
               : "memory");
}
TFHE_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
TFHE_DEV void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
TFHE_DEV void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// v < q 2^32 -> v 2^-32 mod q in [0, 2q).  Stage 1 leaves P in [0, 2q): stage 2
// only byte-splits it (any 32-bit value; the fold bounds hold) and the result
// is exact mod q
TFHE_DEV uint32_t mont_reduce_lazy(uint64_t v, const PrimeConst& pc) {
  const uint32_t mq = (uint32_t)v * pc.qneg_inv;
  return (uint32_t)((v + (uint64_t)mq * pc.q) >> 32);
}
TFHE_DEV uint32_t mont_reduce(uint64_t v, const PrimeConst& pc) {
  const uint32_t mq = (uint32_t)v * pc.qneg_inv;
  const uint32_t t = (uint32_t)((v + (uint64_t)mq * pc.q) >> 32);
  return t >= pc.q ? t - pc.q : t;
}

// x = sum_{s=0..6} C_s 2^(8s) (C_s < 2^26, x < 2^76) -> x * 2^-64 mod q, by two
// Montgomery rounds: A = C_0..C_3 part (< 2^51), t = A 2^-32 (< 2^30), then
// u = t + C_4 + C_5 2^8 + C_6 2^16 (< 2^44, built on the ALU pipe) and
// y = u 2^-32 < q + 2^12.  Four multiplies instead of seven 64-bit ones: the
// epilogue is bound by the integer-multiply pipe.  kLazy skips the final
// correction (y < q + 2^12): a following Montgomery product with a factor < q
// stays < q 2^32 and corrects once itself.
template <bool kLazy = false>
TFHE_DEV uint32_t fold_redc(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t c4,
                            uint32_t c5, uint32_t c6, const PrimeConst& pc) {
  const uint64_t A = (uint64_t)c0 + ((uint64_t)c1 << 8) + ((uint64_t)c2 << 16) + ((uint64_t)c3 << 24);
  const uint32_t m0 = (uint32_t)A * pc.qneg_inv;
  const uint32_t t = (uint32_t)((A + (uint64_t)m0 * pc.q) >> 32);
  uint32_t lo, hi;
  asm("{\n\t.reg .u32 s5, h5, s6, h6;\n\t"
      "shl.b32 s5, %3, 8;\n\tshr.b32 h5, %3, 24;\n\t"
      "shl.b32 s6, %4, 16;\n\tshr.b32 h6, %4, 16;\n\t"
      "add.u32 %0, %2, %5;\n\t"
      "add.cc.u32 %0, %0, s5;\n\taddc.u32 %1, h5, h6;\n\t"
      "add.cc.u32 %0, %0, s6;\n\taddc.u32 %1, %1, 0;\n\t}"
      : "=r"(lo), "=r"(hi)
      : "r"(c4), "r"(c5), "r"(c6), "r"(t));
  const uint32_t m1 = lo * pc.qneg_inv;
  const uint32_t y = (uint32_t)(((((uint64_t)hi << 32) | lo) + (uint64_t)m1 * pc.q) >> 32);
  if (kLazy) return y;
  return y >= pc.q ? y - pc.q : y;
}

template <int STAGE, int K, int MODE>
__global__ void __launch_bounds__(kThreadsTS, 1) ntt_ts_kernel(const __grid_constant__ TsArgs a) {
  constexpr int kStageBytes = ring_stage_bytes<K>();
  constexpr int KC = K / 32;
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int kRawBytes = K * 64;            // one raw data chunk (16 u32 x K)
  constexpr int kRaw = raw_slots<STAGE, K, MODE>();
  static_assert(kRaw >= 2, "shared memory budget leaves no TMA ring");
  constexpr int kWarpStg = warp_stg_bytes<STAGE, MODE>();
  constexpr int kStgBytes = kEpiWarps * kWarpStg;
  constexpr int kInBuf = in_tiles<STAGE, MODE>() * 1024;  // one prefetch buffer
  uint8_t* stg = smem + kRing * kStageBytes;  // epilogue staging
  uint64_t* b_full = reinterpret_cast<uint64_t*>(stg + kStgBytes + kRaw * kRawBytes);
  uint64_t* b_empty = b_full + kRing;
  uint64_t* acc_full = b_empty + kRing;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* tw_full = acc_empty + 2;
  uint64_t* raw_full = tw_full + 1;
  uint64_t* raw_empty = raw_full + kRaw;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(raw_empty + kRaw);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // work split: units u = limb * C + chunk over this CTA's half
  int h, grp, groups;
  if (a.H == 2) {
    h = blockIdx.x & 1;
    grp = blockIdx.x >> 1;
    groups = gridDim.x >> 1;
  } else {
    h = 0;
    grp = blockIdx.x;
    groups = gridDim.x;
  }
  // groups = (limb, chunk); each group is S consecutive units (one per slice)
  const long long G = (long long)a.n_limbs * a.C;
  const long long g0 = G * grp / groups;
  const int cnt = (int)(G * (grp + 1) / groups - g0) * a.S;
  const int C = a.C;

  if (tid == 0) {
    for (int s = 0; s < kRing; ++s) {
      mbar_init(&b_full[s], 128);
      mbar_init(&b_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 32 * kEpiWarps);
    }
    mbar_init(tw_full, 32 * kEpiWarps);
    for (int s = 0; s < kRaw; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&raw_empty[s], 128);
    }
    fence_mbar_init();
  }
  if (warp == kMmaWarp) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  UnitIter w;
  w.init(g0, C, a.R, a.S, MODE == EPI_KS_ACC && !(kDbg & 65536) ? a.batch : 0);
  // Each role's register budget is set at the top of its own branch so that
  // ptxas allocates every role's code under the matching setmaxnreg limit.
  if (warp < 4) {
    reg_dealloc<kRegsProducer>();
    if (kDbg & (4 | 512)) goto role_done;
    // ---------------------------------------------------------------- producers
    // Raw data chunks arrive by TMA (one elected thread, kRaw chunks in
    // flight) in a staging ring; the 4 producer warps byte-split them into the
    // MMA operand ring.
    // Stage 1 (X_b[k][x0 + c], columns contiguous): raw [K rows][16 u32];
    // B' is stored MN-major -- each thread reads 16 B (4 columns of one k
    // row) and writes one 4-byte word per byte plane; a warp covers 8 k rows
    // x 64 B = one conflict-free 128-byte span per plane.
    // Stage 2 (blocked P, k contiguous): raw [K/16][16 rows][16 u32] with the
    // TMA 64-byte swizzle; B' is stored K-major -- each thread reads 16
    // consecutive k of one row and writes one 16-byte vector per plane; a
    // quarter warp covers 8 rows = 8 distinct 16-byte slots on both sides.
    const int c4 = (tid & 3) * 4, krow0 = tid >> 2;   // stage 1 mapping
    const int col = tid & 15, kb0 = tid >> 4;         // stage 2 mapping
    uint8_t* raw = smem + kRing * kStageBytes + kStgBytes;
    auto issue_raw = [&](const UnitIter& it, int slot) {
      uint8_t* dst = raw + slot * kRawBytes;
      mbar_arrive_expect_tx(&raw_full[slot], kRawBytes);
      if (STAGE == 1)
        tma_load_3d(dst, &a.tmap, it.x0, 0, a.map.in_row[it.limb] * a.batch + it.b,
                    &raw_full[slot]);
      else
        tma_load_4d(dst, &a.tmap, 0, it.x0, 0,
                    (it.sl * a.n_limbs + it.limb) * a.batch + it.b, &raw_full[slot]);
    };
    UnitIter ahead = w;
    if (tid == 0 && !(kDbg & 32)) {
      for (int i = 0; i < kRaw && i < cnt; ++i, ahead.next(C)) issue_raw(ahead, i);
    }
    for (int i = 0; i < cnt; ++i, w.next(C)) {
      const int rs = i % kRaw;
      const uint32_t rph = (uint32_t)((i / kRaw) & 1);
      if (warp == 0) TS_TRACE(7, i);
      if (!(kDbg & 32)) mbar_wait(&raw_full[rs], rph);
      if (warp == 0) TS_TRACE(8, i);
      const uint8_t* rw = raw + rs * kRawBytes;
      if (i >= kRing) mbar_wait(&b_empty[w.s], w.rph ^ 1);
      if (warp == 0) TS_TRACE(9, i);
      uint8_t* st = smem + w.s * kStageBytes;
      if (kDbg & 16) {
      } else if (STAGE == 1) {
#pragma unroll
        for (int m = 0; m < K / 32; ++m) {
          const int k = krow0 + 32 * m;
          const uint4 x = *reinterpret_cast<const uint4*>(rw + k * 64 + c4 * 4);
          uint32_t pw[4];
          planes4(x.x, x.y, x.z, x.w, pw);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            *reinterpret_cast<uint32_t*>(st + ring_off_mn(j, c4, k)) = pw[j];
        }
      } else {
#pragma unroll
        for (int t = 0; t < K / 128; ++t) {
          const int kb = kb0 + 8 * t, k0 = kb * 16;
          uint32_t v[16];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint4 x = *reinterpret_cast<const uint4*>(rw + kb * 1024 + stg_off(col, q));
            v[4 * q] = x.x; v[4 * q + 1] = x.y; v[4 * q + 2] = x.z; v[4 * q + 3] = x.w;
          }
          uint32_t pw[4][4];  // [group][plane]
#pragma unroll
          for (int g = 0; g < 4; ++g) planes4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3], pw[g]);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            *reinterpret_cast<uint4*>(st + ring_off(j * 16 + col, k0)) =
                make_uint4(pw[0][j], pw[1][j], pw[2][j], pw[3][j]);
        }
      }
      fence_proxy_async_smem();
      mbar_arrive(&b_full[w.s]);
      mbar_arrive(&raw_empty[rs]);
      if (warp == 0) TS_TRACE(10, i);
      if (tid == 0 && i + kRaw < cnt && !(kDbg & 32)) {
        // refill this raw slot once every producer thread has read it
        mbar_wait(&raw_empty[rs], rph);
        issue_raw(ahead, rs);
        ahead.next(C);
      }
    }
  } else if (warp < 4 + kEpiWarps) {
    reg_alloc<kRegsEpilogue>();
    if (kDbg & (4 | 1024)) goto role_done;
    // ---------------------------------------------------------------- epilogue
    // Two warps per TMEM lane quarter (one per SMSP pair of the two epilogue
    // warpgroups): warp 4 + 4 hf + wq owns rows wq*32..+31 and chunk columns
    // [8 hf, 8 hf + 8).  Two independent warps per SMSP hide the latency of the
    // 64-bit fold / Montgomery chains that one warp alone stalls on.
    const int wq = warp & 3, hf = (warp - 4) >> 2, cb = hf * kCW;
    const int m = wq * 32 + lane;          // TMEM lane = twiddle row within the half
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    uint8_t* wstg = stg + (warp - 4) * kWarpStg;   // in[2][T] tiles | out[2] tiles (1 KB each)
    constexpr int mode = STAGE == 2 ? MODE : EPI_STORE;
    // Epilogue operands (W2 tile, x/base rows, key rows, accumulators) are
    // fetched one chunk ahead with cp.async into a double-buffered staging
    // area: 32 rows x 32 bytes per tile, 2 lanes per row (full sectors).
    auto prefetch = [&](const UnitIter& it, int buf) {
      uint8_t* dstb = wstg + buf * kInBuf;
      if (STAGE == 1) {
        // W2 * 2^96 in [prime][i2][k1] layout: for each of this warp's 8 i2
        // columns the warp's 32 k1 rows are 128 contiguous bytes -> staged as
        // [8][32] words
        const int pr = a.map.prime[it.limb];
        const uint32_t* wp = a.w2 + (size_t)pr * a.n + (size_t)(it.x0 + cb) * a.n1 + h * 128 + wq * 32;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int idx = q * 32 + lane, e = idx >> 3, part = idx & 7;
          cp_async16(dstb + e * 128 + part * 16, wp + (size_t)e * a.n1 + part * 4);
        }
        return;
      }
      const size_t wrow = (size_t)(h * 128 + wq * 32) * a.n1 + it.x0 + cb;  // warp's first row
      const uint32_t* src[4] = {nullptr, nullptr, nullptr, nullptr};
      if (mode == EPI_SUB_SCALE) {
        src[0] = a.epi.x + ((size_t)a.epi.x_row[it.limb] * a.batch + it.b) * a.n + wrow;
        const int br = a.epi.base_row[it.limb];
        if (br >= 0) src[1] = a.epi.base + ((size_t)br * a.batch + it.b) * a.n + wrow;
      } else if (mode == EPI_KS_MAC) {
        src[0] = a.epi.kb + (size_t)a.epi.key_row[it.limb] * a.n + wrow;
        src[1] = a.epi.ka + (size_t)a.epi.key_row[it.limb] * a.n + wrow;
        if (!a.epi.first) {
          const size_t ar = ((size_t)a.map.out_row[it.limb] * a.batch + it.b) * a.n + wrow;
          src[2] = a.epi.acc_b + ar;
          src[3] = a.epi.acc_a + ar;
        }
      } else if (mode == EPI_KS_ACC) {
        // key rows of slice j0 + sl for this target; accumulators at group start
        const uint32_t* kbj = a.epi.key + (size_t)(a.epi.j0 + it.sl) * a.epi.key_pair +
                              (size_t)a.epi.key_row[it.limb] * a.n + wrow;
        src[0] = kbj;
        src[1] = kbj + a.epi.key_pair / 2;
        if (it.sl == 0 && a.epi.init_acc[it.limb]) {
          const size_t ar = ((size_t)a.map.out_row[it.limb] * a.batch + it.b) * a.n + wrow;
          src[2] = a.epi.acc_b + ar;
          src[3] = a.epi.acc_a + ar;
        }
      }
#pragma unroll
      for (int tI = 0; tI < 4; ++tI) {
        if (!src[tI]) continue;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int r = 16 * q + (lane >> 1), p = lane & 1;
          cp_async16(dstb + tI * 1024 + stg8_off(r, p), src[tI] + (size_t)r * a.n1 + 4 * p);
        }
      }
    };
    auto read_row = [&](int buf, int tI, uint32_t (&v)[kCW]) {
      const uint8_t* t = wstg + buf * kInBuf + tI * 1024;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        uint4 u = *reinterpret_cast<const uint4*>(t + stg8_off(lane, q));
        v[4 * q] = u.x; v[4 * q + 1] = u.y; v[4 * q + 2] = u.z; v[4 * q + 3] = u.w;
      }
    };
    // coalesced store of this warp's 32 rows x 8 values (row stride in elements):
    // transposed through smem so each store instruction writes 16 full sectors
    auto store_tile = [&](int oI, const uint32_t (&v)[kCW], uint32_t* dst, size_t row_stride) {
      uint8_t* t = wstg + 2 * kInBuf + oI * 1024;
#pragma unroll
      for (int q = 0; q < 2; ++q)
        *reinterpret_cast<uint4*>(t + stg8_off(lane, q)) =
            make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int r = 16 * q + (lane >> 1), p = lane & 1;
        *reinterpret_cast<uint4*>(dst + (size_t)r * row_stride + 4 * p) =
            *reinterpret_cast<const uint4*>(t + stg8_off(r, p));
      }
    };
    UnitIter ahead = w;
    if (cnt > 0 && !(kDbg & 64)) prefetch(ahead, 0);
    uint32_t regb[kCW], rega[kCW];   // EPI_KS_ACC group accumulators
    uint64_t lzb[kCW], lza[kCW];     // ... and their pending lazy sums
    int npend = 0;
    cp_async_commit();
    int prev = -1;
    PrimeConst pc;
    for (int i = 0; i < cnt; ++i, w.next(C)) {
      const int limb = w.limb;
      const int prime = a.map.prime[limb];
      const int buf = i & 1;
      if (limb != prev) {
        // per-prime constants stay in registers for the whole limb (a
        // per-chunk global load would sit on the fold's critical path)
        pc = a.pc[prime];
        // load this (limb, half)'s twiddle planes into TMEM columns [0, K):
        // each of the quarter's two warps writes half of the columns
        prev = limb;
        const uint32_t* src = a.twa + (((size_t)prime * a.H + h) * 128 + m) * K;
#pragma unroll 1
        for (int w0 = hf * (K / 2); w0 < (hf + 1) * (K / 2) && !(kDbg & 2048); w0 += 16) {
          uint32_t r[16];
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            uint4 v = __ldg(reinterpret_cast<const uint4*>(src + w0 + 4 * q4));
            r[4 * q4] = v.x; r[4 * q4 + 1] = v.y; r[4 * q4 + 2] = v.z; r[4 * q4 + 3] = v.w;
          }
          tmem_st16(tmem + lane_off + w0, r);
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(tw_full);
      }
      const int b = w.b;
      __syncwarp();  // every lane is done with the staging buffer about to be refilled
      if (i + 1 < cnt) {
        ahead.next(C);
        if (!(kDbg & 64)) prefetch(ahead, buf ^ 1);
      }
      cp_async_commit();
      if (warp == 4 || warp == 8) TS_TRACE(warp == 4 ? 4 : 11, i);
      if (!(kDbg & 4096)) mbar_wait(&acc_full[w.ab], w.aph);
      if (warp == 4 || warp == 8) TS_TRACE(warp == 4 ? 5 : 12, i);
      if (!(kDbg & 16384)) tc_fence_after();
      // all 7 x 8 accumulators are read back-to-back and this warp's share of
      // the TMEM buffer is released before any math
      const uint32_t abase = tmem + lane_off + (w.ab ? kAccCol1 : kAccCol0) + cb;
      uint32_t acc[7][kCW];
      if (!(kDbg & 8)) {
#pragma unroll
        for (int s = 0; s < 7; ++s) tmem_ld8(abase + 16 * s, acc[s]);
        tmem_ld_wait();
        if (warp == 4) TS_TRACE(6, i);
      } else {
#pragma unroll
        for (int s = 0; s < 7; ++s)
#pragma unroll
          for (int e = 0; e < kCW; ++e) acc[s][e] = s + e;
      }
      if (!(kDbg & 16384)) tc_fence_before();
      if (!(kDbg & 32768)) mbar_arrive(&acc_empty[w.ab]);
      if (kDbg & 8192) continue;
      uint32_t y[kCW];
#pragma unroll
      for (int e = 0; e < kCW; ++e) {
        // y = (sum_s C_s 2^(8s)) * 2^-64 mod q (the twiddles carry the 2^64 back)
        // stage 1 (Hadamard) and the key-switch MAC multiply y by a factor < q
        // in Montgomery form next, so they take it uncorrected
        y[e] = fold_redc<STAGE == 1 || MODE == EPI_KS_MAC>(acc[0][e], acc[1][e], acc[2][e],
                                                           acc[3][e], acc[4][e], acc[5][e],
                                                           acc[6][e], pc);
      }
      if (warp == 4) TS_TRACE(15, i);
      if (kDbg & 2) {
        if (y[0] == 0x7fffffff && y[kCW - 1] == 1) a.out[0] = 0;  // keep the work live
        continue;
      }
      cp_async_wait1();   // this chunk's operand tiles have landed (own copies)
      __syncwarp();       // ... and every lane's copies are visible
      if (STAGE == 1) {
        const uint8_t* wt = wstg + buf * kInBuf;
#pragma unroll
        for (int e = 0; e < kCW; ++e)
          y[e] = mont_reduce_lazy((uint64_t)y[e] * *reinterpret_cast<const uint32_t*>(wt + e * 128 + lane * 4), pc);
        // blocked P layout [limb][b][i2/16][k1][16]: the warp's rows are 64 B apart
        uint32_t* dst = a.out + (((size_t)limb * a.batch + b) * (a.n2 / kNC) + w.x0 / kNC) * kNC * a.n1 +
                        (size_t)(h * 128 + wq * 32) * kNC + cb;
        store_tile(0, y, dst, kNC);
        if (warp == 4 || warp == 8) TS_TRACE(warp == 4 ? 13 : 14, i);
        continue;
      }
      const size_t wrow = (size_t)(h * 128 + wq * 32) * a.n1 + w.x0 + cb;
      if (mode == EPI_KS_ACC) {
        // y is in Montgomery form (twiddles carry 2^96); the S slices of this
        // (target, chunk) group accumulate in registers, acc touches HBM once.
        // Products y R * k (< q^2) are summed lazily in 64 bits -- one
        // IMAD.WIDE each -- and reduced (Barrett, then one Montgomery step to
        // drop R) every ks_lazy slices and at the group end.
        if (w.sl == 0) {
          if (a.epi.init_acc[limb]) {
            read_row(buf, 2, regb);
            read_row(buf, 3, rega);
          } else {
#pragma unroll
            for (int e = 0; e < kCW; ++e) regb[e] = rega[e] = 0;
          }
#pragma unroll
          for (int e = 0; e < kCW; ++e) lzb[e] = lza[e] = 0;
          npend = 0;
        }
        if (a.epi.j0 + w.sl != a.epi.js[limb]) {
          uint32_t kb[kCW], ka[kCW];
          read_row(buf, 0, kb);
          read_row(buf, 1, ka);
#pragma unroll
          for (int e = 0; e < kCW; ++e) {
            lzb[e] += (uint64_t)y[e] * kb[e];
            lza[e] += (uint64_t)y[e] * ka[e];
          }
          ++npend;
        }
        if (npend && (npend == a.epi.ks_lazy || w.sl == w.S - 1)) {
#pragma unroll
          for (int e = 0; e < kCW; ++e) {
            regb[e] = add_mod(regb[e], mont_reduce(reduce64(lzb[e], pc.q, pc.mu), pc), pc.q);
            rega[e] = add_mod(rega[e], mont_reduce(reduce64(lza[e], pc.q, pc.mu), pc), pc.q);
            lzb[e] = lza[e] = 0;
          }
          npend = 0;
        }
        if (w.sl == w.S - 1) {
          const size_t ar = ((size_t)a.map.out_row[limb] * a.batch + b) * a.n + wrow;
          store_tile(0, regb, a.epi.acc_b + ar, a.n1);
          store_tile(1, rega, a.epi.acc_a + ar, a.n1);
        }
        continue;
      }
      if (mode == EPI_KS_MAC) {
        // y is in Montgomery form (y R: twiddles carry 2^96), so one Montgomery
        // product per key gives y * k exactly
        uint32_t kb[kCW], ka[kCW], ob[kCW], oa[kCW];
        read_row(buf, 0, kb);
        read_row(buf, 1, ka);
        if (!a.epi.first) {
          read_row(buf, 2, ob);
          read_row(buf, 3, oa);
        }
#pragma unroll
        for (int e = 0; e < kCW; ++e) {
          const uint32_t tb = mont_reduce((uint64_t)y[e] * kb[e], pc);
          const uint32_t ta = mont_reduce((uint64_t)y[e] * ka[e], pc);
          ob[e] = a.epi.first ? tb : add_mod(ob[e], tb, pc.q);
          oa[e] = a.epi.first ? ta : add_mod(oa[e], ta, pc.q);
        }
        const size_t ar = ((size_t)a.map.out_row[limb] * a.batch + b) * a.n + wrow;
        store_tile(0, ob, a.epi.acc_b + ar, a.n1);
        store_tile(1, oa, a.epi.acc_a + ar, a.n1);
        continue;
      }
      if (mode == EPI_SUB_SCALE) {
        uint32_t xrow[kCW], brow[kCW];
        read_row(buf, 0, xrow);
        const bool has_base = a.epi.base_row[limb] >= 0;
        if (has_base) read_row(buf, 1, brow);
        const uint32_t s = a.epi.s[limb], sp = a.epi.s_shoup[limb];
#pragma unroll
        for (int e = 0; e < kCW; ++e) {
          uint32_t t = mul_shoup(sub_mod(xrow[e], y[e], pc.q), s, sp, pc.q);
          y[e] = has_base ? add_mod(brow[e], t, pc.q) : t;
        }
      }
      store_tile(0, y, a.out + ((size_t)a.map.out_row[limb] * a.batch + b) * a.n + wrow, a.n1);
      if (warp == 4) TS_TRACE(13, i);
    }
    cp_async_wait0();
  } else {
    reg_dealloc<kRegsMma>();
    if (warp >= kMmaWarp + kMmaIssuers) goto role_done;
    const int mw = warp - kMmaWarp;   // this issuer owns the chunks i = mw (mod kMmaIssuers)
    // ---------------------------------------------------------------- MMA issuer
    // The whole warp walks the loop (so descriptors stay warp-uniform and live
    // in uniform registers); one elected lane issues the tcgen05 ops.
    // stage 1 streams B' MN-major (b_major bit 16), stage 2 K-major
    constexpr uint32_t bmaj = STAGE == 1 ? (1u << 16) : 0u;
    constexpr uint32_t id64 = idesc_i8(128, 64) | bmaj, id48 = idesc_i8(128, 48) | bmaj,
                       id16 = idesc_i8(128, 16) | bmaj;
    constexpr uint32_t kLbo = STAGE == 1 ? 128 : 1024, kSbo = STAGE == 1 ? 512 : 128;
    constexpr uint32_t kPlane3 = STAGE == 1 ? 3 * 512 : 6 * 128;  // start of B' plane 3
    // The epilogue may only overwrite the twiddle (limb change) once every
    // MMA of the previous limb has completed: tw_full is waited per limb.
    const bool handshake = !(kDbg & 4);
    auto issue = [&](const UnitIter& it, int kc0, int kc1) {
      const uint32_t d = tmem + (it.ab ? kAccCol1 : kAccCol0);
      const uint32_t sb = smem_u32(smem + it.s * kStageBytes);
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
        if (kc < kc0 || kc >= kc1) continue;
        const uint32_t bt = sb + kc * 2048;
        const uint64_t bd = smem_desc_kmajor(bt, kLbo, kSbo);
        const uint32_t a0 = tmem + 0 * (K / 4) + kc * 8, a1 = tmem + 1 * (K / 4) + kc * 8;
        const uint32_t a2 = tmem + 2 * (K / 4) + kc * 8, a3 = tmem + 3 * (K / 4) + kc * 8;
        if (kc == 0) {
          mma_i8_ts(d + 48, a3, bd, id64, 0);   // blocks 3..6 = T_3 X_0..3 (init)
          mma_i8_ts(d + 0, a0, bd, id48, 0);    // blocks 0..2 = T_0 X_0..2 (init)
          mma_i8_ts(d + 48, a0, smem_desc_kmajor(bt + kPlane3, kLbo, kSbo), id16, 1);  // + T_0 X_3
          mma_i8_ts(d + 16, a1, bd, id64, 1);
          mma_i8_ts(d + 32, a2, bd, id64, 1);
        } else {
          mma_i8_ts(d + 0, a0, bd, id64, 1);
          mma_i8_ts(d + 16, a1, bd, id64, 1);
          mma_i8_ts(d + 32, a2, bd, id64, 1);
          mma_i8_ts(d + 48, a3, bd, id64, 1);
        }
      }
    };
    // data / accumulator readiness of chunk `it` (index i)
    auto wait_ready = [&](const UnitIter& it, int i) {
      if (!handshake) return;
      if (!(kDbg & 256)) mbar_wait(&b_full[it.s], it.rph);
      if (i >= 2 && !(kDbg & 128)) mbar_wait(&acc_empty[it.ab], it.aph ^ 1);
    };
    int prev = -1;
    uint32_t twph = 0;
    for (int i = 0; i < cnt; ++i, w.next(C)) {
      if (w.limb != prev) {
        if (handshake) {
          if (prev >= 0) twph ^= 1;
          if (!(kDbg & 1024)) mbar_wait(tw_full, twph);
        }
        prev = w.limb;
      }
      if (kMmaIssuers > 1 && (i % kMmaIssuers) != mw) continue;
      TS_TRACE(0, i);
      wait_ready(w, i);
      TS_TRACE(1, i);
      tc_fence_after();
      if (elect_one()) {
        issue(w, 0, KC);
        mma_commit(&b_empty[w.s]);
        mma_commit(&acc_full[w.ab]);
      }
      TS_TRACE(2, i);
      __syncwarp();
    }
  }

role_done:
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int STAGE, int K, int MODE>
int launch_ts(const Ctx& c, TsArgs& a, cudaStream_t st) {
  constexpr int kRaw = raw_slots<STAGE, K, MODE>();
  const int smem = kRing * ring_stage_bytes<K>() + kEpiWarps * warp_stg_bytes<STAGE, MODE>() +
                   kRaw * K * 64 + (2 * kRing + 5 + 2 * kRaw) * 8 + 16;
  auto kern = ntt_ts_kernel<STAGE, K, MODE>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const long long U = (long long)a.n_limbs * a.C;
  int grid;
  if (a.H == 2) grid = 2 * (int)std::min<long long>(c.sms / 2, U);
  else grid = (int)std::min<long long>(c.sms, U);
  if (grid <= 0) return 0;
#ifdef TFHE_TS_TRACE
  static unsigned long long* tbuf = nullptr;
  if (!tbuf) cudaMalloc(&tbuf, 16 * kTraceN * 8);
  cudaMemset(tbuf, 0, 16 * kTraceN * 8);
  a.trace = tbuf;
#endif
  kern<<<grid, kThreadsTS, smem, st>>>(a);
#ifdef TFHE_TS_TRACE
  {
    std::vector<unsigned long long> h(16 * kTraceN);
    cudaMemcpy(h.data(), tbuf, h.size() * 8, cudaMemcpyDeviceToHost);
    static int seq = 0;
    char fn[256];
    snprintf(fn, sizeof(fn), "gpurun_out/trace_s%d_%d.bin", STAGE, seq++);
    if (FILE* f = fopen(fn, "wb")) {
      fwrite(h.data(), 8, h.size(), f);
      fclose(f);
    }
  }
#endif
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("ntt ts launch: ") + cudaGetErrorString(e));
    return 3;
  }
  return 0;
}

template <int STAGE>
int launch_ts_k(const Ctx& c, int K, TsArgs& a, cudaStream_t st) {
  const int mode = STAGE == 2 ? a.epi.mode : EPI_STORE;
#define TFHE_TS_CASE(KK, MM) \
  if (K == KK && mode == MM) return launch_ts<STAGE, KK, (STAGE == 2 ? MM : EPI_STORE)>(c, a, st);
  TFHE_TS_CASE(256, EPI_STORE)
  TFHE_TS_CASE(128, EPI_STORE)
  if (STAGE == 2) {
    TFHE_TS_CASE(256, EPI_SUB_SCALE)
    TFHE_TS_CASE(128, EPI_SUB_SCALE)
    TFHE_TS_CASE(256, EPI_KS_MAC)
    TFHE_TS_CASE(128, EPI_KS_MAC)
    TFHE_TS_CASE(256, EPI_KS_ACC)
    TFHE_TS_CASE(128, EPI_KS_ACC)
  }
#undef TFHE_TS_CASE
  set_error("ts kernel: unsupported contraction length");
  return 2;
}

uint32_t mulmod_h(uint64_t x, uint64_t y, uint32_t q) { return (uint32_t)(x * y % q); }
uint32_t powmod_h(uint64_t b, uint64_t e, uint32_t q) {
  uint64_t r = 1, x = b % q;
  while (e) {
    if (e & 1) r = r * x % q;
    x = x * x % q;
    e >>= 1;
  }
  return (uint32_t)r;
}


// ---- TMA tensor maps (driver entry point fetched once through the runtime)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// stage-1 input: (rows*B, n1, n2) u32, box {16, K, 1}
int make_tmap_stage1(const Ctx& c, CUtensorMap* m, const uint32_t* in, int rows, int batch) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return 3;
  }
  cuuint64_t dims[3] = {(cuuint64_t)c.n2, (cuuint64_t)c.n1, (cuuint64_t)rows * batch};
  cuuint64_t strides[2] = {(cuuint64_t)c.n2 * 4, (cuuint64_t)c.n * 4};
  cuuint32_t box[3] = {16, (cuuint32_t)c.n1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  if (fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<uint32_t*>(in), dims, strides, box, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    set_error("stage-1 tensor map encode failed");
    return 3;
  }
  return 0;
}

// stage-2 input: blocked P (rows*B, n2/16, n1, 16) u32, box {16, 16, K/16, 1},
// 64-byte swizzle (conflict-free converter reads)
int make_tmap_stage2(const Ctx& c, CUtensorMap* m, const uint32_t* P, int rows, int batch) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return 3;
  }
  cuuint64_t dims[4] = {16, (cuuint64_t)c.n1, (cuuint64_t)c.n2 / 16, (cuuint64_t)rows * batch};
  cuuint64_t strides[3] = {64, (cuuint64_t)c.n1 * 64, (cuuint64_t)c.n * 4};
  cuuint32_t box[4] = {16, 16, (cuuint32_t)c.n2 / 16, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  if (fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, const_cast<uint32_t*>(P), dims, strides, box, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    set_error("stage-2 tensor map encode failed");
    return 3;
  }
  return 0;
}

int max_in_row(const LimbMap& m) {
  int r = 0;
  for (int l = 0; l < m.n; ++l) r = std::max(r, (int)m.in_row[l]);
  return r + 1;
}
}  // namespace

int build_ts_tables(Ctx& c) {
  const int n = c.n, n1 = c.n1, n2 = c.n2, np = c.n_primes;
  const uint64_t two_n = 2ull * n;
  std::vector<uint32_t> pw(two_n);
  // variants 0..3: (inv, stage) = (v>>1, v&1); variant 4: forward stage 2
  // scaled by 2^96 for the fused key-switch MAC epilogue
  for (int var = 0; var < 5; ++var) {
      const int inv = var < 4 ? var >> 1 : 0, s = var < 4 ? var & 1 : 1;
      const bool ks = var == 4;
      if (s == 0 && n1 < 128) continue;   // ts_stage2: stage 1 runs on the resident kernel
      const int ntw = s == 0 ? n1 : n2, K = ntw, H = ntw / 128;
      std::vector<uint32_t> tw((size_t)np * ntw * K);  // K words per row (4 planes x K/4)
      for (int p = 0; p < np; ++p) {
        const uint32_t q = c.primes[p];
        const uint32_t root = inv ? powmod_h(c.psis[p], q - 2, q) : c.psis[p];
        pw[0] = 1;
        for (uint64_t e = 1; e < two_n; ++e) pw[e] = mulmod_h(pw[e - 1], root, q);
        const uint32_t n_inv = powmod_h(n, q - 2, q);
        for (int r = 0; r < ntw; ++r) {
          const int hh = r / 128, m = r % 128;
          uint32_t* row = tw.data() + (((size_t)p * H + hh) * 128 + m) * K;
          for (int kq = 0; kq < K / 4; ++kq) {
            uint32_t words[4] = {0, 0, 0, 0};
            for (int e = 0; e < 4; ++e) {
              const uint64_t k = 4 * kq + e;
              uint64_t ex;
              if (s == 0)  // W1[k1 = r][i1 = k]
                ex = inv ? (uint64_t)n2 * (2ull * r * k) : (uint64_t)n2 * (2ull * r * k + k);
              else  // W3[i2 = k][k2 = r]
                ex = inv ? (uint64_t)n1 * (2ull * k * r + r) : (uint64_t)n1 * (2ull * k * r);
              uint32_t v = pw[ex % two_n];
              if (s == 1 && inv) v = mulmod_h(v, n_inv, q);
              // stage 2 twiddles carry 2^64: the two-round Montgomery fold divides it out
              if (s == 1) v = (uint32_t)(((((uint64_t)v << 32) % q) << 32) % q);
              if (ks) v = (uint32_t)(((uint64_t)v << 32) % q);
              for (int i = 0; i < 4; ++i) words[i] |= ((v >> (8 * i)) & 0xFFu) << (8 * e);
            }
            for (int i = 0; i < 4; ++i) row[i * (K / 4) + kq] = words[i];
          }
        }
      }
      const size_t bytes = tw.size() * 4;
      uint32_t** dst = ks ? &c.d_twa_ks : &c.d_twa[inv][s];
      if (cudaMalloc(dst, bytes) != cudaSuccess ||
          cudaMemcpy(*dst, tw.data(), bytes, cudaMemcpyHostToDevice) != cudaSuccess) {
        set_error("ts twiddle upload failed");
        return 3;
      }
  }
  if (n1 < 128) return 0;   // ts_stage2: the resident stage 1 applies W2 itself
  // W2 * 2^96 mod q in [prime][i2/16][e][k1] layout: stage 1 multiplies its
  // folded result (S 2^-64) by this with another Montgomery step -> S * W2;
  // the layout makes the epilogue's per-row loads warp-coalesced
  for (int inv = 0; inv < 2; ++inv) {
    std::vector<uint32_t> w2((size_t)np * n), w2t((size_t)np * n);
    if (cudaMemcpy(w2.data(), c.d_w2[inv], w2.size() * 4, cudaMemcpyDeviceToHost) != cudaSuccess) {
      set_error("w2 readback failed");
      return 3;
    }
    for (int p = 0; p < np; ++p) {
      const uint32_t q = c.primes[p];
      const uint64_t r1 = ((uint64_t)1 << 32) % q, r3 = r1 * r1 % q * r1 % q;
      for (int k1 = 0; k1 < n1; ++k1)
        for (int i2 = 0; i2 < n2; ++i2) {
          const uint64_t v = (uint64_t)w2[(size_t)p * n + (size_t)k1 * n2 + i2] * r3 % q;
          w2t[(size_t)p * n + ((size_t)(i2 / 16) * 16 + (i2 % 16)) * n1 + k1] = (uint32_t)v;
        }
    }
    const size_t bytes = w2t.size() * 4;
    if (cudaMalloc(&c.d_w2r[inv], bytes) != cudaSuccess ||
        cudaMemcpy(c.d_w2r[inv], w2t.data(), bytes, cudaMemcpyHostToDevice) != cudaSuccess) {
      set_error("w2r upload failed");
      return 3;
    }
  }
  return 0;
}

int launch_ntt_ts_stage1(const Ctx& c, const uint32_t* in, uint32_t* P, const LimbMap& map,
                         int batch, int inverse, cudaStream_t st) {
  TsArgs a;
  memset(&a, 0, sizeof(a));
  a.pc = c.d_pc;
  a.n = c.n;
  a.n1 = c.n1;
  a.n2 = c.n2;
  a.batch = batch;
  a.n_limbs = map.n;
  a.S = 1;
  a.map = map;
  a.epi.mode = EPI_STORE;
  a.in = in;
  a.out = P;
  a.twa = c.d_twa[inverse][0];
  a.w2 = c.d_w2r[inverse];
  a.R = c.n2;
  a.H = c.n1 / 128;
  a.C = batch * c.n2 / kNC;
  int rc = make_tmap_stage1(c, &a.tmap, in, max_in_row(map), batch);
  if (rc) return rc;
  return launch_ts_k<1>(c, c.n1, a, st);
}

int launch_ntt_ts(const Ctx& c, const uint32_t* in, uint32_t* out, const LimbMap& map, int batch,
                  int inverse, const EpiArgs* epi, void* ws, cudaStream_t st) {
  TsArgs a;
  memset(&a, 0, sizeof(a));
  a.pc = c.d_pc;
  a.n = c.n;
  a.n1 = c.n1;
  a.n2 = c.n2;
  a.batch = batch;
  a.n_limbs = map.n;
  a.S = 1;
  static const int dbg = getenv("TFHE_DBG") ? atoi(getenv("TFHE_DBG")) : 0;
  a.dbg = dbg;  // (only read when built with -DTFHE_TS_DBG)
  a.map = map;
  if (epi) a.epi = *epi;
  else a.epi.mode = EPI_STORE;
  uint32_t* P = static_cast<uint32_t*>(ws);
  // stage 1: rows k1 (n1 twiddle rows), data columns (b, i2)
  a.in = in;
  a.out = P;
  a.twa = c.d_twa[inverse][0];
  a.w2 = c.d_w2r[inverse];
  a.w2s = nullptr;
  a.R = c.n2;
  a.H = c.n1 / 128;
  a.C = batch * c.n2 / kNC;
  int rc = make_tmap_stage1(c, &a.tmap, in, max_in_row(map), batch);
  if (rc) return rc;
  rc = launch_ts_k<1>(c, c.n1, a, st);
  if (rc) return rc;
  return launch_ntt_ts_stage2(c, P, out, map, batch, inverse, epi, st);
}

int launch_ntt_ts_stage2(const Ctx& c, const uint32_t* P, uint32_t* out, const LimbMap& map,
                         int batch, int inverse, const EpiArgs* epi, cudaStream_t st) {
  TsArgs a;
  memset(&a, 0, sizeof(a));
  a.pc = c.d_pc;
  a.n = c.n;
  a.n1 = c.n1;
  a.n2 = c.n2;
  a.batch = batch;
  a.n_limbs = map.n;
  a.S = 1;
  static const int dbg = getenv("TFHE_DBG") ? atoi(getenv("TFHE_DBG")) : 0;
  a.dbg = dbg;
  a.map = map;
  if (epi) a.epi = *epi;
  else a.epi.mode = EPI_STORE;
  // stage 2: rows k2 (n2 twiddle rows), data columns (b, k1)
  a.in = P;
  a.out = out;
  int rc = make_tmap_stage2(c, &a.tmap, P, map.n, batch);
  if (rc) return rc;
  a.twa = (epi && epi->mode == EPI_KS_MAC) ? c.d_twa_ks : c.d_twa[inverse][1];
  if (epi && epi->mode == EPI_KS_MAC && inverse) {
    set_error("fused key-switch MAC needs a forward transform");
    return 2;
  }
  a.R = c.n1;
  a.H = c.n2 / 128;
  a.C = batch * c.n1 / kNC;
  return launch_ts_k<2>(c, c.n2, a, st);
}

int launch_ntt_ts_ks_group(const Ctx& c, const uint32_t* in, void* ws, const LimbMap& s1map,
                           const LimbMap& tmap, int S, int batch, const EpiArgs& epi,
                           cudaStream_t st) {
  if (c.use_p3) return launch_ntt_p3_ks_group(c, in, ws, s1map, tmap, S, batch, epi, st);
  if (s1map.n != S * tmap.n) {
    set_error("key-switch group: stage-1 map must hold S * T limbs");
    return 2;
  }
  // stage 1 (forward) over every (slice, target) limb into the workspace
  int rc = launch_ntt_ts_stage1(c, in, static_cast<uint32_t*>(ws), s1map, batch, 0, st);
  if (rc) return rc;
  TsArgs a;
  memset(&a, 0, sizeof(a));
  a.pc = c.d_pc;
  a.n = c.n;
  a.n1 = c.n1;
  a.n2 = c.n2;
  a.batch = batch;
  a.n_limbs = tmap.n;
  a.S = S;
  a.map = tmap;
  a.epi = epi;
  a.epi.mode = EPI_KS_ACC;
  {
    // lazy slice sums: k products of (q-1)^2 must fit in 64 bits
    uint64_t qm = 2;
    for (int l = 0; l < tmap.n; ++l) qm = std::max<uint64_t>(qm, c.primes[tmap.prime[l]]);
    const unsigned __int128 sq = (unsigned __int128)(qm - 1) * (qm - 1);
    const uint64_t k = (uint64_t)(((unsigned __int128)~0ull) / sq);
    a.epi.ks_lazy = (int)std::max<uint64_t>(1, std::min<uint64_t>(k, 1u << 20));
  }
  a.in = static_cast<const uint32_t*>(ws);
  a.out = nullptr;
  a.twa = c.d_twa_ks;
  if ((rc = make_tmap_stage2(c, &a.tmap, a.in, S * tmap.n, batch))) return rc;
  a.R = c.n1;
  a.H = c.n2 / 128;
  a.C = batch * c.n1 / kNC;
  return launch_ts_k<2>(c, c.n2, a, st);
}

}  // namespace tfhe
