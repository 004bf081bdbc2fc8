// Batched negacyclic NTT / INTT on the int8 tensor cores (tcgen05, sm_100a).
//
// TensorFHE's formulation (§IV; reference emulation
// pkg/src/rnsckks/ntt.py:212-222 "gemm", :249-340 "segmented"): with
// n = n1*n2 and A[i1][i2] = a[i1*n2 + i2],
//     S = W1 @ A,   P = S .* W2,   Y = P @ W3,   out[n1*k2 + k1] = Y[k1][k2]
// (inverse: same with the inverse twiddles and a final n^-1, ntt.py:218-222).
//
// Each mod-q matrix product is computed EXACTLY on u8 x u8 -> s32 MMAs.  The
// data operand X is split into byte planes X_j (j = 0..3).  The constant
// twiddle operand T is pre-multiplied, V_j = 2^(8j) T mod q, and V_j is split
// into bytes V_{j,i}.  Then
//     T X = sum_j V_j X_j = sum_i 2^(8i) C_i  (mod q),   C_i = sum_j V_{j,i} X_j
// i.e. 4 s32 accumulators C_i (in TMEM), each a K' = 4K contraction of bytes
// (C_i < 4 K 255^2 < 2^31 for K <= 8192).  This is SURVEY Appendix B's
// 4-accumulator form; the epilogue folds sum_i 2^(8i) C_i, reduces mod q
// (Barrett), applies the Hadamard twiddle (stage 1) or the fused output
// epilogue (stage 2) and stores.  Because every step is exact modular
// arithmetic the result is bit-identical to the reference's butterfly backend.
//
// Roles ("data-as-A"): the MMA M dimension runs over data rows, N over the
// twiddle's output index, K over the contraction:
//   stage 1:  D[(b,i2)][k1] = sum_i1 A_b[i1][i2] * W1[k1][i1]   -> P (workspace)
//   stage 2:  D[(b,k1)][k2] = sum_i2 P_b[k1][i2] * W3[i2][k2]   -> out[k2*n1+k1]
// so both epilogues store coalesced along the TMEM lane (= data row) index.
//
// v1 kernel structure: one 128-row x BN-column output tile per CTA;
// warps 0-3 load + byte-split data into smem and later run the epilogue,
// one thread bulk-copies (TMA engine) the pre-split twiddle tiles, warp 4
// owns TMEM and issues the MMAs; a 2-stage mbarrier ring overlaps loads with
// MMAs.
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "tfhe_internal.h"

namespace tfhe {

namespace {

constexpr int kRows = 128;        // MMA M (data rows per tile)
constexpr int kStages = 2;        // smem pipeline depth
constexpr int kKC = 32;           // K values per pipeline stage (one MMA K-step per plane)
constexpr int kThreads = 160;     // 4 load/epilogue warps + 1 MMA warp
constexpr int kATile = kRows * kKC;  // bytes of one A plane tile (4 KB)

struct StageArgs {
  const uint32_t* in;    // stage 1: (rows, batch, n) input; stage 2: P workspace (L, batch, n)
  uint32_t* out;         // stage 1: P workspace; stage 2: (rows, batch, n) output
  const uint8_t* tw;     // twiddle tiles for this (direction, stage)
  size_t tw_stride;      // bytes per prime
  const uint32_t* w2;    // stage 1: hadamard twiddles (prime, n1*n2)
  const uint32_t* w2s;
  const PrimeConst* pc;
  int n, n1, n2, batch;
  int R;                 // data rows per member (stage 1: n2, stage 2: n1)
  int K, KC;             // contraction length, number of 32-chunks (padded)
  int Ntw;               // twiddle columns
  int total_rows;        // batch * R
  int p_blocked;         // stage 1 (resident kernel): write P in the TS blocked layout
  LimbMap map;
  EpiArgs epi;
};

// fold of the 4 accumulators, v = sum_i 2^(8i) C_i (< 2^49), to the residue.
// Primes > 2^20 (pc.pad[0] = 1) have twiddles pre-scaled by 2^32, so one
// Montgomery step (v < q 2^32) replaces the 64-bit Barrett reduction.  With
// K <= 64 (KC <= 2) every C_i < 4 K 255^2 <= 2^24, so the pairs C_0 + 2^8 C_1
// and C_2 + 2^8 C_3 fit 32 bits; larger K folds in 64 bits throughout.
// kLazy: the Montgomery result is left in [0, 2q) for a consumer that takes
// any 32-bit operand (the stage-1 Shoup Hadamard).
template <int KC, bool kLazy = false>
TFHE_DEV uint32_t fold4(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, const PrimeConst& pc) {
  const uint64_t v =
      KC <= 2 ? (uint64_t)(c0 + (c1 << 8)) + ((uint64_t)(c2 + (c3 << 8)) << 16)
              : (uint64_t)c0 + ((uint64_t)c1 << 8) + ((uint64_t)c2 << 16) + ((uint64_t)c3 << 24);
  if (pc.pad[0]) {
    const uint32_t m = (uint32_t)v * pc.qneg_inv;
    const uint32_t t = (uint32_t)((v + (uint64_t)m * pc.q) >> 32);
    if (kLazy) return t;
    return t >= pc.q ? t - pc.q : t;
  }
  return reduce64(v, pc.q, pc.mu);
}

// key-switch MAC product y k mod q: y arrives in Montgomery form (y 2^32, from
// the 2^64-scaled stage-2 twiddles) for Montgomery primes, else plain (Barrett)
TFHE_DEV uint32_t mac_mul(uint32_t y, uint32_t k, const PrimeConst& pc) {
  if (pc.pad[0]) {
    const uint64_t v = (uint64_t)y * k;
    const uint32_t m = (uint32_t)v * pc.qneg_inv;
    const uint32_t t = (uint32_t)((v + (uint64_t)m * pc.q) >> 32);
    return t >= pc.q ? t - pc.q : t;
  }
  return mul_mod(y, k, pc.q, pc.mu);
}

// Stage-2 epilogue operands of W consecutive output columns col0.. of row
// (b, x): the accumulator (EPI_KS_MAC, not first) or x and base (EPI_SUB_SCALE).
// Every load is issued before any of the row's stores: written inline, each
// column's load would wait on the previous column's store (the pointers may
// alias), one full memory latency per output.
template <int W, bool kGuard = true>
TFHE_DEV void epi2_load(const StageArgs& a, int limb, int b, int x, int col0, bool valid,
                        uint32_t (&p0)[W], uint32_t (&p1)[W]) {
  if (!valid || a.epi.mode == EPI_STORE || (a.epi.mode == EPI_KS_MAC && a.epi.first)) return;
  const uint32_t* s0;
  const uint32_t* s1 = nullptr;
  if (a.epi.mode == EPI_KS_MAC) {
    const size_t orow = ((size_t)a.map.out_row[limb] * a.batch + b) * a.n;
    s0 = a.epi.acc_b + orow;
    s1 = a.epi.acc_a + orow;
  } else {
    s0 = a.epi.x + ((size_t)a.epi.x_row[limb] * a.batch + b) * a.n;
    const int br = a.epi.base_row[limb];
    if (br >= 0) s1 = a.epi.base + ((size_t)br * a.batch + b) * a.n;
  }
#pragma unroll
  for (int e = 0; e < W; ++e) {
    const size_t pos = (size_t)(col0 + e) * a.n1 + x;
    if (!kGuard || col0 + e < a.Ntw) {
      p0[e] = s0[pos];
      if (s1) p1[e] = s1[pos];
    }
  }
}

// stage-2 epilogue of one output y at column col of row (b, x), operands from
// epi2_load; kb / ka are the key rows of EPI_KS_MAC (indexed by position)
TFHE_DEV void epi2_store(const StageArgs& a, int limb, int b, int x, int col, uint32_t y,
                         uint32_t p0, uint32_t p1, const uint32_t* kb, const uint32_t* ka,
                         const PrimeConst& pc) {
  const size_t pos = (size_t)col * a.n1 + x;   // out[n1*k2 + k1], k2 = col, k1 = x
  const size_t orow = ((size_t)a.map.out_row[limb] * a.batch + b) * a.n;
  if (a.epi.mode == EPI_KS_MAC) {
    const uint32_t tb = mac_mul(y, kb[pos], pc);
    const uint32_t ta = mac_mul(y, ka[pos], pc);
    a.epi.acc_b[orow + pos] = a.epi.first ? tb : add_mod(p0, tb, pc.q);
    a.epi.acc_a[orow + pos] = a.epi.first ? ta : add_mod(p1, ta, pc.q);
    return;
  }
  if (a.epi.mode == EPI_SUB_SCALE) {
    y = mul_shoup(sub_mod(p0, y, pc.q), a.epi.s[limb], a.epi.s_shoup[limb], pc.q);
    if (a.epi.base_row[limb] >= 0) y = add_mod(p1, y, pc.q);
  }
  a.out[orow + pos] = y;
}

__host__ __device__ constexpr int tmem_cols_for(int bn) {
  return 4 * bn <= 32 ? 32 : 4 * bn <= 64 ? 64 : 4 * bn <= 128 ? 128 : 4 * bn <= 256 ? 256 : 512;
}

// offset of (row r, k) inside a K-major SWIZZLE_NONE tile of `rows` x 32 bytes
TFHE_DEV uint32_t tile_off(int r, int k, int rows) {
  return (uint32_t)((k >> 4) * (rows * 16) + (r >> 3) * 128 + (r & 7) * 16 + (k & 15));
}

// 4x4 byte transpose: plane j gets byte j of v0..v3 (v0 in the low byte)
TFHE_DEV void byte_planes(uint32_t v0, uint32_t v1, uint32_t v2, uint32_t v3, uint32_t (&w)[4]) {
  uint32_t lo01 = __byte_perm(v0, v1, 0x5140), hi01 = __byte_perm(v0, v1, 0x7362);
  uint32_t lo23 = __byte_perm(v2, v3, 0x5140), hi23 = __byte_perm(v2, v3, 0x7362);
  w[0] = __byte_perm(lo01, lo23, 0x5410);
  w[1] = __byte_perm(lo01, lo23, 0x7632);
  w[2] = __byte_perm(hi01, hi23, 0x5410);
  w[3] = __byte_perm(hi01, hi23, 0x7632);
}

template <int STAGE, int BN>
__global__ void __launch_bounds__(kThreads, 1) ntt_stage_kernel(const __grid_constant__ StageArgs a) {
  constexpr int kBTile = BN * kKC;             // bytes of one twiddle tile
  constexpr int kStageBytes = 4 * kATile + 16 * kBTile;
  constexpr uint32_t kTmemCols = tmem_cols_for(BN);
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int limb = blockIdx.z, ct = blockIdx.y;
  const int r0 = blockIdx.x * kRows;
  const int prime = a.map.prime[limb];
  const PrimeConst pc = a.pc[prime];

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 129);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    fence_mbar_init();
  }
  if (warp == 4) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    // ------------------------------------------------------------ producer
    const int gr = r0 + tid;
    const bool valid = gr < a.total_rows;
    const int b = valid ? gr / a.R : 0;
    const int x = valid ? gr % a.R : 0;
    const uint32_t* src;
    if (STAGE == 1) {
      src = a.in + ((size_t)a.map.in_row[limb] * a.batch + b) * a.n + x;  // X[k][x] = src[k*n2]
    } else {
      src = a.in + ((size_t)limb * a.batch + b) * a.n + (size_t)x * a.n2;  // P[x][k] = src[k]
    }
    const uint8_t* twp = a.tw + (size_t)prime * a.tw_stride + (size_t)ct * a.KC * 16 * kBTile;
    for (int kc = 0; kc < a.KC; ++kc) {
      const int s = kc % kStages;
      if (kc >= kStages) mbar_wait(&empty[s], ((kc / kStages) & 1) ^ 1);
      uint8_t* sA = smem + s * kStageBytes;
      uint8_t* sB = sA + 4 * kATile;
      if (tid == 0) {
        mbar_arrive_expect_tx(&full[s], 16 * kBTile);
        bulk_g2s(sB, twp + (size_t)kc * 16 * kBTile, 16 * kBTile, &full[s]);
      }
#pragma unroll
      for (int kq = 0; kq < kKC / 4; ++kq) {
        const int k = kc * kKC + kq * 4;
        uint32_t v0 = 0, v1 = 0, v2 = 0, v3 = 0;
        if (valid && k < a.K) {
          if (STAGE == 1) {
            const uint32_t* p = src + (size_t)k * a.n2;
            v0 = __ldg(p);
            v1 = __ldg(p + a.n2);
            v2 = __ldg(p + 2 * a.n2);
            v3 = __ldg(p + 3 * a.n2);
          } else {
            uint4 v = __ldg(reinterpret_cast<const uint4*>(src + k));
            v0 = v.x; v1 = v.y; v2 = v.z; v3 = v.w;
          }
        }
        uint32_t w[4];
        byte_planes(v0, v1, v2, v3, w);
        const uint32_t off = tile_off(tid, kq * 4, kRows);
#pragma unroll
        for (int j = 0; j < 4; ++j) *reinterpret_cast<uint32_t*>(sA + j * kATile + off) = w[j];
      }
      fence_proxy_async_smem();
      mbar_arrive(&full[s]);
    }

    // ------------------------------------------------------------ epilogue
    mbar_wait(tfull, 0);
    tc_fence_after();
    const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
      uint32_t acc[4][16];
      uint32_t p0[16], p1[16];
#pragma unroll
      for (int i = 0; i < 4; ++i) tmem_ld16(lane_base + i * BN + c0, acc[i]);
      if (STAGE == 2) epi2_load<16>(a, limb, b, x, ct * BN + c0, valid, p0, p1);
      tmem_ld_wait();
      if (!valid) continue;
      // fold every column first (branch-free, so the 16 folds interleave);
      // columns past Ntw only occur for n1 or n2 < 16 and are dropped at the store
      uint32_t y[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) y[e] = fold4<4>(acc[0][e], acc[1][e], acc[2][e], acc[3][e], pc);
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int col = ct * BN + c0 + e;
        if (col < a.Ntw) {
          if (STAGE == 1) {
            // P[k1=col][i2=x] = S * W2[k1][i2]
            const size_t widx = (size_t)prime * a.n + (size_t)col * a.n2 + x;
            a.out[((size_t)limb * a.batch + b) * a.n + (size_t)col * a.n2 + x] =
                mul_shoup(y[e], __ldg(a.w2 + widx), __ldg(a.w2s + widx), pc.q);
          } else {
            const size_t kr = a.epi.mode == EPI_KS_MAC ? (size_t)a.epi.key_row[limb] * a.n : 0;
            epi2_store(a, limb, b, x, col, y[e], p0[e], p1[e], a.epi.kb + kr, a.epi.ka + kr, pc);
          }
        }
      }
    }
  } else if (lane == 0) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = idesc_i8(kRows, BN);
    for (int kc = 0; kc < a.KC; ++kc) {
      const int s = kc % kStages;
      mbar_wait(&full[s], (kc / kStages) & 1);
      tc_fence_after();
      const uint32_t sA = smem_u32(smem + s * kStageBytes);
      const uint32_t sB = sA + 4 * kATile;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t adesc = smem_desc_kmajor(sA + j * kATile, kRows * 16, 128);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint64_t bdesc = smem_desc_kmajor(sB + (j * 4 + i) * kBTile, BN * 16, 128);
          mma_i8_ss(tmem + i * BN, adesc, bdesc, idesc, (kc | j) != 0);
        }
      }
      mma_commit(&empty[s]);
    }
    mma_commit(tfull);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
}

template <int STAGE, int BN>
int launch_stage(const StageArgs& a, int npad, int n_limbs, cudaStream_t st) {
  constexpr int kStageBytes = 4 * kATile + 16 * BN * kKC;
  const int smem = kStages * kStageBytes + 2 * kStages * 8 + 8 + 16;
  auto kern = ntt_stage_kernel<STAGE, BN>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  dim3 grid((a.total_rows + kRows - 1) / kRows, npad / BN, n_limbs);
  kern<<<grid, kThreads, smem, st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("ntt stage launch: ") + cudaGetErrorString(e));
    return 3;
  }
  return 0;
}

template <int STAGE>
int launch_stage_bn(int bn, const StageArgs& a, int npad, int n_limbs, cudaStream_t st) {
  switch (bn) {
    case 16: return launch_stage<STAGE, 16>(a, npad, n_limbs, st);
    case 32: return launch_stage<STAGE, 32>(a, npad, n_limbs, st);
    case 64: return launch_stage<STAGE, 64>(a, npad, n_limbs, st);
    case 128: return launch_stage<STAGE, 128>(a, npad, n_limbs, st);
  }
  set_error("unsupported tile width");
  return 2;
}

// ---------------------------------------------------------------------------
// Persistent twiddle-resident variant (small n: BN * KC <= 128, e.g. the
// 64 x 64 plan of N = 2^12).  Same math and tile layouts as
// ntt_stage_kernel, but one CTA per SM walks a contiguous range of
// (limb, 128-row tile) units: the byte-split twiddle tiles of the current
// prime (16 * KC tiles, <= 64 KB) are bulk-copied into shared memory once
// per limb instead of once per tile, data tiles stream through a
// kResStages-deep ring, and the TMEM accumulators are double-buffered so the
// epilogue of tile t overlaps the MMAs of tile t+1.
//   warps 0-3  producers (one data row each: load K values, byte-split);
//              thread 0 also reloads the twiddles on a limb change
//   warps 4-11 epilogue (TMEM lane = data row; two warps per lane quarter,
//              each half of the columns, to hide the fold / reduce latency)
//   warp 12    TMEM owner; one elected lane issues the MMAs
// ---------------------------------------------------------------------------
// data (byte-plane) ring depth; stage 2 also stages its contiguous P tiles
// through a kResRaw-deep raw ring by bulk copy (stage 1 loads straight from
// global memory)
template <int STAGE>
__host__ __device__ constexpr int res_stages() { return STAGE == 1 ? 3 : 2; }
constexpr int kResRaw = 2;
constexpr int kResEpiWarps = 8;                     // two per TMEM lane quarter
constexpr int kResMmaWarp = 4 + kResEpiWarps;
constexpr int kResThreads = 32 * (kResMmaWarp + 1);

__host__ __device__ constexpr uint32_t res_tmem_cols(int bn) {
  return 8 * bn <= 32 ? 32 : 8 * bn <= 64 ? 64 : 8 * bn <= 128 ? 128 : 8 * bn <= 256 ? 256 : 512;
}
// per-limb resident operand: stage 1 keeps the prime's Hadamard twiddles W2
// (+ Shoup, n <= 8192); stage 2 with the key-switch MAC epilogue keeps the
// target's two switching-key rows (shared by every batch member, n <= 4096)
constexpr int kResMaxN = 8192;
template <int STAGE>
__host__ __device__ constexpr int res_w2_bytes() { return STAGE == 1 ? 2 * kResMaxN * 4 : 2 * 4096 * 4; }
// stage 2 stages its (contiguous) P tiles through a 2-deep raw ring by bulk copy
template <int STAGE, int KC>
__host__ __device__ constexpr int res_raw_bytes() { return STAGE == 2 ? kResRaw * kRows * KC * kKC * 4 : 0; }
template <int STAGE, int BN, int KC>
__host__ __device__ constexpr int res_smem_bytes() {
  return KC * 16 * BN * kKC + res_w2_bytes<STAGE>() + res_raw_bytes<STAGE, KC>() +
         res_stages<STAGE>() * KC * 4 * kATile + (2 * res_stages<STAGE>() + 2 * kResRaw + 7) * 8 + 16;
}

// Timing probes of the resident kernel (-DTFHE_RES_DBG_VAL=k, tools/ab_res_dbg.sh;
// 0 in normal builds, where every test below folds away): 1 epilogue drops
// all math and stores, 2 epilogue does no stores (most folds then dead), 512
// epilogue folds every column but does not store, 4 producers skip the data
// loads (stage 2: no raw P tiles), 8 producers skip loads and byte split.
#ifndef TFHE_RES_DBG_VAL
#define TFHE_RES_DBG_VAL 0
#endif
constexpr int kResDbg = TFHE_RES_DBG_VAL;

template <int STAGE, int BN, int KC>
__global__ void __launch_bounds__(kResThreads, 1)
    ntt_res_kernel(const __grid_constant__ StageArgs a, int tiles_per_limb, long long units) {
  constexpr int kBTile = BN * kKC;
  constexpr int kTwBytes = KC * 16 * kBTile;
  constexpr int kDataBytes = KC * 4 * kATile;
  constexpr int kResStages = res_stages<STAGE>();
  constexpr uint32_t kAccCols = 4 * BN;
  constexpr uint32_t kTmemCols = res_tmem_cols(BN);
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sTw = smem;
  uint32_t* sW2 = reinterpret_cast<uint32_t*>(smem + kTwBytes);   // stage 1: [n] W2 | [n] Shoup
  uint8_t* sRaw = smem + kTwBytes + res_w2_bytes<STAGE>();          // stage 2: [2] P tiles
  constexpr int kRawTile = kRows * KC * kKC * 4;
  uint8_t* sData = sRaw + res_raw_bytes<STAGE, KC>();
  uint64_t* d_full = reinterpret_cast<uint64_t*>(sData + kResStages * kDataBytes);
  uint64_t* d_empty = d_full + kResStages;
  uint64_t* acc_full = d_empty + kResStages;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* tw_full = acc_empty + 2;
  uint64_t* tw_empty = tw_full + 1;
  uint64_t* epi_done = tw_empty + 1;   // epilogue finished a limb (W2 may be replaced)
  uint64_t* raw_full = epi_done + 1;
  uint64_t* raw_empty = raw_full + kResRaw;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(raw_empty + kResRaw);

  const int tid = threadIdx.x, warp = tid >> 5;
  // a per-limb operand (W2, or the key rows of the MAC epilogue) is resident
  const bool limb_operand = STAGE == 1 || a.epi.mode == EPI_KS_MAC;
  const long long u0 = units * blockIdx.x / gridDim.x;
  const int cnt = (int)(units * (blockIdx.x + 1) / gridDim.x - u0);
  if (tid == 0) {
    for (int s = 0; s < kResStages; ++s) {
      mbar_init(&d_full[s], 128);
      mbar_init(&d_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 32 * kResEpiWarps);
    }
    mbar_init(tw_full, 1);
    mbar_init(tw_empty, 1);
    mbar_init(epi_done, 32 * kResEpiWarps);
    for (int sl = 0; sl < kResRaw; ++sl) {
      mbar_init(&raw_full[sl], 1);
      mbar_init(&raw_empty[sl], 128);
    }
    fence_mbar_init();
  }
  if (warp == kResMmaWarp) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    // ---------------------------------------------------------------- producers
    int prev_limb = -1;
    uint32_t tw_ph = 0;
    auto issue_raw = [&](int it, int rs) {   // stage 2: P tile of unit u0 + it
      const long long u = u0 + it;
      const int limb = (int)(u / tiles_per_limb), tile = (int)(u % tiles_per_limb);
      const int rows = min(kRows, a.total_rows - tile * kRows);
      const uint32_t bytes = (uint32_t)rows * a.K * 4;
      mbar_arrive_expect_tx(&raw_full[rs], bytes);
      bulk_g2s(sRaw + rs * kRawTile,
               a.in + (size_t)limb * a.batch * a.n + (size_t)tile * kRows * a.n2, bytes,
               &raw_full[rs]);
    };
    if (STAGE == 2 && tid == 0 && !(kResDbg & 12))
      for (int it = 0; it < kResRaw && it < cnt; ++it) issue_raw(it, it);
    for (int it = 0; it < cnt; ++it) {
      const long long u = u0 + it;
      const int limb = (int)(u / tiles_per_limb), tile = (int)(u % tiles_per_limb);
      if (limb != prev_limb) {
        if (tid == 0) {
          if (prev_limb >= 0) {
            mbar_wait(tw_empty, tw_ph);   // every MMA of the previous limb has completed
            if (limb_operand) mbar_wait(epi_done, tw_ph);   // ... and its epilogue
            tw_ph ^= 1;
          }
          const int pr = a.map.prime[limb];
          mbar_arrive_expect_tx(tw_full, kTwBytes + (limb_operand ? 2 * a.n * 4 : 0));
          bulk_g2s(sTw, a.tw + (size_t)pr * a.tw_stride, kTwBytes, tw_full);
          if (STAGE == 1) {
            bulk_g2s(sW2, a.w2 + (size_t)pr * a.n, a.n * 4, tw_full);
            bulk_g2s(sW2 + a.n, a.w2s + (size_t)pr * a.n, a.n * 4, tw_full);
          } else if (limb_operand) {
            const size_t kr = (size_t)a.epi.key_row[limb] * a.n;
            bulk_g2s(sW2, a.epi.kb + kr, a.n * 4, tw_full);
            bulk_g2s(sW2 + a.n, a.epi.ka + kr, a.n * 4, tw_full);
          }
        }
        prev_limb = limb;
      }
      const int s = it % kResStages;
      const int gr = tile * kRows + tid;
      const bool valid = gr < a.total_rows;
      uint8_t* sA = sData + s * kDataBytes;
      if (kResDbg & 8) {
        if (it >= kResStages) mbar_wait(&d_empty[s], ((it / kResStages) & 1) ^ 1);
      } else if (STAGE == 2) {
        // P rows of a tile are contiguous (row (b, x) at gr * n2 within the limb):
        // one bulk copy per tile, issued kResRaw tiles ahead
        const int rs = it % kResRaw;
        const uint32_t rph = (uint32_t)((it / kResRaw) & 1);
        if (!(kResDbg & 4)) mbar_wait(&raw_full[rs], rph);
        if (it >= kResStages) mbar_wait(&d_empty[s], ((it / kResStages) & 1) ^ 1);
        const uint8_t* row = sRaw + rs * kRawTile + (size_t)tid * a.K * 4;
        const int ng = (a.K + 3) / 4;
#pragma unroll
        for (int g0 = 0; g0 < KC * 8; ++g0) {
          // groups of 4 k in a per-thread rotated order: conflict-free 16-byte reads
          const int g = g0 < ng ? (g0 + tid) % ng : g0;
          uint4 q = make_uint4(0, 0, 0, 0);
          if (valid && g0 < ng && !(kResDbg & 4)) q = *reinterpret_cast<const uint4*>(row + g * 16);
          uint32_t w[4];
          byte_planes(q.x, q.y, q.z, q.w, w);
          const uint32_t off = tile_off(tid, (g % 8) * 4, kRows);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            *reinterpret_cast<uint32_t*>(sA + ((g / 8) * 4 + j) * kATile + off) = w[j];
        }
        if (!(kResDbg & 4)) {
          fence_proxy_async_smem();   // raw reads before the next bulk copy into the slot
          mbar_arrive(&raw_empty[rs]);
        }
        if (tid == 0 && it + kResRaw < cnt && !(kResDbg & 4)) {
          mbar_wait(&raw_empty[rs], rph);
          issue_raw(it + kResRaw, rs);
        }
      } else {
      const int b = valid ? gr / a.R : 0;
      const int x = valid ? gr % a.R : 0;
      const uint32_t* src = a.in + ((size_t)a.map.in_row[limb] * a.batch + b) * a.n + x;
      // every load of the tile is issued before any is consumed (one memory
      // latency per tile instead of one per 4-value group)
      uint32_t v[KC * 8][4];
#pragma unroll
      for (int g = 0; g < KC * 8; ++g) {
        const int k = g * 4;
        if (valid && k < a.K && !(kResDbg & 4)) {
          const uint32_t* p = src + (size_t)k * a.n2;
          v[g][0] = __ldg(p);
          v[g][1] = __ldg(p + a.n2);
          v[g][2] = __ldg(p + 2 * a.n2);
          v[g][3] = __ldg(p + 3 * a.n2);
        } else {
          v[g][0] = v[g][1] = v[g][2] = v[g][3] = 0;
        }
      }
      if (it >= kResStages) mbar_wait(&d_empty[s], ((it / kResStages) & 1) ^ 1);
#pragma unroll
      for (int g = 0; g < KC * 8; ++g) {
        const int kc = g / 8, kq = g % 8;
        uint32_t w[4];
        byte_planes(v[g][0], v[g][1], v[g][2], v[g][3], w);
        const uint32_t off = tile_off(tid, kq * 4, kRows);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          *reinterpret_cast<uint32_t*>(sA + (kc * 4 + j) * kATile + off) = w[j];
      }
      }
      fence_proxy_async_smem();
      mbar_arrive(&d_full[s]);
    }
  } else if (warp < kResMmaWarp) {
    // ---------------------------------------------------------------- epilogue
    // columns per TMEM load (stage 2 holds the prefetched operands beside them)
    constexpr int kCWr = BN / 2 >= 16 && STAGE == 1 ? 16 : 8;
    const int quarter = warp & 3, half = (warp - 4) >> 2;
    const int r = quarter * 32 + (tid & 31);
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    int prev_limb = -1;
    uint32_t tw_ph = 0;
    for (int it = 0; it < cnt; ++it) {
      const long long u = u0 + it;
      const int limb = (int)(u / tiles_per_limb), tile = (int)(u % tiles_per_limb);
      const int ab = it & 1;
      if (limb_operand && limb != prev_limb) {
        mbar_wait(tw_full, tw_ph);   // this limb's W2 / key rows are resident
        tw_ph ^= 1;
        prev_limb = limb;
      }
      mbar_wait(&acc_full[ab], (it >> 1) & 1);
      tc_fence_after();
      const int gr = tile * kRows + r;
      const bool valid = gr < a.total_rows;
      const int b = valid ? gr / a.R : 0;
      const int x = valid ? gr % a.R : 0;
      const int prime = a.map.prime[limb];
      const PrimeConst pc = a.pc[prime];
      // stage 1: this row's P, row-major [k1][i2] or, when the TS stage 2
      // follows (Ctx::ts_stage2), its blocked [i2/16][k1][16]; column stride ps
      const int ps = a.p_blocked ? 16 : a.n2;
      uint32_t* p_row = a.out + ((size_t)limb * a.batch + b) * a.n +
                        (a.p_blocked ? (size_t)(x >> 4) * a.n1 * 16 + (x & 15) : (size_t)x);
#pragma unroll 1
      for (int c0 = half * (BN / 2); c0 < (half + 1) * (BN / 2); c0 += kCWr) {
        uint32_t acc[4][kCWr];
        uint32_t p0[kCWr], p1[kCWr];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if constexpr (kCWr == 16) tmem_ld16(lane_base + ab * kAccCols + i * BN + c0, acc[i]);
          else tmem_ld8(lane_base + ab * kAccCols + i * BN + c0, acc[i]);
        }
        if (STAGE == 2) epi2_load<kCWr, false>(a, limb, b, x, c0, valid, p0, p1);
        tmem_ld_wait();
        if (c0 + kCWr >= (half + 1) * (BN / 2)) {
          tc_fence_before();
          mbar_arrive(&acc_empty[ab]);   // buffer drained: the next tile's MMAs may start
        }
        if (!valid || (kResDbg & 1)) continue;
        // Ntw == BN on this path: no per-column guard, and every per-unit mode
        // branch sits outside the column loops so the kCWr folds interleave
        uint32_t y[kCWr];
#pragma unroll
        for (int e = 0; e < kCWr; ++e)   // stage 1: the Shoup Hadamard takes y uncorrected
          y[e] = fold4<KC, STAGE == 1>(acc[0][e], acc[1][e], acc[2][e], acc[3][e], pc);
        if (kResDbg & 2) {
          if (y[0] == 0x7fffffff && y[kCWr - 1] == 1) a.out[0] = 0;
          continue;
        }
        if (kResDbg & 512) {
          uint32_t z = 0;
#pragma unroll
          for (int e = 0; e < kCWr; ++e) z ^= y[e] * (2 * e + 1);
          if (z == 0x7fffffff) a.out[0] = 0;
          continue;
        }
        if (STAGE == 1) {
          // P[k1 = col][i2 = x] = S * W2[k1][i2]
          const int n2 = a.n2;
          uint32_t* o = p_row + c0 * ps;
          const uint32_t* w = sW2 + c0 * n2 + x;
#pragma unroll
          for (int e = 0; e < kCWr; ++e)
            o[e * ps] = mul_shoup_lazy(y[e], w[e * n2], w[a.n + e * n2], pc.q);   // P in [0, 2q)
          continue;
        }
        // out[n1*k2 + k1], k2 = col, k1 = x
        const int n1 = a.n1;
        const size_t orow = ((size_t)a.map.out_row[limb] * a.batch + b) * a.n + (size_t)c0 * n1 + x;
        if (a.epi.mode == EPI_KS_MAC) {
          const uint32_t* kb = sW2 + c0 * n1 + x;
          uint32_t* ob = a.epi.acc_b + orow;
          uint32_t* oa = a.epi.acc_a + orow;
          uint32_t tb[kCWr], ta[kCWr];
#pragma unroll
          for (int e = 0; e < kCWr; ++e) {
            tb[e] = mac_mul(y[e], kb[e * n1], pc);
            ta[e] = mac_mul(y[e], kb[a.n + e * n1], pc);
          }
          if (a.epi.first) {
#pragma unroll
            for (int e = 0; e < kCWr; ++e) { ob[e * n1] = tb[e]; oa[e * n1] = ta[e]; }
          } else {
#pragma unroll
            for (int e = 0; e < kCWr; ++e) {
              ob[e * n1] = add_mod(p0[e], tb[e], pc.q);
              oa[e * n1] = add_mod(p1[e], ta[e], pc.q);
            }
          }
          continue;
        }
        uint32_t* o = a.out + orow;
        if (a.epi.mode == EPI_SUB_SCALE) {
          const uint32_t s = a.epi.s[limb], ss = a.epi.s_shoup[limb];
#pragma unroll
          for (int e = 0; e < kCWr; ++e) y[e] = mul_shoup(sub_mod(p0[e], y[e], pc.q), s, ss, pc.q);
          if (a.epi.base_row[limb] >= 0) {
#pragma unroll
            for (int e = 0; e < kCWr; ++e) y[e] = add_mod(p1[e], y[e], pc.q);
          }
        }
#pragma unroll
        for (int e = 0; e < kCWr; ++e) o[e * n1] = y[e];
      }
      if (limb_operand && (it + 1 == cnt || (u + 1) / tiles_per_limb != limb))
        mbar_arrive(epi_done);   // done reading this limb's W2 / key rows
    }
  } else {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = idesc_i8(kRows, BN);
    const bool leader = elect_one();
    int prev_limb = -1;
    uint32_t tw_ph = 0;
    for (int it = 0; it < cnt; ++it) {
      const long long u = u0 + it;
      const int limb = (int)(u / tiles_per_limb);
      if (limb != prev_limb) {
        mbar_wait(tw_full, tw_ph);
        tw_ph ^= 1;
        prev_limb = limb;
      }
      const int s = it % kResStages, ab = it & 1;
      mbar_wait(&d_full[s], (it / kResStages) & 1);
      if (it >= 2) mbar_wait(&acc_empty[ab], ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      if (leader) {
        const uint32_t sA = smem_u32(sData + s * kDataBytes);
        const uint32_t sB = smem_u32(sTw);
#pragma unroll
        for (int kc = 0; kc < KC; ++kc)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint64_t adesc = smem_desc_kmajor(sA + (kc * 4 + j) * kATile, kRows * 16, 128);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint64_t bdesc =
                  smem_desc_kmajor(sB + ((kc * 4 + j) * 4 + i) * kBTile, BN * 16, 128);
              mma_i8_ss(tmem + ab * kAccCols + i * BN, adesc, bdesc, idesc, (kc | j) != 0);
            }
          }
        mma_commit(&d_empty[s]);
        mma_commit(&acc_full[ab]);
        const bool last_of_limb = it + 1 == cnt || (u + 1) / tiles_per_limb != limb;
        if (last_of_limb) mma_commit(tw_empty);
      }
      __syncwarp();
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kResMmaWarp) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
}

template <int STAGE, int BN, int KC>
int launch_res(const Ctx& c, const StageArgs& a, int n_limbs, cudaStream_t st) {
  constexpr int smem = res_smem_bytes<STAGE, BN, KC>();
  auto kern = ntt_res_kernel<STAGE, BN, KC>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int tiles = (a.total_rows + kRows - 1) / kRows;
  const long long units = (long long)tiles * n_limbs;
  const int grid = (int)std::min<long long>(c.sms, units);
  kern<<<grid, kResThreads, smem, st>>>(a, tiles, units);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("ntt resident-stage launch: ") + cudaGetErrorString(e));
    return 3;
  }
  return 0;
}

// the resident variant runs when the prime's twiddle tiles fit (BN * KC <= 128;
// n <= 8192 for stage 1, whose W2 is resident too, n <= 4096 for stage 2) and
// the tile is exactly the twiddle width (its epilogue has no column guard), else v1
template <int STAGE>
int launch_stage_any(const Ctx& c, int bn, int kc, const StageArgs& a, int npad, int n_limbs,
                     cudaStream_t st) {
  if (a.Ntw == bn && npad == bn && c.n <= (STAGE == 1 ? kResMaxN : 4096)) {
    switch (bn * 8 + kc) {
      case 16 * 8 + 1: return launch_res<STAGE, 16, 1>(c, a, n_limbs, st);
      case 32 * 8 + 1: return launch_res<STAGE, 32, 1>(c, a, n_limbs, st);
      case 32 * 8 + 2: return launch_res<STAGE, 32, 2>(c, a, n_limbs, st);
      case 64 * 8 + 1: return launch_res<STAGE, 64, 1>(c, a, n_limbs, st);
      case 64 * 8 + 2: return launch_res<STAGE, 64, 2>(c, a, n_limbs, st);
    }
  }
  if (a.p_blocked) {
    set_error("blocked P output needs the resident stage-1 kernel");
    return 2;
  }
  return launch_stage_bn<STAGE>(bn, a, npad, n_limbs, st);
}

// --------------------------------------------------------------- host tables

uint32_t mulmod_h(uint64_t a, uint64_t b, uint32_t q) { return (uint32_t)(a * b % q); }
uint32_t powmod_h(uint64_t b, uint64_t e, uint32_t q) {
  uint64_t r = 1, x = b % q;
  while (e) {
    if (e & 1) r = r * x % q;
    x = x * x % q;
    e >>= 1;
  }
  return (uint32_t)r;
}
uint32_t shoup_h(uint32_t w, uint32_t q) { return (uint32_t)(((uint64_t)w << 32) / q); }

int round_up(int x, int m) { return (x + m - 1) / m * m; }

}  // namespace

size_t ntt_workspace_bytes(const Ctx& c, int n_limbs, int batch) {
  return (size_t)n_limbs * batch * c.n * sizeof(uint32_t);
}

int build_ntt_tables(Ctx& c) {
  const int n = c.n, n1 = c.n1, n2 = c.n2, np = c.n_primes;
  const uint64_t two_n = 2ull * n;
  // geometry per stage: stage 0 contracts over n1 (twiddle cols n1), stage 1 over n2
  for (int s = 0; s < 2; ++s) {
    const int ntw = s == 0 ? n1 : n2;
    // tiles of at most 64 twiddle columns: two v1 CTAs (96 KB smem each) share an
    // SM, so one CTA's epilogue overlaps the other's loads
    c.bn[s] = ntw >= 64 ? 64 : ntw >= 32 ? 32 : 16;
    c.npad[s] = round_up(ntw, c.bn[s]);
    c.kpad[s] = round_up(ntw, kKC);
    c.tw_stride[s] = (size_t)c.npad[s] * c.kpad[s] * 16;
  }
  c.h_pc.resize(np);
  std::vector<uint8_t> tw;
  std::vector<uint32_t> w2((size_t)np * n), w2s((size_t)np * n);
  std::vector<uint32_t> pw(two_n), T;
  // variants 0..3: (inv, stage) = (v >> 1, v & 1); variant 4: forward stage 2
  // with one more 2^32 for the key-switch MAC epilogue (Montgomery primes): the
  // stage-2 result is then y 2^32, and one Montgomery product per key gives y k
  for (int var = 0; var < 5; ++var) {
    {
      const int inv = var < 4 ? var >> 1 : 0, s = var < 4 ? var & 1 : 1;
      const bool ks = var == 4;
      const int ntw = s == 0 ? n1 : n2, K = ntw, BN = c.bn[s], KC = c.kpad[s] / kKC;
      tw.assign(c.tw_stride[s] * np, 0);
      T.resize((size_t)ntw * K);
      for (int p = 0; p < np; ++p) {
        const uint32_t q = c.primes[p];
        const bool mont = q > (1u << 20);   // Montgomery fold (fold4) for this prime
        const uint32_t r32 = powmod_h(2, 32, q);
        const uint32_t tw_scale = mont ? (ks ? mulmod_h(r32, r32, q) : r32) : 1u;
        uint32_t root = inv ? powmod_h(c.psis[p], q - 2, q) : c.psis[p];
        pw[0] = 1;
        for (uint64_t e = 1; e < two_n; ++e) pw[e] = mulmod_h(pw[e - 1], root, q);
        const uint32_t n_inv = powmod_h(n, q - 2, q);
        if (var == 0) {
          PrimeConst& k = c.h_pc[p];
          k.q = q;
          k.n_inv = n_inv;
          k.n_inv_shoup = shoup_h(n_inv, q);
          k.mu = (uint64_t)(~0ull / q);  // floor((2^64-1)/q) == floor(2^64/q) for non-power-of-2 q
          k.r[0] = powmod_h(2, 32, q);
          k.r[1] = powmod_h(2, 40, q);
          k.r[2] = powmod_h(2, 48, q);
          k.w3 = powmod_h(2, 24, q);
          uint32_t inv = 1;  // Newton iteration for q^-1 mod 2^32
          for (int t = 0; t < 5; ++t) inv *= 2u - q * inv;
          k.qneg_inv = 0u - inv;
          k.pad[0] = mont ? 1u : 0u;   // fold4: twiddles carry 2^32
          k.pad[1] = 0;
        }
        // T[c][k]: value multiplying data index k for output column c
        for (int cc = 0; cc < ntw; ++cc)
          for (int k = 0; k < K; ++k) {
            uint64_t e;
            if (s == 0)  // W1[k1=cc][i1=k]
              e = inv ? (uint64_t)n2 * (2ull * cc * k) : (uint64_t)n2 * (2ull * cc * k + k);
            else  // W3[i2=k][k2=cc]
              e = inv ? (uint64_t)n1 * (2ull * k * cc + cc) : (uint64_t)n1 * (2ull * k * cc);
            uint32_t v = pw[e % two_n];
            if (s == 1 && inv) v = mulmod_h(v, n_inv, q);
            T[(size_t)cc * K + k] = v;
          }
        uint8_t* base = tw.data() + (size_t)p * c.tw_stride[s];
        for (int cc = 0; cc < ntw; ++cc) {
          const int ct = cc / BN, cr = cc % BN;
          for (int k = 0; k < K; ++k) {
            const int kc = k / kKC, kr = k % kKC;
            uint32_t t = T[(size_t)cc * K + k];
            for (int j = 0; j < 4; ++j) {
              // V_j = 2^(8j) T (x 2^32 for the Montgomery fold) mod q
              uint32_t vj = mulmod_h(mulmod_h(t, tw_scale, q), 1ull << (8 * j), q);
              for (int i = 0; i < 4; ++i) {
                size_t tile = ((size_t)(ct * KC + kc) * 4 + j) * 4 + i;
                size_t off = tile * (BN * kKC) + (kr >> 4) * (BN * 16) + (cr >> 3) * 128 +
                             (cr & 7) * 16 + (kr & 15);
                base[off] = (uint8_t)(vj >> (8 * i));
              }
            }
          }
        }
        if (s == 0 && !ks) {
          for (int k1 = 0; k1 < n1; ++k1)
            for (int i2 = 0; i2 < n2; ++i2) {
              uint64_t e = inv ? (2ull * k1 * i2 + k1) : (2ull * k1 * i2 + i2);
              uint32_t v = pw[e % two_n];
              w2[(size_t)p * n + (size_t)k1 * n2 + i2] = v;
              w2s[(size_t)p * n + (size_t)k1 * n2 + i2] = shoup_h(v, q);
            }
        }
      }
      uint8_t** dst = ks ? &c.d_tw_ks : &c.d_tw[inv][s];
      if (cudaMalloc(dst, tw.size()) != cudaSuccess ||
          cudaMemcpy(*dst, tw.data(), tw.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
        set_error("twiddle upload failed");
        return 3;
      }
      if (s == 0 && !ks) {
        size_t bytes = w2.size() * 4;
        if (cudaMalloc(&c.d_w2[inv], bytes) != cudaSuccess ||
            cudaMalloc(&c.d_w2s[inv], bytes) != cudaSuccess ||
            cudaMemcpy(c.d_w2[inv], w2.data(), bytes, cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(c.d_w2s[inv], w2s.data(), bytes, cudaMemcpyHostToDevice) != cudaSuccess) {
          set_error("hadamard twiddle upload failed");
          return 3;
        }
      }
    }
  }
  if (cudaMalloc(&c.d_pc, sizeof(PrimeConst) * np) != cudaSuccess ||
      cudaMemcpy(c.d_pc, c.h_pc.data(), sizeof(PrimeConst) * np, cudaMemcpyHostToDevice) !=
          cudaSuccess) {
    set_error("prime constant upload failed");
    return 3;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev);
  if (c.sms <= 0) c.sms = 148;
  // twiddle-resident tensor-core path for n1, n2 in {128, 256}
  // (its single-correction Montgomery epilogue needs q > 2^20; see ntt_ts.cu)
  const bool big_q = *std::min_element(c.primes.begin(), c.primes.end()) > (1u << 20);
  c.use_ts = c.n1 >= 128 && c.n2 <= 256 && big_q;
  c.ts_stage2 = c.n1 == 64 && c.n2 == 128 && big_q;
  if (c.use_ts || c.ts_stage2) {
    int rc = build_ts_tables(c);
    if (rc) return rc;
    if (c.n == 1 << 16 && big_q && !getenv("TFHE_NO_P3")) {
      if ((rc = build_p3_tables(c))) return rc;
      c.use_p3 = c.d_p3t1[0] != nullptr;
    }
    return 0;
  }
  return build_fused_tables(c);
}

int launch_ntt(const Ctx& c, const uint32_t* in, uint32_t* out, const LimbMap& map, int batch,
               int inverse, const EpiArgs* epi, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (map.n <= 0 || batch <= 0) return 0;
  if (ws_bytes < ntt_workspace_bytes(c, map.n, batch)) {
    set_error("ntt workspace too small");
    return 2;
  }
  if (epi && epi->scatter_t && !(c.use_p3 && inverse && epi->mode == EPI_STORE)) {
    set_error("output automorphism needs the N = 2^16 inverse transform");
    return 2;
  }
  if (c.use_p3 && !(epi && epi->mode == EPI_KS_ACC))
    return launch_ntt_p3(c, in, out, map, batch, inverse, epi, ws, st);
  if (c.use_ts) return launch_ntt_ts(c, in, out, map, batch, inverse, epi, ws, st);
  {
    const int rc = launch_ntt_fused(c, in, out, map, batch, inverse, epi, st);
    if (rc >= 0) return rc;
  }
  StageArgs a;
  memset(&a, 0, sizeof(a));
  a.pc = c.d_pc;
  a.n = c.n;
  a.n1 = c.n1;
  a.n2 = c.n2;
  a.batch = batch;
  a.map = map;
  if (epi) a.epi = *epi;
  else a.epi.mode = EPI_STORE;
  uint32_t* P = static_cast<uint32_t*>(ws);
  // stage 1: columns of W1 (k1), contraction over i1, rows (b, i2)
  a.in = in;
  a.out = P;
  a.tw = c.d_tw[inverse][0];
  a.tw_stride = c.tw_stride[0];
  a.w2 = c.d_w2[inverse];
  a.w2s = c.d_w2s[inverse];
  a.R = c.n2;
  a.K = c.n1;
  a.KC = c.kpad[0] / kKC;
  a.Ntw = c.n1;
  a.total_rows = batch * c.n2;
  a.p_blocked = c.ts_stage2 ? 1 : 0;
  int rc = launch_stage_any<1>(c, c.bn[0], a.KC, a, c.npad[0], map.n, st);
  if (rc) return rc;
  if (c.ts_stage2) return launch_ntt_ts_stage2(c, P, out, map, batch, inverse, epi, st);
  // stage 2: columns of W3 (k2), contraction over i2, rows (b, k1)
  a.in = P;
  a.out = out;
  // the key-switch MAC takes y 2^32 (Montgomery form) from the 2^64 table
  if (a.epi.mode == EPI_KS_MAC && inverse) {
    set_error("fused key-switch MAC needs a forward transform");
    return 2;
  }
  a.tw = a.epi.mode == EPI_KS_MAC ? c.d_tw_ks : c.d_tw[inverse][1];
  a.tw_stride = c.tw_stride[1];
  a.R = c.n1;
  a.K = c.n2;
  a.KC = c.kpad[1] / kKC;
  a.Ntw = c.n2;
  a.total_rows = batch * c.n1;
  return launch_stage_any<2>(c, c.bn[1], a.KC, a, c.npad[1], map.n, st);
}

}  // namespace tfhe
