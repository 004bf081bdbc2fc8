// Fast base conversion on the int8 tensor cores (tcgen05, sm_100a).
//
// fast_basis_conv (ref rns.py:118-152), for every coefficient x of the batch
// and every target prime p_t:
//     y_s[x]   = a_s[x] * [(Q/q_s)^-1]_{q_s} mod q_s          (s < alpha sources)
//     out_t[x] = sum_s y_s[x] * F[s][t] mod p_t,   F[s][t] = (Q/q_s) mod p_t
// (targets whose prime is a source prime copy that source row through).
//
// As a GEMM: M = coefficients (128-row tiles), N = targets, K = sources.  The
// contraction is made exact on u8 x u8 -> s32 MMAs with the 4-accumulator
// split: the data operand is the y values themselves, read as
// bytes -- A[x][4s + j] = byte j of y_s[x], so one source contributes one u32
// word and the producer does no byte shuffling -- and the constant operand
// holds V_j(s,t) = 2^(8j) F[s][t] mod p_t split into bytes:
//     B_i[4s + j][t] = byte i of V_j(s,t),   C_i = A . B_i  (i = 0..3)
//     sum_i 2^(8i) C_i = sum_{s,j} byte_j(y_s) V_j(s,t) == sum_s y_s F[s][t]  (mod p_t)
// C_i <= 32*KC*255^2 < 2^22, so sum_i 2^(8i) C_i < 2^46 < p_t 2^32 and one
// Montgomery step (V_j pre-scaled by 2^32) plus a conditional subtraction
// gives the canonical result -- bit-identical to the reference.
//
// K = 4*alpha bytes (one 32-byte MMA K-step for alpha <= 8, two for <= 16).
// Targets come in chunks of 32, and one MMA (M = 128 coefficients, N = 256)
// covers a chunk PAIR: its B operand holds both chunks' four byte planes
// side by side (n = 128 c + 32 i + t), so a tile costs KC MMAs per pair;
// TMEM holds two pair buffers (2 x 256 columns).
// Persistent, warp-specialised CTA (one per SM, 21 warps, <= 96 registers):
//   warps 0-3   producers: source rows arrive by one TMA tensor load per tile
//               kRawBC tiles ahead; y_s = a_s * qhat_inv (Shoup), 16-byte
//               st.shared of 4 sources per row into the K-major A ring
//   warps 4-19  epilogue: group h (8 warps) drains chunk h of the pair, warp
//               (lane quarter g, half hh) 16 targets of 32 rows: TMEM -> fold
//               -> Montgomery mod p_t -> [32 target][128 coefficient] staging
//               tile in shared memory (double-buffered per group), written by
//               ONE TMA tensor store per chunk (rows past n_dst and
//               coefficients past per_row clipped by the tensor map)
//   warp 20     TMEM owner; one elected lane issues the MMAs
// Copy targets (a target that is source prime s, rns.py:140-142) have the
// factors (Q/q_s) mod q_s and 0, so their column computes a_s mod q_s: the
// copy itself for canonical residues.  Producers flag non-canonical copy
// sources and a fixup launch then copies the raw rows (bit-exact for any u32
// input); callers that never read the copies (the key switch skips a slice's
// own rows) pass exact_copies = false.
// The kernel is HBM-bound by design (alpha*4 bytes read, T*4 written per
// coefficient); the tensor cores remove the alpha*T mul-mods per coefficient
// that bound the CUDA-core form.  Tiny conversions (alpha <= 4, alpha * T <=
// 32) take an element-wise fast path (bconv_small_kernel) instead of
// mostly-padding MMA tiles.  Timeline probes: -DTFHE_BC_TRACE.
#include <algorithm>
#include <atomic>
#include <mutex>
#include <cstring>
#include <string>
#include <vector>
#include <cstdio>

#include <cuda.h>

#include "common.cuh"
#include "poly_ops.h"
#include "tfhe_internal.h"

namespace tfhe {

namespace {

constexpr int kRowsBC = 128;
constexpr int kAStages = 4;
constexpr int kChunk = 32;           // targets per MMA (N)
constexpr int kMaxChunks = kMaxBconvDst / kChunk;
constexpr int kMaxKC = 2;            // 32-byte K-steps (alpha <= 16)
constexpr int kEpiWarpsBC = 16;         // 2 chunks x 2 target halves x 4 lane quarters
constexpr int kMmaWarpBC = 4 + kEpiWarpsBC;
constexpr int kThreadsBC = 32 * (kMmaWarpBC + 1);
constexpr int kATileBC = kRowsBC * 32;           // 4 KB per K-step
constexpr int kPairN = 256;                      // MMA N: two chunks x 4 planes x 32 targets
constexpr int kMaxPairs = kMaxChunks / 2;
constexpr int kBTileBC = kPairN * 32;            // 8 KB per (chunk pair, K-step)
constexpr int kRawBC = 8;                       // raw input tiles in flight (TMA ring)
constexpr int kMaxSrcBC = 16;
constexpr int kRawTileBC = kMaxSrcBC * kRowsBC * 4;   // 8 KB: 128 coefficients x 16 sources
constexpr int kStageWords = 2 * 2 * kChunk * kRowsBC;   // 64 KB: per epilogue group 2 x [32][128]

// timeline probes (-DTFHE_BC_TRACE): per-tile event clocks of CTA 0, lane 0
#ifdef TFHE_BC_TRACE
constexpr int kBTraceN = 128;
#define BTRACE(ev, i)                                                              \
  do {                                                                             \
    if (blockIdx.x == 0 && (tid & 31) == 0 && (i) < kBTraceN)                      \
      a.trace[(ev) * kBTraceN + (i)] = clock64();                                  \
  } while (0)
#else
#define BTRACE(ev, i) do { } while (0)
#endif

struct BconvTcArgs {
  const uint32_t* in;
  uint32_t* out;
  const PrimeConst* pc;
  int64_t per_row;     // batch * n coefficients per row
  int64_t tiles;       // ceil(per_row / 128)
  int KC, nchunks;
  int use_tmap;        // 1: one TMA tensor load per tile (per_row % 128 == 0)
  int use_tstore;      // 1: outputs leave through shared memory by TMA tensor stores
  CUtensorMap tmap;    // sources viewed as [n_src][per_row], box {128, n_src}
  CUtensorMap omap;    // targets viewed as [n_dst][per_row], box {128, 32}
  uint32_t* copy_flag; // tensor-store mode: set to copy_gen if a copy source is non-canonical
  uint32_t copy_gen;
  uint32_t copy_src_mask;   // sources some target copies through
  unsigned long long* trace;   // TFHE_BC_TRACE builds only
};

// st.global predicated on `p` (keeps a warp-uniform skip a predicate, not a branch)
TFHE_DEV void st_global_if(uint32_t* ptr, uint32_t v, bool p) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.global.u32 [%0], %1;\n\t}"
               ::"l"(ptr), "r"(v), "r"((uint32_t)p)
               : "memory");
}

// offset of (row r, byte k) inside a K-major SWIZZLE_NONE tile of `rows` x 32 bytes
TFHE_DEV uint32_t tile_off_bc(int r, int k, int rows) {
  return (uint32_t)((k >> 4) * (rows * 16) + (r >> 3) * 128 + (r & 7) * 16 + (k & 15));
}

__global__ void __launch_bounds__(kThreadsBC, 1)
    bconv_tc_kernel(const __grid_constant__ BconvTcArgs a, const __grid_constant__ BconvArgs ba) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int KC = a.KC, nch = a.nchunks;
  uint8_t* sB = smem;                                              // [i][chunk][kc] tiles
  uint8_t* sA = sB + kMaxPairs * kMaxKC * kBTileBC;                // [stage][kc] tiles
  uint8_t* sRaw = sA + kAStages * kMaxKC * kATileBC;               // [slot][src][128] u32
  uint32_t* sStage = reinterpret_cast<uint32_t*>(sRaw + kRawBC * kRawTileBC);  // [grp][2][32][128]
  uint32_t* sQ = sStage + kStageWords;                             // per target
  uint32_t* sQinv = sQ + kMaxBconvDst;                             // -q^-1 mod 2^32
  int* sCopy = reinterpret_cast<int*>(sQinv + kMaxBconvDst);      // copy list: t | s << 16
  int* sCopyLo = sCopy + kMaxBconvDst;                             // per chunk: first copy
  uint32_t* sSkip = reinterpret_cast<uint32_t*>(sCopyLo + 8);      // per 16 targets
  uint32_t* sSrcQ = sSkip + kMaxBconvDst / 16;                     // per source: q | qhat_inv | Shoup
  uint32_t* sSrcH = sSrcQ + kMaxSrcBC;
  uint32_t* sSrcHs = sSrcH + kMaxSrcBC;
  uint64_t* a_full = reinterpret_cast<uint64_t*>(sSrcHs + kMaxSrcBC);
  uint64_t* a_empty = a_full + kAStages;
  uint64_t* acc_full = a_empty + kAStages;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* raw_full = acc_empty + 2;
  uint64_t* raw_empty = raw_full + kRawBC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(raw_empty + kRawBC);

  const int tid = threadIdx.x, warp = tid >> 5;

  // constant operand: B_i[4s + j][t] = byte i of (2^(8j+32) F[s][t] mod p_t)
  // (the 2^32 is the Montgomery factor the epilogue's REDC removes)
  for (int w = tid; w < kMaxPairs * kMaxKC * kBTileBC / 4; w += blockDim.x)
    reinterpret_cast<uint32_t*>(sB)[w] = 0;
  __syncthreads();
  for (int e = tid; e < ba.n_src * ba.n_dst; e += blockDim.x) {
    const int s = e / ba.n_dst, t = e % ba.n_dst;
    const PrimeConst pt = a.pc[ba.dst_prime[t]];
    const uint64_t f = reduce64((uint64_t)ba.factor[s * kMaxBconvDst + t] << 32, pt.q, pt.mu);
    const int ch = t / kChunk, tr = t % kChunk;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t v = reduce64(f << (8 * j), pt.q, pt.mu);
      const int k = 4 * s + j, kc = k >> 5;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        sB[((ch >> 1) * kMaxKC + kc) * kBTileBC +
           tile_off_bc((ch & 1) * 128 + i * kChunk + tr, k & 31, kPairN)] =
            (uint8_t)(v >> (8 * i));
    }
  }
  for (int t = tid; t < kMaxBconvDst; t += blockDim.x) {
    const bool live = t < ba.n_dst;
    const PrimeConst pt = a.pc[live ? ba.dst_prime[t] : ba.dst_prime[0]];
    sQ[t] = pt.q;
    sQinv[t] = pt.qneg_inv;
  }
  int n_copy = 0;
  for (int t = 0; t < ba.n_dst; ++t) n_copy += ba.copy_from[t] >= 0;
  if (tid < kMaxSrcBC) {
    const bool live = tid < ba.n_src;
    sSrcQ[tid] = live ? a.pc[ba.src_prime[tid]].q : 1u;
    sSrcH[tid] = live ? ba.qhat_inv[tid] : 0u;
    sSrcHs[tid] = live ? ba.qhat_inv_shoup[tid] : 0u;
  }
  if (tid < kMaxBconvDst / 16) {
    // epilogue skip mask per 16 targets: copies (stored by the producers) and padding
    uint32_t m = 0;
    for (int e = 0; e < 16; ++e) {
      const int t = tid * 16 + e;
      if (t >= ba.n_dst || ba.copy_from[t] >= 0) m |= 1u << e;
    }
    sSkip[tid] = m;
  }
  if (tid == 0) {
    // copy list in target order, and each chunk's range of it
    int k = 0;
    for (int ch = 0; ch <= kMaxChunks; ++ch) {
      sCopyLo[ch] = k;
      if (ch == kMaxChunks) break;
      for (int t = ch * kChunk; t < (ch + 1) * kChunk && t < ba.n_dst; ++t)
        if (ba.copy_from[t] >= 0) sCopy[k++] = t | (ba.copy_from[t] << 16);
    }
  }
  if (tid == 0) {
    for (int s = 0; s < kAStages; ++s) {
      mbar_init(&a_full[s], 128);
      mbar_init(&a_empty[s], 1);
    }
    for (int s = 0; s < kRawBC; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&raw_empty[s], 128);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 32 * kEpiWarpsBC);   // both epilogue groups
    }
    fence_mbar_init();
  }
  if (warp == kMmaWarpBC) tmem_alloc<512>(tmem_slot);
  fence_proxy_async_smem();  // B tiles written by the generic proxy, read by the MMA
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // contiguous tile range of this CTA
  const int64_t t_lo = a.tiles * blockIdx.x / gridDim.x;
  const int64_t t_hi = a.tiles * (blockIdx.x + 1) / gridDim.x;
  const int n_tiles = (int)(t_hi - t_lo);

  if (warp < 4) {
    // ---------------------------------------------------------------- producers
    // Raw tiles (128 coefficients of each source row, contiguous 512-byte
    // segments) arrive by bulk copy kRawBC tiles ahead (one elected thread);
    // each thread then converts its coefficient: y_s = a_s * qhat_inv_s.
    const int r = tid;
    const int nsrc = ba.n_src;
    auto issue = [&](int it) {
      const int slot = it % kRawBC;
      const int64_t x0 = (t_lo + it) * kRowsBC;
      const uint32_t cnt = (uint32_t)std::min<int64_t>(kRowsBC, a.per_row - x0);
      mbar_arrive_expect_tx(&raw_full[slot], cnt * 4 * nsrc);
      if (a.use_tmap) {   // every source row of the tile in one tensor load
        tma_load_2d(sRaw + slot * kRawTileBC, &a.tmap, (int)x0, 0, &raw_full[slot]);
        return;
      }
      for (int s = 0; s < nsrc; ++s)
        bulk_g2s(sRaw + slot * kRawTileBC + s * kRowsBC * 4, a.in + (int64_t)s * a.per_row + x0,
                 cnt * 4, &raw_full[slot]);
    };
    if (tid == 0)
      for (int it = 0; it < kRawBC && it < n_tiles; ++it) issue(it);
    bool noncanon = false;
    for (int it = 0; it < n_tiles; ++it) {
      const int st = it % kAStages, slot = it % kRawBC;
      if (it >= kAStages) mbar_wait(&a_empty[st], ((it / kAStages) & 1) ^ 1);
      if (warp == 0) BTRACE(0, it);
      mbar_wait(&raw_full[slot], (it / kRawBC) & 1);
      if (warp == 0) BTRACE(1, it);
      const int64_t x = (t_lo + it) * kRowsBC + r;
      const bool valid = x < a.per_row;
      const uint32_t* raw = reinterpret_cast<const uint32_t*>(sRaw + slot * kRawTileBC);
      // branch-free: the source rows of the K-steps in use are read (rows >=
      // nsrc hold stale data; their qhat_inv = 0, q = 1 give y = 0), four
      // sources = one 16-byte segment of the A tile; rows past per_row are
      // clipped at the store.  Tensor-store mode computes a copy target as
      // y_s (Q/q_s) mod q_s = a_s mod q_s (a target that is source s has
      // factors (Q/q_s) and 0), a copy only if a_s < q_s: non-canonical copy
      // sources are flagged for the fixup launch.
      uint32_t y[kMaxSrcBC];
#pragma unroll
      for (int s0 = 0; s0 < kMaxSrcBC; s0 += 4) {
        if (s0 >= 8 * KC) break;
        const uint4 q4 = *reinterpret_cast<const uint4*>(sSrcQ + s0);
        const uint4 h4 = *reinterpret_cast<const uint4*>(sSrcH + s0);
        const uint4 p4 = *reinterpret_cast<const uint4*>(sSrcHs + s0);
        const uint32_t qv[4] = {q4.x, q4.y, q4.z, q4.w}, hv[4] = {h4.x, h4.y, h4.z, h4.w},
                       pv[4] = {p4.x, p4.y, p4.z, p4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t xs = raw[(s0 + e) * kRowsBC + r];
          y[s0 + e] = mul_shoup(xs, hv[e], pv[e], qv[e]);
          noncanon |= ((a.copy_src_mask >> (s0 + e)) & 1) && valid && xs >= qv[e];
        }
      }
      // targets that are source primes copy the source row through (rns.py:140-142):
      // per thread here, or row copies after the kernel (tensor-store mode)
      if (!a.use_tstore && valid) {
        for (int c = 0; c < n_copy; ++c) {
          const int e = sCopy[c];
          a.out[(int64_t)(e & 0xFFFF) * a.per_row + x] = raw[(e >> 16) * kRowsBC + r];
        }
      }
#ifdef TFHE_BC_TRACE_P
      if (warp == 0) BTRACE(13, it);
#endif
      mbar_arrive(&raw_empty[slot]);
      uint8_t* tile = sA + st * kMaxKC * kATileBC;
#pragma unroll
      for (int s0 = 0; s0 < kMaxSrcBC; s0 += 4) {   // 4 sources = one 16-byte segment
        if (s0 >= 8 * KC) break;
        const int k = 4 * s0;
        *reinterpret_cast<uint4*>(tile + (k >> 5) * kATileBC + tile_off_bc(r, k & 31, kRowsBC)) =
            make_uint4(y[s0], y[s0 + 1], y[s0 + 2], y[s0 + 3]);
      }
#ifdef TFHE_BC_TRACE_P
      if (warp == 0) BTRACE(14, it);
#endif
      fence_proxy_async_smem();
      mbar_arrive(&a_full[st]);
      if (warp == 0) BTRACE(2, it);
      // refill this raw slot once every producer thread has read it
      if (tid == 0 && it + kRawBC < n_tiles) {
        mbar_wait(&raw_empty[slot], (it / kRawBC) & 1);
        issue(it + kRawBC);
        BTRACE(12, it);
      }
    }
    if (noncanon) *a.copy_flag = a.copy_gen;   // same value from every writer
  } else if (warp < 4 + kEpiWarpsBC) {
    // ---------------------------------------------------------------- epilogue
    // Two groups of 4 warps take alternate (tile, chunk) units u (group h: u
    // odd / even, TMEM buffers {h, h + 2}), so two chunks drain at once; warp
    // 4 + 4h + g reads TMEM lane group g (rows 32g..32g+31) and all 32 targets
    // of its chunk in two halves.  The fold v = sum_i 2^(8i) C_i (< 2^48) is
    // reduced by one Montgomery step (R = 2^32, compensated in the constant
    // operand: V_j carries 2^32).  Tensor-store mode: results go to a
    // [32 target][128 coefficient] staging tile (double-buffered per group)
    // and one TMA tensor store per chunk writes the box (rows past n_dst and
    // coefficients past per_row clipped); a copy target's column computes
    // a_s mod q_s, i.e. the copy for canonical inputs (fixup kernel otherwise).
    const int we = warp - 4, g = we & 3, h = we >> 3, hh = (we >> 2) & 1;
    const int r = g * 32 + (tid & 31);
    const bool issuer = g == 0 && hh == 0 && (tid & 31) == 0;   // the group's store thread
    const uint32_t lane_base = tmem + ((uint32_t)(g * 32) << 16);
    uint32_t* stage0 = sStage + h * 2 * kChunk * kRowsBC;
    const int npairs = (nch + 1) >> 1;
    int v = 0, k = 0;
    for (int it = 0; it < n_tiles; ++it) {
      const int64_t x0 = (t_lo + it) * kRowsBC;
      const int64_t x = x0 + r;
      const bool valid = x < a.per_row;
      for (int cp = 0; cp < npairs; ++cp, ++v) {
        // unit v = (tile, chunk pair): group h drains chunk 2 cp + h, warp
        // (g, hh) its TMEM lane quarter g and targets [16 hh, 16 hh + 16)
        const int buf = v & 1, ch = 2 * cp + h;
        mbar_wait(&acc_full[buf], (v >> 1) & 1);
        if (ch >= nch) {   // odd last pair: nothing to drain, release at once
          mbar_arrive(&acc_empty[buf]);
          continue;
        }
        uint32_t* stg = stage0 + (k & 1) * kChunk * kRowsBC;
        if (g == 0 && hh == 0) BTRACE(6 + 3 * h, it);
        tc_fence_after();
        if (a.use_tstore) named_bar(1 + h, 16 * kEpiWarpsBC);   // staging buffer free again
#pragma unroll
        for (int q8 = 0; q8 < 2; ++q8) {
          uint32_t c[4][8];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            tmem_ld8(lane_base + buf * kPairN + h * 128 + i * kChunk + hh * 16 + q8 * 8, c[i]);
          tmem_ld_wait();
          if (q8 == 1) {
            tc_fence_before();
            mbar_arrive(&acc_empty[buf]);
            if (g == 0 && hh == 0) BTRACE(7 + 3 * h, it);
          }
          const int tb = ch * kChunk + hh * 16 + q8 * 8;
          if (tb >= ba.n_dst) continue;
          const uint4 qa = *reinterpret_cast<const uint4*>(sQ + tb);
          const uint4 qb = *reinterpret_cast<const uint4*>(sQ + tb + 4);
          const uint4 ia = *reinterpret_cast<const uint4*>(sQinv + tb);
          const uint4 ib = *reinterpret_cast<const uint4*>(sQinv + tb + 4);
          const uint32_t qv[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
          const uint32_t qi[8] = {ia.x, ia.y, ia.z, ia.w, ib.x, ib.y, ib.z, ib.w};
          uint32_t w[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const uint32_t t = fold4_redc(c[0][e], c[1][e], c[2][e], c[3][e], qv[e], qi[e]);
            w[e] = min(t, t - qv[e]);   // [0, 2q) -> [0, q)
          }
          if (a.use_tstore) {
#pragma unroll
            for (int e = 0; e < 8; ++e) stg[(tb - ch * kChunk + e) * kRowsBC + r] = w[e];
          } else if (valid) {
            // per-thread stores down the target rows (skip = copies and padding)
            const uint32_t skip = sSkip[tb >> 4] >> (tb & 15);
            uint32_t* o = a.out + (int64_t)tb * a.per_row + x;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              st_global_if(o, w[e], ((skip >> e) & 1) == 0);
              o += a.per_row;
            }
          }
        }
        if (a.use_tstore) {
          fence_proxy_async_smem();   // generic-proxy staging writes -> TMA reads
          named_bar(1 + h, 16 * kEpiWarpsBC);
          if (issuer) {
            tma_store_2d(&a.omap, stg, (int)x0, ch * kChunk);
            bulk_commit();
            bulk_wait_read<1>();   // the other staging buffer is free for the next chunk
          }
          __syncwarp();
        }
        if (g == 0 && hh == 0) BTRACE(8 + 3 * h, it);
        ++k;
      }
    }
    if (issuer && a.use_tstore) bulk_wait_all();
  } else {
    // ---------------------------------------------------------------- MMA issuer
    // one MMA per (tile, chunk pair, K-step): N = 256 covers both chunks'
    // four byte-plane accumulators side by side (n = 128 c + 32 i + t)
    constexpr uint32_t idesc2 = idesc_i8(kRowsBC, kPairN), idesc1 = idesc_i8(kRowsBC, kPairN / 2);
    const bool leader = elect_one();
    const int npairs = (nch + 1) >> 1;
    int v = 0;
    for (int it = 0; it < n_tiles; ++it) {
      const int st = it % kAStages;
      mbar_wait(&a_full[st], (it / kAStages) & 1);
      BTRACE(3, it);
      tc_fence_after();
      const uint32_t aBase = smem_u32(sA + st * kMaxKC * kATileBC);
      for (int cp = 0; cp < npairs; ++cp, ++v) {
        const int buf = v & 1;
        if (v >= 2) mbar_wait(&acc_empty[buf], ((v >> 1) & 1) ^ 1);
        BTRACE(4 + (cp & 1), it);
        tc_fence_after();
        if (leader) {
          const uint32_t id = 2 * cp + 1 < nch ? idesc2 : idesc1;
          for (int kc = 0; kc < KC; ++kc) {
            const uint64_t adesc = smem_desc_kmajor(aBase + kc * kATileBC, kRowsBC * 16, 128);
            const uint64_t bdesc =
                smem_desc_kmajor(smem_u32(sB + (cp * kMaxKC + kc) * kBTileBC), kPairN * 16, 128);
            mma_i8_ss(tmem + buf * kPairN, adesc, bdesc, id, kc != 0);
          }
          mma_commit(&acc_full[buf]);
        }
        __syncwarp();
#ifdef TFHE_BC_TRACE_M
        mbar_wait(&acc_full[buf], (v >> 1) & 1);   // trace only: MMA completion latency
        BTRACE(5, it);
#endif
      }
      if (leader) mma_commit(&a_empty[st]);
      __syncwarp();
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarpBC) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// Element-wise fast path for tiny conversions (n_src <= 4, n_src * n_dst <=
// 32: ModDown with K = 2..4 specials, ModUp slices of alpha = 2..4 onto a
// few targets), where a 128-row MMA tile would carry mostly padding: each
// thread converts 4 coefficients (uint4) for every target -- the alpha
// products of one target (< 4 * 2^62) are summed in 64 bits and reduced once.
template <int NS>
__global__ void __launch_bounds__(256)
    bconv_small_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                       const PrimeConst* __restrict__ pcs, const __grid_constant__ BconvArgs ba,
                       int64_t per_row, int64_t in_cstride, int64_t out_cstride) {
  in += blockIdx.y * in_cstride;     // component (blockIdx.y) of a multi-component launch
  out += blockIdx.y * out_cstride;
  // NS sources (compile time): all source loads of two 4-coefficient groups
  // are issued before any arithmetic (memory-level parallelism)
  const int64_t step = (int64_t)gridDim.x * blockDim.x * 4;
  for (int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4; i0 < per_row;
       i0 += 2 * step) {
    uint4 v[2][NS];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int s = 0; s < NS; ++s)
        v[h][s] = i0 + h * step < per_row
                      ? __ldg(reinterpret_cast<const uint4*>(in + (int64_t)s * per_row + i0 + h * step))
                      : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t i = i0 + h * step;
      if (i >= per_row) break;
      uint32_t a[NS][4], y[NS][4];
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        a[s][0] = v[h][s].x; a[s][1] = v[h][s].y; a[s][2] = v[h][s].z; a[s][3] = v[h][s].w;
        const uint32_t q = pcs[ba.src_prime[s]].q;
#pragma unroll
        for (int e = 0; e < 4; ++e)
          y[s][e] = mul_shoup(a[s][e], ba.qhat_inv[s], ba.qhat_inv_shoup[s], q);
      }
      for (int t = 0; t < ba.n_dst; ++t) {
        uint32_t r[4];
        const int cp = ba.copy_from[t];
        if (cp >= 0) {
#pragma unroll
          for (int s = 0; s < NS; ++s)
            if (s == cp) {
#pragma unroll
              for (int e = 0; e < 4; ++e) r[e] = a[s][e];
            }
        } else {
          const PrimeConst pt = pcs[ba.dst_prime[t]];
          uint64_t acc[4] = {0, 0, 0, 0};
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            const uint64_t f = ba.factor[s * kMaxBconvDst + t];
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[e] += (uint64_t)y[s][e] * f;
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) r[e] = reduce64(acc[e], pt.q, pt.mu);
        }
        *reinterpret_cast<uint4*>(out + (int64_t)t * per_row + i) = make_uint4(r[0], r[1], r[2], r[3]);
      }
    }
  }
}

// Copy-through fixup of the tensor-store mode: runs after bconv_tc_kernel and
// does nothing unless that launch flagged a non-canonical copy source (then
// the copy targets get the raw source rows, rns.py:140-142).
__global__ void __launch_bounds__(256)
    bconv_copy_fixup_kernel(const uint32_t* __restrict__ flag, uint32_t gen,
                            const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                            const __grid_constant__ BconvArgs ba, int64_t per_row) {
  if (*flag != gen) return;
  for (int t = 0; t < ba.n_dst; ++t) {
    const int s = ba.copy_from[t];
    if (s < 0) continue;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < per_row;
         i += (int64_t)gridDim.x * blockDim.x)
      out[(int64_t)t * per_row + i] = in[(int64_t)s * per_row + i];
  }
}

}  // namespace

int launch_bconv(const Ctx& c, const uint32_t* in, uint32_t* out, const BconvArgs& ba, int batch,
                 cudaStream_t st, bool exact_copies, int n_comp, int64_t in_cstride,
                 int64_t out_cstride) {
  if (ba.n_dst <= 0) return 0;
  if (ba.n_src < 1 || ba.n_src > 4 * kMaxKC * 2 || ba.n_dst > kMaxBconvDst || n_comp < 1) {
    set_error("base conversion: 1..16 sources and at most 128 targets");
    return 2;
  }
  if (ba.n_src <= 4 && ba.n_src * ba.n_dst <= 32 && (batch * (int64_t)c.n) % 4 == 0) {
    // element-wise path: every component in one launch (blockIdx.y)
    const int64_t per_row = (int64_t)batch * c.n;
    const int64_t blocks =
        std::min<int64_t>((per_row / 4 + 255) / 256, (int64_t)c.sms * 8 / n_comp);
    const dim3 grid((unsigned)std::max<int64_t>(blocks, 1), n_comp);
    switch (ba.n_src) {
      case 1: bconv_small_kernel<1><<<grid, 256, 0, st>>>(in, out, c.d_pc, ba, per_row, in_cstride, out_cstride); break;
      case 2: bconv_small_kernel<2><<<grid, 256, 0, st>>>(in, out, c.d_pc, ba, per_row, in_cstride, out_cstride); break;
      case 3: bconv_small_kernel<3><<<grid, 256, 0, st>>>(in, out, c.d_pc, ba, per_row, in_cstride, out_cstride); break;
      default: bconv_small_kernel<4><<<grid, 256, 0, st>>>(in, out, c.d_pc, ba, per_row, in_cstride, out_cstride); break;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      set_error(std::string("bconv_small launch: ") + cudaGetErrorString(e));
      return 3;
    }
    return 0;
  }
  if (n_comp > 1) {
    for (int k = 0; k < n_comp; ++k) {
      const int rc = launch_bconv(c, in + k * in_cstride, out + k * out_cstride, ba, batch, st,
                                  exact_copies);
      if (rc) return rc;
    }
    return 0;
  }
  BconvTcArgs a;
  memset(&a, 0, sizeof(a));
  a.in = in;
  a.out = out;
  a.pc = c.d_pc;
  a.per_row = (int64_t)batch * c.n;
  a.tiles = (a.per_row + kRowsBC - 1) / kRowsBC;
  a.KC = (4 * ba.n_src + 31) / 32;
  a.nchunks = (ba.n_dst + kChunk - 1) / kChunk;
  a.use_tmap = 0;
  if (a.per_row % kRowsBC == 0) {
    typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn fn = nullptr;
    if (!fn) {
      cudaDriverEntryPointQueryResult qr;
      void* p = nullptr;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) ==
              cudaSuccess &&
          qr == cudaDriverEntryPointSuccess)
        fn = reinterpret_cast<EncodeFn>(p);
    }
    cuuint64_t dims[2] = {(cuuint64_t)a.per_row, (cuuint64_t)ba.n_src};
    cuuint64_t strides[1] = {(cuuint64_t)a.per_row * 4};
    cuuint32_t box[2] = {(cuuint32_t)kRowsBC, (cuuint32_t)ba.n_src};
    cuuint32_t es[2] = {1, 1};
    if (fn && fn(&a.tmap, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint32_t*>(in), dims,
                 strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
      a.use_tmap = 1;
  }
  a.use_tstore = 0;
  if (a.use_tmap && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
    // (encoder fetched above with the input map; per_row % 128 == 0 there)
    typedef CUresult (*EncodeFn2)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    cudaDriverEntryPointQueryResult qr;
    void* pfn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &pfn, cudaEnableDefault, &qr) ==
            cudaSuccess && qr == cudaDriverEntryPointSuccess) {
      cuuint64_t od[2] = {(cuuint64_t)a.per_row, (cuuint64_t)ba.n_dst};
      cuuint64_t os[1] = {(cuuint64_t)a.per_row * 4};
      cuuint32_t ob[2] = {(cuuint32_t)kRowsBC, (cuuint32_t)kChunk};
      cuuint32_t oe[2] = {1, 1};
      if (reinterpret_cast<EncodeFn2>(pfn)(&a.omap, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, out, od, os,
                                           ob, oe, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                           CU_TENSOR_MAP_SWIZZLE_NONE,
                                           CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
        a.use_tstore = 1;
    }
  }
  if (getenv("TFHE_BC_NO_TSTORE")) a.use_tstore = 0;
  // copy-through bookkeeping (tensor-store mode, callers that read the copies)
  a.copy_src_mask = 0;
  if (a.use_tstore && exact_copies) {
    for (int t = 0; t < ba.n_dst; ++t)
      if (ba.copy_from[t] >= 0) a.copy_src_mask |= 1u << ba.copy_from[t];
    if (a.copy_src_mask) {
      // one flag word per launch from a per-device ring, tagged with a
      // process-wide launch generation: concurrent launches (other streams or
      // threads) never share a word unless kFlagSlots are in flight at once
      constexpr int kFlagSlots = 1024;
      static std::mutex mu;
      static uint32_t* flags[64] = {nullptr};
      static std::atomic<uint32_t> gen{0};
      uint32_t* f;
      {
        std::lock_guard<std::mutex> g(mu);
        uint32_t*& slot = flags[c.dev & 63];
        if (!slot) {
          if (cudaMalloc(&slot, kFlagSlots * 4) != cudaSuccess ||
              cudaMemset(slot, 0, kFlagSlots * 4) != cudaSuccess) {
            slot = nullptr;
            set_error("bconv copy flag allocation failed");
            return 3;
          }
        }
        f = slot;
      }
      uint32_t gg = ++gen;
      if (gg == 0) gg = ++gen;
      a.copy_flag = f + gg % kFlagSlots;
      a.copy_gen = gg;
    }
  }
  const int smem = kMaxPairs * kMaxKC * kBTileBC + kAStages * kMaxKC * kATileBC +
                   kRawBC * kRawTileBC + kStageWords * 4 + kMaxBconvDst * (4 + 4 + 4) +
                   8 * 4 + 3 * kMaxSrcBC * 4 +
                   kMaxBconvDst / 16 * 4 +
                   (2 * kAStages + 4 + 2 * kRawBC) * 8 + 16;
  static std::atomic<bool> attr[64];   // function attributes are per device
  if (!attr[c.dev & 63].load(std::memory_order_relaxed)) {
    cudaFuncSetAttribute(bconv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr[c.dev & 63].store(true, std::memory_order_relaxed);
  }
  const int grid = (int)std::min<int64_t>(a.tiles, c.sms);
#ifdef TFHE_BC_TRACE
  static unsigned long long* tbuf = nullptr;
  if (!tbuf) cudaMalloc(&tbuf, 16 * kBTraceN * 8);
  cudaMemsetAsync(tbuf, 0, 16 * kBTraceN * 8, st);
  a.trace = tbuf;
#endif
  prof_begin("bconv_tc_kernel", st);
  bconv_tc_kernel<<<grid, kThreadsBC, smem, st>>>(a, ba);
  prof_end(st);
  // tensor-store mode: copy targets (rns.py:140-142) equal a_s mod q_s, the
  // copy itself unless the input was non-canonical -- then the fixup copies
  if (a.copy_src_mask) {
    bconv_copy_fixup_kernel<<<c.sms * 4, 256, 0, st>>>(a.copy_flag, a.copy_gen, in, out, ba,
                                                        a.per_row);
  }
#ifdef TFHE_BC_TRACE
  {
    std::vector<unsigned long long> hb(16 * kBTraceN);
    cudaMemcpy(hb.data(), tbuf, hb.size() * 8, cudaMemcpyDeviceToHost);
    static int seq = 0;
    char fn[256];
    snprintf(fn, sizeof(fn), "gpurun_out/btrace_%d.bin", seq++);
    if (FILE* f = fopen(fn, "wb")) {
      fwrite(hb.data(), 8, hb.size(), f);
      fclose(f);
    }
  }
#endif
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("bconv_tc launch: ") + cudaGetErrorString(e));
    return 3;
  }
  return 0;
}

}  // namespace tfhe
