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
// C_i <= 32*KC*255^2 < 2^24, so sum_i 2^(8i) C_i < 2^48 and one Barrett step
// gives the canonical result -- bit-identical to the reference.
//
// K = 4*alpha bytes (one 32-byte MMA K-step for alpha <= 8, two for <= 16);
// targets are processed in chunks of 32 (N = 32): a chunk is 4 MMAs into
// 4 x 32 TMEM columns, and TMEM holds 4 chunk buffers (512 columns).
// Persistent, warp-specialised CTA (one per SM):
//   warps 0-3  producers: y_s = a_s * qhat_inv (Shoup), 16-byte st.shared of
//              4 sources per row into the K-major A ring (kAStages tiles)
//   warps 4-7  epilogue: TMEM -> fold -> Barrett mod p_t -> coalesced stores
//   warp 8     TMEM owner; one elected lane issues the MMAs
// The kernel is HBM-bound for small alpha (alpha*4 bytes read, T*4 written
// per coefficient); the tensor cores remove the alpha*T mul-mods per
// coefficient that bound the CUDA-core form at large alpha.
#include <cstring>
#include <string>

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
constexpr int kThreadsBC = 288;
constexpr int kATileBC = kRowsBC * 32;           // 4 KB per K-step
constexpr int kBTileBC = kChunk * 32;            // 1 KB per (i, chunk, K-step)

struct BconvTcArgs {
  const uint32_t* in;
  uint32_t* out;
  const PrimeConst* pc;
  int64_t per_row;     // batch * n coefficients per row
  int64_t tiles;       // ceil(per_row / 128)
  int KC, nchunks;
};

// offset of (row r, byte k) inside a K-major SWIZZLE_NONE tile of `rows` x 32 bytes
TFHE_DEV uint32_t tile_off_bc(int r, int k, int rows) {
  return (uint32_t)((k >> 4) * (rows * 16) + (r >> 3) * 128 + (r & 7) * 16 + (k & 15));
}

__global__ void __launch_bounds__(kThreadsBC, 1)
    bconv_tc_kernel(const __grid_constant__ BconvTcArgs a, const __grid_constant__ BconvArgs ba) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int KC = a.KC, nch = a.nchunks;
  uint8_t* sB = smem;                                              // [i][chunk][kc] tiles
  uint8_t* sA = sB + 4 * kMaxChunks * kMaxKC * kBTileBC;           // [stage][kc] tiles
  uint64_t* a_full = reinterpret_cast<uint64_t*>(sA + kAStages * kMaxKC * kATileBC);
  uint64_t* a_empty = a_full + kAStages;
  uint64_t* acc_full = a_empty + kAStages;
  uint64_t* acc_empty = acc_full + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 4);

  const int tid = threadIdx.x, warp = tid >> 5;

  // constant operand: B_i[4s + j][t] = byte i of (2^(8j) F[s][t] mod p_t)
  for (int w = tid; w < 4 * kMaxChunks * kMaxKC * kBTileBC / 4; w += blockDim.x)
    reinterpret_cast<uint32_t*>(sB)[w] = 0;
  __syncthreads();
  for (int e = tid; e < ba.n_src * ba.n_dst; e += blockDim.x) {
    const int s = e / ba.n_dst, t = e % ba.n_dst;
    const PrimeConst pt = a.pc[ba.dst_prime[t]];
    const uint64_t f = ba.factor[s * kMaxBconvDst + t];
    const int ch = t / kChunk, tr = t % kChunk;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t v = reduce64(f << (8 * j), pt.q, pt.mu);
      const int k = 4 * s + j, kc = k >> 5;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        sB[((i * kMaxChunks + ch) * kMaxKC + kc) * kBTileBC + tile_off_bc(tr, k & 31, kChunk)] =
            (uint8_t)(v >> (8 * i));
    }
  }
  if (tid == 0) {
    for (int s = 0; s < kAStages; ++s) {
      mbar_init(&a_full[s], 128);
      mbar_init(&a_empty[s], 1);
    }
    for (int b = 0; b < 4; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 128);
    }
    fence_mbar_init();
  }
  if (warp == 8) tmem_alloc<512>(tmem_slot);
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
    const int r = tid;
    for (int it = 0; it < n_tiles; ++it) {
      const int st = it % kAStages;
      if (it >= kAStages) mbar_wait(&a_empty[st], ((it / kAStages) & 1) ^ 1);
      const int64_t x = (t_lo + it) * kRowsBC + r;
      const bool valid = x < a.per_row;
      uint8_t* tile = sA + st * kMaxKC * kATileBC;
      for (int s0 = 0; s0 < 8 * KC; s0 += 4) {   // 4 sources = one 16-byte segment
        uint32_t y[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int s = s0 + q;
          y[q] = 0;
          if (valid && s < ba.n_src) {
            const uint32_t v = __ldg(a.in + (int64_t)s * a.per_row + x);
            y[q] = mul_shoup(v, ba.qhat_inv[s], ba.qhat_inv_shoup[s],
                             a.pc[ba.src_prime[s]].q);
          }
        }
        const int k = 4 * s0;
        *reinterpret_cast<uint4*>(tile + (k >> 5) * kATileBC + tile_off_bc(r, k & 31, kRowsBC)) =
            make_uint4(y[0], y[1], y[2], y[3]);
      }
      fence_proxy_async_smem();
      mbar_arrive(&a_full[st]);
    }
  } else if (warp < 8) {
    // ---------------------------------------------------------------- epilogue
    const int ew = warp - 4, r = ew * 32 + (tid & 31);
    const uint32_t lane_base = tmem + ((uint32_t)(ew * 32) << 16);
    int u = 0;
    for (int it = 0; it < n_tiles; ++it) {
      const int64_t x = (t_lo + it) * kRowsBC + r;
      const bool valid = x < a.per_row;
      for (int ch = 0; ch < nch; ++ch, ++u) {
        const int buf = u & 3;
        mbar_wait(&acc_full[buf], (u >> 2) & 1);
        tc_fence_after();
        uint32_t c[4][16], d[4][16];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          tmem_ld16(lane_base + buf * 128 + i * kChunk, c[i]);
          tmem_ld16(lane_base + buf * 128 + i * kChunk + 16, d[i]);
        }
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&acc_empty[buf]);
        if (!valid) continue;
        const int tb = ch * kChunk;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int t = tb + h * 16 + e;
            if (t >= ba.n_dst) break;
            const uint32_t c0 = h ? d[0][e] : c[0][e], c1 = h ? d[1][e] : c[1][e];
            const uint32_t c2 = h ? d[2][e] : c[2][e], c3 = h ? d[3][e] : c[3][e];
            uint32_t v;
            const int cp = ba.copy_from[t];
            if (cp >= 0) {
              v = __ldg(a.in + (int64_t)cp * a.per_row + x);
            } else {
              const PrimeConst pt = a.pc[ba.dst_prime[t]];
              const uint64_t f = (uint64_t)c0 + ((uint64_t)c1 << 8) + ((uint64_t)c2 << 16) +
                                 ((uint64_t)c3 << 24);
              v = reduce64(f, pt.q, pt.mu);
            }
            a.out[(int64_t)t * a.per_row + x] = v;
          }
        }
      }
    }
  } else {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = idesc_i8(kRowsBC, kChunk);
    const bool leader = elect_one();
    int u = 0;
    for (int it = 0; it < n_tiles; ++it) {
      const int st = it % kAStages;
      mbar_wait(&a_full[st], (it / kAStages) & 1);
      tc_fence_after();
      const uint32_t aBase = smem_u32(sA + st * kMaxKC * kATileBC);
      for (int ch = 0; ch < nch; ++ch, ++u) {
        const int buf = u & 3;
        if (u >= 4) mbar_wait(&acc_empty[buf], ((u >> 2) & 1) ^ 1);
        tc_fence_after();
        if (leader) {
          for (int kc = 0; kc < KC; ++kc) {
            const uint64_t adesc = smem_desc_kmajor(aBase + kc * kATileBC, kRowsBC * 16, 128);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint32_t bAddr =
                  smem_u32(sB + ((i * kMaxChunks + ch) * kMaxKC + kc) * kBTileBC);
              const uint64_t bdesc = smem_desc_kmajor(bAddr, kChunk * 16, 128);
              mma_i8_ss(tmem + buf * 128 + i * kChunk, adesc, bdesc, idesc, kc != 0);
            }
          }
          mma_commit(&acc_full[buf]);
        }
        __syncwarp();
      }
      if (leader) mma_commit(&a_empty[st]);
      __syncwarp();
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace

int launch_bconv(const Ctx& c, const uint32_t* in, uint32_t* out, const BconvArgs& ba, int batch,
                 cudaStream_t st) {
  if (ba.n_dst <= 0) return 0;
  if (ba.n_src < 1 || ba.n_src > 4 * kMaxKC * 2 || ba.n_dst > kMaxBconvDst) {
    set_error("base conversion: 1..16 sources and at most 128 targets");
    return 2;
  }
  BconvTcArgs a;
  a.in = in;
  a.out = out;
  a.pc = c.d_pc;
  a.per_row = (int64_t)batch * c.n;
  a.tiles = (a.per_row + kRowsBC - 1) / kRowsBC;
  a.KC = (4 * ba.n_src + 31) / 32;
  a.nchunks = (ba.n_dst + kChunk - 1) / kChunk;
  const int smem = 4 * kMaxChunks * kMaxKC * kBTileBC + kAStages * kMaxKC * kATileBC +
                   (2 * kAStages + 8) * 8 + 16;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(bconv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  const int grid = (int)std::min<int64_t>(a.tiles, c.sms);
  bconv_tc_kernel<<<grid, kThreadsBC, smem, st>>>(a, ba);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("bconv_tc launch: ") + cudaGetErrorString(e));
    return 3;
  }
  return 0;
}

}  // namespace tfhe
