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
// K = 4*alpha bytes (one 32-byte MMA K-step for alpha <= 8, two for <= 16);
// targets are processed in chunks of 32 (N = 32): a chunk is 4 MMAs into
// 4 x 32 TMEM columns, and TMEM holds 4 chunk buffers (512 columns).
// Persistent, warp-specialised CTA (one per SM):
//   warps 0-3  producers: source segments arrive by bulk copy (TMA engine)
//              kRawBC tiles ahead; y_s = a_s * qhat_inv (Shoup), 16-byte
//              st.shared of 4 sources per row into the K-major A ring
//   warps 4-11 epilogue: TMEM -> fold -> Montgomery mod p_t -> coalesced stores
//              (two warps per TMEM lane group, each half of a target chunk)
//   warp 12    TMEM owner; one elected lane issues the MMAs
// The kernel is HBM-bound for small alpha (alpha*4 bytes read, T*4 written
// per coefficient); the tensor cores remove the alpha*T mul-mods per
// coefficient that bound the CUDA-core form at large alpha.  Tiny
// conversions (alpha <= 4, alpha * T <= 32) take an element-wise fast path
// (bconv_small_kernel) instead of mostly-padding MMA tiles.
#include <algorithm>
#include <cstring>
#include <string>

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
constexpr int kEpiWarpsBC = 8;
constexpr int kMmaWarpBC = 4 + kEpiWarpsBC;
constexpr int kThreadsBC = 32 * (kMmaWarpBC + 1);
constexpr int kATileBC = kRowsBC * 32;           // 4 KB per K-step
constexpr int kBTileBC = kChunk * 32;            // 1 KB per (i, chunk, K-step)
constexpr int kRawBC = 6;                        // raw input tiles in flight (TMA ring)
constexpr int kMaxSrcBC = 16;
constexpr int kRawTileBC = kMaxSrcBC * kRowsBC * 4;   // 8 KB: 128 coefficients x 16 sources

struct BconvTcArgs {
  const uint32_t* in;
  uint32_t* out;
  const PrimeConst* pc;
  int64_t per_row;     // batch * n coefficients per row
  int64_t tiles;       // ceil(per_row / 128)
  int KC, nchunks;
  int use_tmap;        // 1: one TMA tensor load per tile (per_row % 128 == 0)
  CUtensorMap tmap;    // sources viewed as [n_src][per_row], box {128, n_src}
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
  uint8_t* sA = sB + 4 * kMaxChunks * kMaxKC * kBTileBC;           // [stage][kc] tiles
  uint8_t* sRaw = sA + kAStages * kMaxKC * kATileBC;               // [slot][src][128] u32
  uint32_t* sQ = reinterpret_cast<uint32_t*>(sRaw + kRawBC * kRawTileBC);  // per target
  uint32_t* sQinv = sQ + kMaxBconvDst;                             // -q^-1 mod 2^32
  int* sCopy = reinterpret_cast<int*>(sQinv + kMaxBconvDst);      // copy list: t | s << 16
  uint32_t* sSkip = reinterpret_cast<uint32_t*>(sCopy + kMaxBconvDst);  // per 16 targets
  uint64_t* a_full = reinterpret_cast<uint64_t*>(sSkip + kMaxBconvDst / 16);
  uint64_t* a_empty = a_full + kAStages;
  uint64_t* acc_full = a_empty + kAStages;
  uint64_t* acc_empty = acc_full + 4;
  uint64_t* raw_full = acc_empty + 4;
  uint64_t* raw_empty = raw_full + kRawBC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(raw_empty + kRawBC);

  const int tid = threadIdx.x, warp = tid >> 5;

  // constant operand: B_i[4s + j][t] = byte i of (2^(8j+32) F[s][t] mod p_t)
  // (the 2^32 is the Montgomery factor the epilogue's REDC removes)
  for (int w = tid; w < 4 * kMaxChunks * kMaxKC * kBTileBC / 4; w += blockDim.x)
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
        sB[((i * kMaxChunks + ch) * kMaxKC + kc) * kBTileBC + tile_off_bc(tr, k & 31, kChunk)] =
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
    int k = 0;
    for (int t = 0; t < ba.n_dst; ++t)
      if (ba.copy_from[t] >= 0) sCopy[k++] = t | (ba.copy_from[t] << 16);
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
    for (int b = 0; b < 4; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 32 * kEpiWarpsBC / 2);   // one epilogue group per buffer
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
    uint32_t qs[kMaxSrcBC], hs[kMaxSrcBC], hss[kMaxSrcBC];
#pragma unroll
    for (int s = 0; s < kMaxSrcBC; ++s) {
      qs[s] = s < nsrc ? a.pc[ba.src_prime[s]].q : 1;
      hs[s] = s < nsrc ? ba.qhat_inv[s] : 0;
      hss[s] = s < nsrc ? ba.qhat_inv_shoup[s] : 0;
    }
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
    for (int it = 0; it < n_tiles; ++it) {
      const int st = it % kAStages, slot = it % kRawBC;
      if (it >= kAStages) mbar_wait(&a_empty[st], ((it / kAStages) & 1) ^ 1);
      mbar_wait(&raw_full[slot], (it / kRawBC) & 1);
      const int64_t x = (t_lo + it) * kRowsBC + r;
      const bool valid = x < a.per_row;
      const uint32_t* raw = reinterpret_cast<const uint32_t*>(sRaw + slot * kRawTileBC);
      uint32_t y[kMaxSrcBC];
#pragma unroll
      for (int s = 0; s < kMaxSrcBC; ++s)
        y[s] = (valid && s < nsrc) ? mul_shoup(raw[s * kRowsBC + r], hs[s], hss[s], qs[s]) : 0;
      // targets that are source primes copy the source row through (rns.py:140-142)
      if (valid)
        for (int c = 0; c < n_copy; ++c) {
          const int e = sCopy[c];
          a.out[(int64_t)(e & 0xFFFF) * a.per_row + x] = raw[(e >> 16) * kRowsBC + r];
        }
      mbar_arrive(&raw_empty[slot]);
      uint8_t* tile = sA + st * kMaxKC * kATileBC;
#pragma unroll
      for (int s0 = 0; s0 < kMaxSrcBC; s0 += 4) {   // 4 sources = one 16-byte segment
        if (s0 >= 8 * KC) break;
        const int k = 4 * s0;
        *reinterpret_cast<uint4*>(tile + (k >> 5) * kATileBC + tile_off_bc(r, k & 31, kRowsBC)) =
            make_uint4(y[s0], y[s0 + 1], y[s0 + 2], y[s0 + 3]);
      }
      fence_proxy_async_smem();
      mbar_arrive(&a_full[st]);
      // refill this raw slot once every producer thread has read it
      if (tid == 0 && it + kRawBC < n_tiles) {
        mbar_wait(&raw_empty[slot], (it / kRawBC) & 1);
        issue(it + kRawBC);
      }
    }
  } else if (warp < 4 + kEpiWarpsBC) {
    // ---------------------------------------------------------------- epilogue
    // Two groups of 4 warps take alternate (tile, chunk) units u (group h: u
    // odd / even, TMEM buffers {h, h + 2}), so two chunks drain at once; warp
    // 4 + 4h + g reads TMEM lane group g (rows 32g..32g+31) and all 32 targets
    // of its chunk in two halves.  The fold v = sum_i 2^(8i) C_i (< 2^48) is
    // reduced by one Montgomery step (R = 2^32, compensated in the constant
    // operand: V_j carries 2^32).
    const int g = (warp - 4) & 3, h = (warp - 4) >> 2, r = g * 32 + (tid & 31);
    const uint32_t lane_base = tmem + ((uint32_t)(g * 32) << 16);
    int u = 0;
    for (int it = 0; it < n_tiles; ++it) {
      const int64_t x = (t_lo + it) * kRowsBC + r;
      const bool valid = x < a.per_row;
      for (int ch = 0; ch < nch; ++ch, ++u) {
        if ((u & 1) != h) continue;
        const int buf = u & 3;
        mbar_wait(&acc_full[buf], (u >> 2) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t c[4][16];
#pragma unroll
          for (int i = 0; i < 4; ++i) tmem_ld16(lane_base + buf * 128 + i * kChunk + hh * 16, c[i]);
          tmem_ld_wait();
          if (hh == 1) {
            tc_fence_before();
            mbar_arrive(&acc_empty[buf]);
          }
          const int tb = ch * kChunk + hh * 16;
          if (!valid || tb >= ba.n_dst) continue;
          const uint32_t skip = sSkip[tb >> 4];
          uint32_t qv[16], qi[16];
#pragma unroll
          for (int e = 0; e < 16; e += 4) {
            const uint4 q4 = *reinterpret_cast<const uint4*>(sQ + tb + e);
            const uint4 i4 = *reinterpret_cast<const uint4*>(sQinv + tb + e);
            qv[e] = q4.x; qv[e + 1] = q4.y; qv[e + 2] = q4.z; qv[e + 3] = q4.w;
            qi[e] = i4.x; qi[e + 1] = i4.y; qi[e + 2] = i4.z; qi[e + 3] = i4.w;
          }
          // predicated stores down the target rows (skip = copies stored by the
          // producers, and padding): no per-output branch or 64-bit multiply
          uint32_t* o = a.out + (int64_t)tb * a.per_row + x;
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const uint32_t lo = c[0][e] + (c[1][e] << 8), hi = c[2][e] + (c[3][e] << 8);
            const uint64_t f = (uint64_t)lo + ((uint64_t)hi << 16);
            const uint32_t m = (uint32_t)f * qi[e];
            const uint32_t w = (uint32_t)((f + (uint64_t)m * qv[e]) >> 32);
            st_global_if(o, w >= qv[e] ? w - qv[e] : w, ((skip >> e) & 1) == 0);
            o += a.per_row;
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
__global__ void __launch_bounds__(256)
    bconv_small_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                       const PrimeConst* __restrict__ pcs, const __grid_constant__ BconvArgs ba,
                       int64_t per_row) {
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4; i < per_row;
       i += (int64_t)gridDim.x * blockDim.x * 4) {
    uint32_t a[4][4], y[4][4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if (s >= ba.n_src) break;
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(in + (int64_t)s * per_row + i));
      a[s][0] = v.x; a[s][1] = v.y; a[s][2] = v.z; a[s][3] = v.w;
      const uint32_t q = pcs[ba.src_prime[s]].q;
#pragma unroll
      for (int e = 0; e < 4; ++e) y[s][e] = mul_shoup(a[s][e], ba.qhat_inv[s], ba.qhat_inv_shoup[s], q);
    }
    for (int t = 0; t < ba.n_dst; ++t) {
      uint32_t r[4];
      const int cp = ba.copy_from[t];
      if (cp >= 0) {
#pragma unroll
        for (int s = 0; s < 4; ++s)
          if (s == cp) {
#pragma unroll
            for (int e = 0; e < 4; ++e) r[e] = a[s][e];
          }
      } else {
        const PrimeConst pt = pcs[ba.dst_prime[t]];
        uint64_t acc[4] = {0, 0, 0, 0};
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          if (s >= ba.n_src) break;
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

}  // namespace

int launch_bconv(const Ctx& c, const uint32_t* in, uint32_t* out, const BconvArgs& ba, int batch,
                 cudaStream_t st) {
  if (ba.n_dst <= 0) return 0;
  if (ba.n_src < 1 || ba.n_src > 4 * kMaxKC * 2 || ba.n_dst > kMaxBconvDst) {
    set_error("base conversion: 1..16 sources and at most 128 targets");
    return 2;
  }
  if (ba.n_src <= 4 && ba.n_src * ba.n_dst <= 32 && (batch * (int64_t)c.n) % 4 == 0) {
    const int64_t per_row = (int64_t)batch * c.n;
    const int64_t blocks = std::min<int64_t>((per_row / 4 + 255) / 256, (int64_t)c.sms * 8);
    bconv_small_kernel<<<(int)std::max<int64_t>(blocks, 1), 256, 0, st>>>(in, out, c.d_pc, ba,
                                                                        per_row);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      set_error(std::string("bconv_small launch: ") + cudaGetErrorString(e));
      return 3;
    }
    return 0;
  }
  BconvTcArgs a;
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
  const int smem = 4 * kMaxChunks * kMaxKC * kBTileBC + kAStages * kMaxKC * kATileBC +
                   kRawBC * kRawTileBC + kMaxBconvDst * (4 + 4 + 4) + kMaxBconvDst / 16 * 4 +
                   (2 * kAStages + 8 + 2 * kRawBC) * 8 + 16;
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
