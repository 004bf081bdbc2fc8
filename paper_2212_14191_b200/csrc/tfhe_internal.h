// Internal (C++) view of the context and kernel launch interfaces.
// Not part of the C ABI (that is include/tfhe_b200.h).
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

namespace tfhe {

constexpr int kMaxLimbs = 512;  // rows one launch may address (kernel params <= 32 KB)

struct PrimeConst {
  uint32_t q;
  uint32_t n_inv;       // n^-1 mod q
  uint64_t mu;          // floor(2^64 / q)
  uint32_t n_inv_shoup;
  uint32_t r[3];        // 2^32, 2^40, 2^48 mod q (byte weights 4..6 of the TS kernel)
  uint32_t w3;          // 2^24 mod q
  uint32_t qneg_inv;    // -q^-1 mod 2^32 (Montgomery, R = 2^32)
  uint32_t pad[2];      // pad[0] = 1: small-n (ntt_tc.cu) twiddles carry 2^32 (fold4)
};

// Per-launch limb map: output row l uses prime `prime[l]`, reads input row
// `in_row[l]` and writes output row `out_row[l]` (rows index the leading
// axis of (rows, batch, n) buffers).
struct LimbMap {
  int n;
  int16_t prime[kMaxLimbs];
  int16_t in_row[kMaxLimbs];
  int16_t out_row[kMaxLimbs];
};

enum EpiMode : int {
  EPI_STORE = 0,       // out = NTT(in)
  EPI_SUB_SCALE = 1,   // out = (x - NTT(in)) * s  [+ base]   (ModDown, rescale)
  EPI_KS_MAC = 2,      // acc_b (+)= NTT(in) * kb[key_row], acc_a (+)= NTT(in) * ka[key_row]
                       // (key-switch inner product fused into ModUp, ckks.py:345-351);
                       // acc rows = out_row[l]; `first` overwrites instead of adding
  EPI_KS_ACC = 3,      // TS stage 2 over a group of S key-switch slices per target:
                       // acc (=|+=) sum_s NTT(P_s) * k_{j0+s}[key_row], accumulated on
                       // chip, one acc read/write per group (ckks.py:337-351)
};

struct EpiArgs {
  int mode;
  const uint32_t* x;      // (x_rows, batch, n): subtrahend source, row = x_row[l]
  const uint32_t* base;   // optional addend (base_rows, batch, n), row = base_row[l] (-1: none)
  int16_t x_row[kMaxLimbs];
  int16_t base_row[kMaxLimbs];
  uint32_t s[kMaxLimbs];        // per-limb scale
  uint32_t s_shoup[kMaxLimbs];
  // EPI_KS_MAC
  const uint32_t* kb;     // (key_rows, n) NTT-domain key rows, shared by the batch
  const uint32_t* ka;
  uint32_t* acc_b;        // (acc_rows, batch, n)
  uint32_t* acc_a;
  int16_t key_row[kMaxLimbs];
  int first;
  // EPI_KS_ACC
  const uint32_t* key;      // (dnum, 2, key_rows, n) switching key
  long long key_pair;       // elements per (b_j, a_j) pair
  int j0;                   // first slice of the group
  int16_t js[kMaxLimbs];    // slice that owns target row l (-1: none) -> skipped
  int16_t init_acc[kMaxLimbs];  // 1: start from acc, 0: start from zero
  int ks_lazy;                  // slice products summed in 64 bits between reductions
  // EPI_STORE of an inverse transform: != 0 applies the coefficient-domain
  // automorphism x -> x^t to the output (coefficient i lands at t i mod 2n,
  // negated past n; kernels.py:97-107) -- the hoisted HROTATE (p3 plan only)
  uint32_t scatter_t;
};

struct Ctx {
  int dev = 0;
  int log_n = 0, n = 0, n1 = 0, n2 = 0;
  int n_primes = 0;
  std::vector<uint32_t> primes, psis;
  // device tables
  PrimeConst* d_pc = nullptr;
  uint8_t* d_tw[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [inverse][stage]
  uint8_t* d_tw_ks = nullptr;   // forward stage 2, x 2^64 (key-switch MAC epilogue)
  size_t tw_stride[2] = {0, 0};                                   // bytes per prime, per stage
  int kpad[2] = {0, 0}, npad[2] = {0, 0}, bn[2] = {0, 0};
  uint32_t* d_w2[2] = {nullptr, nullptr};   // [inverse] (prime, n1*n2) hadamard twiddles
  uint32_t* d_w2s[2] = {nullptr, nullptr};  // Shoup companions
  // twiddle-resident (TS) kernel: per [inverse][stage] words
  // [prime][half][row 128][plane 4][K/4], used when n1 >= 128
  uint32_t* d_twa[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  // stage-1 hadamard twiddles (W2 * 2^96, transposed) for the TS epilogue
  uint32_t* d_w2r[2] = {nullptr, nullptr};
  uint32_t* d_w2rs[2] = {nullptr, nullptr};
  // forward stage-2 twiddle planes scaled by 2^96 (not 2^64): the stage-2 result
  // is then y*2^32, the Montgomery form the fused key-switch MAC multiplies with
  uint32_t* d_twa_ks = nullptr;
  bool use_ts = false;
  // N = 2^13 (n1 = 64, n2 = 128): stage 1 on the resident small-n kernel,
  // writing P in the TS blocked layout, stage 2 on the TS kernel (K = 128),
  // whose twiddles live in TMEM -- the resident kernel cannot hold K = 128
  bool ts_stage2 = false;
  // fused single-launch n = 4096 transform (ntt_fused.cu): per [inverse]
  // twisted 64-point DFT byte-plane tiles and the matching Hadamard W2' R
  // (+ the key-switch MAC variant W2' R^2)
  uint8_t* d_fdft[2] = {nullptr, nullptr};
  uint32_t* d_fw2[2] = {nullptr, nullptr};
  uint32_t* d_fw2_ks = nullptr;
  // three-factor n = 2^16 transform (ntt_p3.cu), per [inverse]: column-pass
  // 32-point tiles, inner / outer Hadamard tables, row-pass 64-point tiles
  // (+ the key-switch MAC variant of the forward row tiles)
  bool use_p3 = false;
  uint8_t* d_p3t1[2] = {nullptr, nullptr};
  uint32_t* d_p3hin[2] = {nullptr, nullptr};
  uint32_t* d_p3hout[2] = {nullptr, nullptr};
  uint8_t* d_p3t2[2] = {nullptr, nullptr};
  uint8_t* d_p3t2ks = nullptr;
  int sms = 148;
  std::vector<PrimeConst> h_pc;
};

// twiddle-resident tensor-core stages (ntt_ts.cu)
int build_ts_tables(Ctx& c);
// Key-switch group: stage 1 over the S*T limbs of `s1map` (limb s*T + t =
// slice s, target t) into ws, then stage 2 over the T targets of `tmap`
// (prime, out_row = accumulator row) accumulating the S slices per target on
// chip into epi.acc_b / epi.acc_a (EPI_KS_ACC).  ws >= S*T*batch*n words.
int launch_ntt_ts_ks_group(const Ctx& c, const uint32_t* in, void* ws, const LimbMap& s1map,
                           const LimbMap& tmap, int S, int batch, const EpiArgs& epi,
                           cudaStream_t st);
int launch_ntt_ts_stage1(const Ctx& c, const uint32_t* in, uint32_t* P, const LimbMap& map,
                         int batch, int inverse, cudaStream_t st);
int launch_ntt_ts(const Ctx& c, const uint32_t* in, uint32_t* out, const LimbMap& map, int batch,
                  int inverse, const EpiArgs* epi, void* ws, cudaStream_t st);
// TS stage 2 alone over the blocked P workspace (see Ctx::ts_stage2)
int launch_ntt_ts_stage2(const Ctx& c, const uint32_t* P, uint32_t* out, const LimbMap& map,
                         int batch, int inverse, const EpiArgs* epi, cudaStream_t st);

// fused n = 4096 transform (ntt_fused.cu): tables (no-op for other shapes)
// and the launch; -1 = not applicable, run the two-stage kernels
int build_fused_tables(Ctx& c);
int launch_ntt_fused(const Ctx& c, const uint32_t* in, uint32_t* out, const LimbMap& map,
                     int batch, int inverse, const EpiArgs* epi, cudaStream_t st);

// three-factor n = 2^16 transform (ntt_p3.cu)
int build_p3_tables(Ctx& c);
int launch_ntt_p3(const Ctx& c, const uint32_t* in, uint32_t* out, const LimbMap& map, int batch,
                  int inverse, const EpiArgs* epi, void* ws, cudaStream_t st);
// key-switch group on the p3 plan (same contract as launch_ntt_ts_ks_group)
int launch_ntt_p3_ks_group(const Ctx& c, const uint32_t* in, void* ws, const LimbMap& s1map,
                           const LimbMap& tmap, int S, int batch, const EpiArgs& epi,
                           cudaStream_t st);

// kernels (ntt_tc.cu)
size_t ntt_workspace_bytes(const Ctx& c, int n_limbs, int batch);
int launch_ntt(const Ctx& c, const uint32_t* in, uint32_t* out, const LimbMap& map, int batch,
               int inverse, const EpiArgs* epi, void* ws, size_t ws_bytes, cudaStream_t st);
int build_ntt_tables(Ctx& c);

void set_error(const std::string& msg);
// per-kernel device timing (tfhe_profile_enable): events around a launch on
// its stream; no-ops unless enabled
void prof_begin(const char* name, cudaStream_t st);
void prof_end(cudaStream_t st);

}  // namespace tfhe
