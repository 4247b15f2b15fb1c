// lffn_gpu.cu -- the C-ABI of include/lffn_gpu.h: device context, table
// upload, and the stream-ordered launches of the hash (K1/K2) and gather (K3)
// kernels.  No CPU compute path exists: every forward runs on the device and
// a missing / failing CUDA runtime is reported as status 3.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <mutex>
#include <unordered_map>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "gather_kernels.cuh"
#include "hash_kernels.cuh"
#include "dense_tcgen05.cuh"
#include "hash_bh_kernel.cuh"
#include "backward_kernels.cuh"
#include "hash_sf_kernel.cuh"
#include "small_kernels.cuh"
#include "lffn_gpu.h"
#include "lffn_internal.h"
#include "neighbor_kernels.cuh"

namespace lffn_gpu {

namespace {
thread_local std::string g_last_error;
thread_local int g_last_class = 0;

// Status 1 splits into the reference's two validation exceptions
// (common.hpp:17-23): the shape / size checks it throws as SizeError
// (lookup.cpp:28-36, 176-181, 300; projection.cpp:31-40, 141, 170, 284-286;
// checkpoint.cpp:56-58) and everything else as UsageError (unknown names,
// checkpoint I/O, calls in the wrong state).
int classify(int status, const std::string& msg) {
  if (status == LFFN_ERR_NUMERIC) return LFFN_CLASS_NUMERIC;
  if (status != LFFN_ERR_USAGE) return LFFN_CLASS_RUNTIME;
  static const char* const kSize[] = {
      "lookup config: d_in", "lookup config: table count", "lookup config: code bits",
      "lookup config: neighbor count", "lookup config: tau-1", "lookup forward: input width",
      "lookup forward: projection must map", "lookup forward: table stack shape",
      "lookup forward: table slice", "projection: d_in and d_out", "bh projection:",
      "acdc projection:", "projection blob:", "projection forward: input has",
      "checkpoint save: projection spec inconsistent", "checkpoint save: table stack inconsistent",
      "neighbor_codes:", "lookup backward: grad_y shape", "projection backward: grad_out",
      "projection backward: grad_params", "lookup forward: the device path supports"};
  for (const char* pre : kSize)
    if (msg.compare(0, std::strlen(pre), pre) == 0) return LFFN_CLASS_SIZE;
  // our own row-count limits are size errors as well
  if (msg.find("exceed the context's max_tokens") != std::string::npos) return LFFN_CLASS_SIZE;
  return LFFN_CLASS_USAGE;
}
}  // namespace

int fail(int status, const std::string& msg) {
  g_last_error = msg;
  g_last_class = classify(status, msg);
  return status;
}

}  // namespace lffn_gpu

using namespace lffn_gpu;

namespace {
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and size:
// a host API call per launch is measurable at small batches
void set_smem(const void* fn, int bytes) {
  static std::mutex mu;
  static std::unordered_map<uint64_t, int> done;  // (kernel, device) -> bytes set
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t key = reinterpret_cast<uintptr_t>(fn) * 64u + uint64_t(dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  done[key] = bytes;
}
}  // namespace

#define LFFN_CUDA(call)                                                                   \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(LFFN_ERR_RUNTIME, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct lffn_ctx {
  int device = 0;
  int64_t max_tokens = 0;
  lffn_cfg cfg{};
  lffn_proj proj{};  // blob pointer cleared after the copy
  int64_t D = 1, logD = 0, code_width = 0, rows = 0, kb = 0, ke = 0, h_loc = 0;
  int64_t nc = 1;  // neighbor_count: records per (token, table)
  int n_transforms = 0;

  // projection parameters on the device
  uint32_t* d_signmask = nullptr;
  double* d_diag = nullptr;
  double* d_W = nullptr;
  double* d_bh = nullptr;   // bh: m x (D/b) x b x b blocks (float64)
  double* d_bhT = nullptr;  // bh backward: the same blocks, each transposed (built on first use)
  void* d_wp[3] = {nullptr, nullptr, nullptr};  // dense (tcgen05): W^T slice split planes
  double* d_wt64 = nullptr;  // dense: slice of W^T in float64 (exact near-zero fixups)
  int dense_ntile = 0;       // N tile of the tcgen05 dense GEMM (0: exact path only)
  int dense_exact = 0;       // 1: exact float64 dense projection
  alignas(64) DenseMaps dense_maps{};  // TMA maps of the split planes (dense)
  void* d_xp[3] = {nullptr, nullptr, nullptr};  // dense: per-call split of x (max_tokens x d_in)
  int dense_split = kSplitTf32;  // kSplitTf32 | kSplitBf16x3 (bf16 x3 when d_in % 8 == 0)
  uint2* d_fix_list = nullptr;  // dense tcgen05: deferred exact fixups
  float* d_xnorm = nullptr;     // dense tcgen05: ||x_t||_2 per token (fixup band)
  float* d_wnorm = nullptr;     // dense tcgen05: ||W[:, c]||_2 per slice column
  int* d_fix_count = nullptr;
  int fix_cap = 0;
  double* d_zbuf = nullptr;  // dense: [max_tokens x code_width] float64
  // backward scratch (allocated by the first lffn_backward / lffn_proj_backward)
  double* d_gzbuf = nullptr;       // [max_tokens x code_width] float64 grad_z
  uint32_t* d_bwd_offs = nullptr;  // [h_loc * rows + 1]
  uint32_t* d_bwd_hist = nullptr;  // [h_loc * kBwdBlocks * rows]
  uint32_t* d_bwd_rank = nullptr;  // [max_tokens * h_loc * nc]
  double* d_bwd_gdot = nullptr;    // [max_tokens * h_loc * nc] <grad_y, row> per record
  uint32_t* d_bwd_list = nullptr;  // [max_tokens * h_loc * nc]
  uint32_t* d_bwd_mask = nullptr;  // signflip: masks (0, s_2, s_1)
  double* d_bwd_rows = nullptr;    // acdc / bh: (2 + stage inputs) x [max_tokens x D]

  // tables
  const void* d_T = nullptr;
  void* d_T_owned = nullptr;
  int t_dtype = LFFN_F32;

  // workspace
  uint32_t* d_codes = nullptr;
  float* d_coeff = nullptr;
  int* d_flag = nullptr;
  int* h_flag = nullptr;  // pinned
  float* d_xbuf = nullptr;
  float* d_ybuf = nullptr;
  cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_comp2 = nullptr, s_d2h = nullptr;
  static constexpr int kChunks = 16;
  cudaEvent_t ev_h2d[kChunks] = {}, ev_comp[kChunks] = {};
  cudaEvent_t ev_t0 = nullptr, ev_t1 = nullptr, ev_t2 = nullptr;
  bool timing = false;
  bool timed = false;

  int64_t launches = 0;
  int num_sms = 148;
  size_t table_group_bytes = 0;  // >0: walk tables in groups of this many bytes (measured slower on c2)
  int64_t gather_variant = 0;    // LFFN_OPT_GATHER_VARIANT (0 = default choice)
  int bf16w = 1;                 // LFFN_OPT_BF16_COEFF_FMA: exact FHFMA path for bf16 tables
  int bwd_one_pass = 0;          // LFFN_OPT_BWD_ONE_PASS: single-pass KB1 (A/B reference)
  int hash_exact = 0;            // LFFN_OPT_HASH_EXACT: always K1 (z bit-identical)
  int host_chunks = 8;           // LFFN_OPT_HOST_CHUNKS: lffn_forward_host pipeline chunks
  bool host_direct = true;       // LFFN_OPT_HOST_DIRECT: small batches write y / the flag straight to pinned memory
  int64_t host_direct_max = 128; // ... and two-kernel batches up to this size (y written in place)
  int* h_flag_dev = nullptr;     // device address of h_flag
  bool hash_exact_bh_old = false;  // (A/B: the round-1 BH kernel)
  int gather_sms = 0;            // LFFN_OPT_GATHER_SMS: persistent gather grid over this many SMs (0 = all)
  unsigned long long* d_sfmask = nullptr;  // K1f: per-thread sign masks [3][D/64]
  int small_max = 64;                // LFFN_OPT_SMALL_MAX_TOKENS: K5 up to this batch size
  static constexpr int kSmallTokens = 64;
  // host path of small batches: one CUDA graph per batch size (H2D, K5, D2H,
  // flag read + reset), its two host pointers patched per call
  struct HostGraph {
    cudaGraphExec_t exec = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphNode_t h2d = nullptr, d2h = nullptr;
  };
  HostGraph host_graph[kSmallTokens + 1];
};

namespace {

int flag_message(int flag) {
  if (flag & kFlagInput) return fail(LFFN_ERR_NUMERIC, "non-finite values in projection forward input");
  if (flag & kFlagHash) return fail(LFFN_ERR_NUMERIC, "non-finite values in hash stage");
  if (flag & kFlagGather) return fail(LFFN_ERR_NUMERIC, "non-finite values in gather stage");
  if (flag & kFlagBwdInput) return fail(LFFN_ERR_NUMERIC, "non-finite values in lookup backward input");
  if (flag & kFlagBwdOutput) return fail(LFFN_ERR_NUMERIC, "non-finite values in projection backward output");
  if (flag & kFlagBwdTables) return fail(LFFN_ERR_NUMERIC, "non-finite values in lookup backward tables");
  return LFFN_OK;
}

class DeviceGuard {
 public:
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev_);
    if (prev_ != dev) cudaSetDevice(dev);
    dev_ = dev;
  }
  ~DeviceGuard() {
    if (prev_ != dev_) cudaSetDevice(prev_);
  }

 private:
  int prev_ = 0, dev_ = 0;
};

int ilog2(int64_t v) {
  int l = 0;
  while ((int64_t(1) << l) < v) ++l;
  return l;
}

void destroy_ctx(lffn_ctx* c) {
  if (!c) return;
  DeviceGuard g(c->device);
  cudaFree(c->d_signmask);
  cudaFree(c->d_diag);
  cudaFree(c->d_W);
  cudaFree(c->d_bh);
  cudaFree(c->d_bhT);
  for (int q = 0; q < 3; ++q) cudaFree(c->d_wp[q]);
  cudaFree(c->d_wt64);
  for (int q = 0; q < 3; ++q) cudaFree(c->d_xp[q]);
  cudaFree(c->d_fix_list);
  cudaFree(c->d_xnorm);
  cudaFree(c->d_wnorm);
  cudaFree(c->d_fix_count);
  cudaFree(c->d_sfmask);
  for (auto& hg : c->host_graph) {
    if (hg.exec) cudaGraphExecDestroy(hg.exec);
    if (hg.graph) cudaGraphDestroy(hg.graph);
  }
  cudaFree(c->d_zbuf);
  cudaFree(c->d_gzbuf);
  cudaFree(c->d_bwd_offs);
  cudaFree(c->d_bwd_hist);
  cudaFree(c->d_bwd_rank);
  cudaFree(c->d_bwd_gdot);
  cudaFree(c->d_bwd_list);
  cudaFree(c->d_bwd_mask);
  cudaFree(c->d_bwd_rows);
  cudaFree(c->d_T_owned);
  cudaFree(c->d_codes);
  cudaFree(c->d_coeff);
  cudaFree(c->d_flag);
  if (c->h_flag) cudaFreeHost(c->h_flag);
  cudaFree(c->d_xbuf);
  cudaFree(c->d_ybuf);
  if (c->s_h2d) cudaStreamDestroy(c->s_h2d);
  if (c->s_comp) cudaStreamDestroy(c->s_comp);
  if (c->s_comp2) cudaStreamDestroy(c->s_comp2);
  if (c->s_d2h) cudaStreamDestroy(c->s_d2h);
  for (int i = 0; i < lffn_ctx::kChunks; ++i) {
    if (c->ev_h2d[i]) cudaEventDestroy(c->ev_h2d[i]);
    if (c->ev_comp[i]) cudaEventDestroy(c->ev_comp[i]);
  }
  if (c->ev_t0) cudaEventDestroy(c->ev_t0);
  if (c->ev_t1) cudaEventDestroy(c->ev_t1);
  if (c->ev_t2) cudaEventDestroy(c->ev_t2);
  delete c;
}

// 2-D fp32 TMA map (inner dimension contiguous), SWIZZLE_128B boxes of
// box_inner x box_outer, zero fill out of bounds.
// tau values whose lcm(tau, 16) <= 128 (the tcgen05 path's N tile holds whole tables)
template <int TAU>
void launch_dense_tau(int split, dim3 grid, size_t smem, cudaStream_t st, const DenseMaps& m,
                      const DenseParams& p) {
  static bool attr = [&] {
    cudaFuncSetAttribute(dense_tcgen05_kernel<TAU, kSplitTf32>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(dense_smem_bytes(128, kSplitTf32)));
    cudaFuncSetAttribute(dense_tcgen05_kernel<TAU, kSplitBf16x3>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(dense_smem_bytes(128, kSplitBf16x3)));
    return true;
  }();
  (void)attr;
  if (split == kSplitBf16x3) dense_tcgen05_kernel<TAU, kSplitBf16x3><<<grid, 128, smem, st>>>(m, p);
  else dense_tcgen05_kernel<TAU, kSplitTf32><<<grid, 128, smem, st>>>(m, p);
}

int launch_dense_tcgen05(int tau, int split, dim3 grid, size_t smem, cudaStream_t st,
                         const DenseMaps& m, const DenseParams& p) {
  switch (tau) {
#define LFFN_TAU(T) \
  case T:           \
    launch_dense_tau<T>(split, grid, smem, st, m, p); \
    return LFFN_OK;
    LFFN_TAU(1) LFFN_TAU(2) LFFN_TAU(3) LFFN_TAU(4) LFFN_TAU(5) LFFN_TAU(6) LFFN_TAU(7)
    LFFN_TAU(8) LFFN_TAU(10) LFFN_TAU(12) LFFN_TAU(14) LFFN_TAU(16) LFFN_TAU(20) LFFN_TAU(24)
#undef LFFN_TAU
    default:
      return fail(LFFN_ERR_USAGE, "dense tcgen05: unsupported code_bits " + std::to_string(tau));
  }
}

int make_tma_map(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                 uint32_t box_inner, uint32_t box_outer, bool bf16 = false, bool swizzle = true) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!encode) return fail(LFFN_ERR_RUNTIME, "cuTensorMapEncodeTiled unavailable");
  const size_t eb = bf16 ? 2 : 4;
  const cuuint64_t dims[2] = {inner, std::max<uint64_t>(outer, 1)};
  const cuuint64_t strides[1] = {inner * eb};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                            2, const_cast<void*>(base), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE,
                            !swizzle               ? CU_TENSOR_MAP_SWIZZLE_NONE
                            : box_inner * eb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                            : box_inner * eb == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                   : CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(LFFN_ERR_RUNTIME, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return LFFN_OK;
}

int check_n(const lffn_ctx* c, int64_t n) {
  if (n < 0) return fail(LFFN_ERR_USAGE, "lookup forward: negative row count");
  if (n > c->max_tokens)
    return fail(LFFN_ERR_USAGE, "lookup forward: " + std::to_string(n) +
                                    " rows exceed the context's max_tokens " +
                                    std::to_string(c->max_tokens));
  return LFFN_OK;
}

// ---------------------------------------------------------------- launches

int launch_hash_top1(lffn_ctx* c, const float* d_x, int64_t n, uint32_t* codes, float* coeff,
                     double* z_out, cudaStream_t st, bool exact_z);

// Hash stage.  nc == 1: codes / coefficients of the top-1 code.  nc > 1: the
// projection writes z (float64, exact: the dense kind takes the float64
// kernel so neighbour ORDER follows the reference's |z|), then one thread per
// (token, table) enumerates the nc neighbour codes and their coefficients
// (neighbor_kernels.cuh); codes / coeff are [n][h_loc][nc].
int launch_hash(lffn_ctx* c, const float* d_x, int64_t n, uint32_t* codes, float* coeff,
                double* z_out, cudaStream_t st) {
  if (c->nc == 1) return launch_hash_top1(c, d_x, n, codes, coeff, z_out, st, false);
  if (n == 0) return LFFN_OK;
  double* z = z_out ? z_out : c->d_zbuf;
  // the top-1 outputs of the projection kernel land in the first n*h_loc
  // records and are overwritten below
  if (int rc = launch_hash_top1(c, d_x, n, codes, coeff, z, st, true)) return rc;
  if (c->h_loc == 0) return LFFN_OK;
  NeighborParams q{};
  q.z = z;
  q.n = n;
  q.code_width = int(c->code_width);
  q.tau = int(c->cfg.code_bits);
  q.kb = int(c->kb);
  q.ke = int(c->ke);
  q.nc = int(c->nc);
  q.scaled = (c->cfg.variant == LFFN_SCALED || c->cfg.variant == LFFN_GELU_TAU1) ? 1 : 0;
  q.codes = codes;
  q.coeff = coeff;
  q.flag = c->d_flag;
  const unsigned grid = unsigned((n * c->h_loc + 127) / 128);
  if (c->nc <= 4) neighbor_kernel<4><<<grid, 128, 0, st>>>(q);
  else if (c->nc <= 16) neighbor_kernel<16><<<grid, 128, 0, st>>>(q);
  else if (c->nc <= 64) neighbor_kernel<64><<<grid, 128, 0, st>>>(q);
  else neighbor_kernel<256><<<grid, 128, 0, st>>>(q);
  ++c->launches;
  LFFN_CUDA(cudaGetLastError());
  return LFFN_OK;
}

void fill_hash_params(const lffn_ctx* c, HashParams& p, const float* d_x, int64_t n) {
  p.x = d_x;
  p.n = n;
  p.d_in = int(c->cfg.d_in);
  p.D = int(c->D);
  p.logD = int(c->logD);
  p.code_width = int(c->code_width);
  p.tau = int(c->cfg.code_bits);
  p.kb = int(c->kb);
  p.ke = int(c->ke);
  p.scaled = (c->cfg.variant == LFFN_SCALED || c->cfg.variant == LFFN_GELU_TAU1) ? 1 : 0;
  p.n_transforms = c->n_transforms;
  p.signmask = c->d_signmask;
  p.diag = c->d_diag;
  p.flag = c->d_flag;
}

int launch_hash_top1(lffn_ctx* c, const float* d_x, int64_t n, uint32_t* codes, float* coeff,
                     double* z_out, cudaStream_t st, bool exact_z) {
  if (n == 0) return LFFN_OK;
  HashParams p{};
  p.x = d_x;
  p.n = n;
  p.d_in = int(c->cfg.d_in);
  p.D = int(c->D);
  p.logD = int(c->logD);
  p.code_width = int(c->code_width);
  p.tau = int(c->cfg.code_bits);
  p.kb = int(c->kb);
  p.ke = int(c->ke);
  p.scaled = (c->cfg.variant == LFFN_SCALED || c->cfg.variant == LFFN_GELU_TAU1) ? 1 : 0;
  p.n_transforms = c->n_transforms;
  p.signmask = c->d_signmask;
  p.diag = c->d_diag;
  p.z_out = z_out;
  p.codes = codes;
  p.coeff = coeff;
  p.flag = c->d_flag;
  if (c->proj.kind == LFFN_PROJ_BH) {
    // BH{m}: fused block-diagonal + Hadamard stages (hash_bh_kernel.cuh)
    const int loge5 = c->logD >= 5 ? 5 : int(c->logD);
    const int E5 = 1 << loge5;
    BhParams bh{};
    bh.blocks = c->d_bh;
    bh.b = int(c->proj.block == 0 ? c->D : c->proj.block);
    bh.logb = ilog2(bh.b);
    bh.stages = int(c->proj.stages);
    if (c->D == 2048 && bh.b == 64 && !c->hash_exact_bh_old) {
      // the paper's shape: 8-column x 8-token register tiles, B rows three
      // ahead in registers (hash_bh64_kernel); exact unless no z is requested
      const size_t smem64 = size_t(8) * size_t(padded_len(2048)) * sizeof(double) + size_t(4) * 4 * 256 * 16 +
                            size_t(8) * 128 * sizeof(uint32_t);  // tokens, B ring, sign / small words
      const unsigned grid64 = (unsigned)((n + 7) / 8);
      p.tokens_per_block = 8;
      p.threads_per_token = 64;
      const bool fused = !z_out && !exact_z && !c->hash_exact;
      if (fused) {
        set_smem(reinterpret_cast<const void*>(hash_bh64_kernel<true>), int(smem64));
        hash_bh64_kernel<true><<<grid64, 256, smem64, st>>>(p, bh);
      } else {
        set_smem(reinterpret_cast<const void*>(hash_bh64_kernel<false>), int(smem64));
        hash_bh64_kernel<false><<<grid64, 256, smem64, st>>>(p, bh);
      }
      ++c->launches;
      LFFN_CUDA(cudaGetLastError());
      return LFFN_OK;
    }
    p.tokens_per_block = int(16384 / c->D);
    p.threads_per_token = int(c->D / E5);
    const size_t smem = size_t(p.tokens_per_block) * size_t(padded_len(int(c->D))) * sizeof(double);
    const unsigned grid = (unsigned)((n + p.tokens_per_block - 1) / p.tokens_per_block);
    auto gob = [&](auto kernel) {
      set_smem(reinterpret_cast<const void*>(kernel), int(smem));
      kernel<<<grid, 512, smem, st>>>(p, bh);
    };
    switch (loge5) {
      case 0: gob(hash_bh_kernel<0, 1>); break;
      case 1: gob(hash_bh_kernel<1, 1>); break;
      case 2: gob(hash_bh_kernel<2, 1>); break;
      case 3: gob(hash_bh_kernel<3, 1>); break;
      case 4: gob(hash_bh_kernel<4, 1>); break;
      default:
        // column quads per thread: D / 2048 for D >= 2048
        if (c->D <= 2048) gob(hash_bh_kernel<5, 1>);
        else if (c->D == 4096) gob(hash_bh_kernel<5, 2>);
        else if (c->D == 8192) gob(hash_bh_kernel<5, 4>);
        else gob(hash_bh_kernel<5, 8>);
        break;
    }
    ++c->launches;
    LFFN_CUDA(cudaGetLastError());
    return LFFN_OK;
  }
  if (c->proj.kind == LFFN_PROJ_DENSE && !c->dense_exact && !exact_z && c->dense_ntile > 0) {
    // tcgen05 split-precision GEMM fused with codes / coefficients (dense_tcgen05.cuh)
    DenseParams d{};
    d.x = d_x;
    d.wt64 = c->d_wt64;
    d.n = n;
    d.d_in = int(c->cfg.d_in);
    d.col_begin = int(c->kb * c->cfg.code_bits);
    d.ncols = int(c->h_loc * c->cfg.code_bits);
    d.ntile = c->dense_ntile;
    d.tau = int(c->cfg.code_bits);
    d.scaled = p.scaled;
    d.z_out = z_out;
    d.code_width = int(c->code_width);
    d.codes = codes;
    d.coeff = coeff;
    d.flag = c->d_flag;
    d.fix_scale = dense_fix_scale(d.d_in);
    d.xnorm = c->d_xnorm;
    d.wnorm = c->d_wnorm;
    d.fix_list = c->d_fix_list;
    d.fix_count = c->d_fix_count;
    d.fix_cap = c->fix_cap;
    // split x into tf32 hi / lo (ctx scratch; the TMA maps are built once)
    const unsigned gs = unsigned(std::min<int64_t>(int64_t(c->num_sms) * 8, (n * 32 + 255) / 256));
    const int din = int(c->cfg.d_in);
    if (c->dense_split != kSplitTf32)
      dense_split_x_bf16x3_kernel<<<gs, 256, 0, st>>>(
          d_x, n, din, static_cast<__nv_bfloat16*>(c->d_xp[0]), static_cast<__nv_bfloat16*>(c->d_xp[1]),
          static_cast<__nv_bfloat16*>(c->d_xp[2]), c->d_xnorm, c->d_flag, c->d_fix_count);
    else
      dense_split_x_kernel<<<gs, 256, 0, st>>>(d_x, n, din, static_cast<float*>(c->d_xp[0]),
                                               static_cast<float*>(c->d_xp[1]), c->d_xnorm, c->d_flag,
                                               c->d_fix_count);
    ++c->launches;
    const size_t smem = dense_smem_bytes(d.ntile, c->dense_split);

    dim3 grid((unsigned)((d.ncols + d.ntile - 1) / d.ntile), (unsigned)((n + umma::BM - 1) / umma::BM));
    const int rc = launch_dense_tcgen05(int(c->cfg.code_bits), c->dense_split, grid, smem, st,
                                        c->dense_maps, d);
    if (rc != LFFN_OK) return rc;
    ++c->launches;
    // fixups of the band, one warp per listed entry (the list length is on
    // the device: a grid-stride loop); exact serial sums when z is returned
    if (z_out) {
      // d_in <= 6144 keeps the per-warp product rows in 192 KB
      const size_t fsm = size_t(kFixupWarps) * size_t(d.d_in) * sizeof(double);
      set_smem(reinterpret_cast<const void*>(dense_fixup_kernel<true>), int(fsm));
      dense_fixup_kernel<true><<<unsigned(c->num_sms * 8), 32 * kFixupWarps, fsm, st>>>(d);
    } else {
      dense_fixup_kernel<false><<<unsigned(c->num_sms * 8), 32 * kFixupWarps, 0, st>>>(d);
    }
    ++c->launches;
    LFFN_CUDA(cudaGetLastError());
    return LFFN_OK;
  }
  if (c->proj.kind == LFFN_PROJ_DENSE) {
    dim3 grid((unsigned)((c->code_width + 63) / 64), (unsigned)((n + 63) / 64));
    dense_proj_f64_kernel<<<grid, 256, 0, st>>>(d_x, c->d_W, c->d_zbuf, n, int(c->cfg.d_in),
                                                int(c->code_width), c->d_flag);
    ++c->launches;
    p.z_in = c->d_zbuf;
  }
  const int kind = c->proj.kind == LFFN_PROJ_SIGNFLIP ? kPreSign
                   : c->proj.kind == LFFN_PROJ_ACDC   ? kPreDiag
                                                      : kPreNone;
  if (kind == kPreSign && c->d_sfmask && !z_out && !exact_z && !c->hash_exact && !p.scaled &&
      n > 16) {
    // K1f (hash_sf_kernel.cuh): the production signflip hash at D = 2048 /
    // 4096 -- three transposes per token, codes from warp ballots; z not
    // bit-identical (stage order), codes bit-exact wherever |z| > 1e-5
    HashSfParams q{};
    q.x = d_x;
    q.n = n;
    q.d_in = int(c->cfg.d_in);
    q.code_width = int(c->code_width);
    q.tau = int(c->cfg.code_bits);
    q.kb = int(c->kb);
    q.ke = int(c->ke);
    q.masks = c->d_sfmask;
    q.transforms = 3;
    q.codes = codes;
    q.coeff = coeff;
    q.flag = c->d_flag;
    auto gof = [&](auto kernel, int logd) {
      const int tpt = (1 << logd) / 64, tpb = sf_threads(logd) / tpt;
      const int slot = (1 << logd) + 2 * ((1 << logd) >> 6) + (1 << logd) / 32;
      const size_t smem = size_t(tpb) * size_t(slot) * sizeof(double);
      set_smem(reinterpret_cast<const void*>(kernel), int(smem));
      kernel<<<unsigned((n + tpb - 1) / tpb), sf_threads(logd), smem, st>>>(q);
    };
    // instantiated per class of live (non-padding) registers of the start layout
    const int live = sf_live_class(int(c->logD), q.d_in);
    if (c->logD == 11) {
      if (live == 16) gof(hash_sf_kernel<11, 16>, 11);
      else if (live == 24) gof(hash_sf_kernel<11, 24>, 11);
      else if (live == 32) gof(hash_sf_kernel<11, 32>, 11);
      else if (live == 48) gof(hash_sf_kernel<11, 48>, 11);
      else gof(hash_sf_kernel<11, 64>, 11);
    } else {
      if (live == 32) gof(hash_sf_kernel<12, 32>, 12);
      else gof(hash_sf_kernel<12, 64>, 12);
    }
    ++c->launches;
    LFFN_CUDA(cudaGetLastError());
    return LFFN_OK;
  }
  int loge = c->logD >= kMaxLogE ? kMaxLogE : int(c->logD);
  // a handful of tokens cannot fill the GPU: 16 coordinates per thread (4x
  // the threads per token) shortens each token's serial chain (c5, n = 1:
  // 14.9 -> 12.9 us)
  if (n <= 16 && loge == 6 && (c->D >> 4) <= 256) loge = 4;
  const int E = 1 << loge;
  const int tpt = int(c->D / E);  // <= 256 for D <= 16384
  // LOGE 6 (one warp per D <= 2048 token): 128-thread CTAs measured fastest
  // (c2 hash 0.233 ms vs 0.251 ms with 256-thread CTAs)
  const int nt = (loge == 6 && tpt <= 128) ? 128 : 256;
  const int block = std::max(tpt, (nt / tpt) * tpt);
  const int tpb = block / tpt;
  p.tokens_per_block = tpb;
  p.threads_per_token = tpt;
  const size_t smem = size_t(tpb) * size_t(padded_len(int(c->D))) * sizeof(double);
  const unsigned grid = (unsigned)((n + tpb - 1) / tpb);
  auto go = [&](auto kernel) {
    set_smem(reinterpret_cast<const void*>(kernel), int(smem));
    kernel<<<grid, block, smem, st>>>(p);
  };
  if (nt == 128 && kind == kPreSign) {
    // compile-time geometry for the BASELINE widths (D = 2048: c2, c3, c5;
    // D = 4096: c4) and the signflip transform count
    if (c->logD == 11 && c->n_transforms == 3) go(hash_structured_kernel<6, kPreSign, 128, 3, 11, 3>);
    else if (c->logD == 12 && c->n_transforms == 3) go(hash_structured_kernel<6, kPreSign, 128, 3, 12, 3>);
    else go(hash_structured_kernel<6, kPreSign, 128, 2>);
    ++c->launches;
    LFFN_CUDA(cudaGetLastError());
    return LFFN_OK;
  }
  if (nt == 128 && kind == kPreDiag && c->logD == 11 && c->n_transforms == 4) {
    // acdc depth 2 at D = 2048: the same compile-time geometry
    go(hash_structured_kernel<6, kPreDiag, 128, 3, 11, 4>);
    ++c->launches;
    LFFN_CUDA(cudaGetLastError());
    return LFFN_OK;
  }
#define LFFN_HASH_CASE(L)                                              \
  case L:                                                              \
    if (kind == kPreSign) go(hash_structured_kernel<L, kPreSign>);     \
    else if (kind == kPreDiag) go(hash_structured_kernel<L, kPreDiag>); \
    else go(hash_structured_kernel<L, kPreNone>);                      \
    break;
  switch (loge) {
    LFFN_HASH_CASE(0)
    LFFN_HASH_CASE(1)
    LFFN_HASH_CASE(2)
    LFFN_HASH_CASE(3)
    LFFN_HASH_CASE(4)
    LFFN_HASH_CASE(5)
    LFFN_HASH_CASE(6)
  }
#undef LFFN_HASH_CASE
  ++c->launches;
  LFFN_CUDA(cudaGetLastError());
  return LFFN_OK;
}

// One gather launch over tables [k0, k0 + nk) of the context's slice.
int launch_gather_group(lffn_ctx* c, const uint32_t* codes, const float* coeff, int64_t n,
                        float* y, int accumulate, int64_t k0, int64_t nk, cudaStream_t st) {
  GatherParams p{};
  const size_t esz = c->t_dtype == LFFN_F32 ? 4 : 2;
  p.T = static_cast<const char*>(c->d_T) + size_t(k0) * size_t(c->rows) * size_t(c->cfg.d_out) * esz;
  p.codes = codes + k0 * c->nc;
  p.coeff = coeff + k0 * c->nc;
  p.y = y;
  p.n = n;
  p.ld = int(c->h_loc * c->nc);
  p.nk = int(nk * c->nc);
  p.nc = int(c->nc);
  p.rows = int(c->rows);
  p.d_out = int(c->cfg.d_out);
  p.accumulate = accumulate;
  p.flag = c->d_flag;
  p.bf16w = c->bf16w;
  // odd rounds of resident tokens walk the tables backwards (the tables the
  // previous round finished with are still in L2): with the exact bf16-
  // coefficient FMA, measured +4% (c2 bf16) and +4% (c3) for bf16 tables
  // walked one warp per token, -6% for c4 (four warps per token,
  // part-major) and -2% for c2 fp32; set per launch below
  p.reverse_odd_rounds = c->t_dtype == LFFN_BF16 ? 1 : 0;
  const bool f32 = c->t_dtype == LFFN_F32;
  const int vec = f32 ? ((p.d_out % 4 == 0) ? 4 : 1) : ((p.d_out % 8 == 0) ? 8 : 1);
  if (vec > 1 && p.nc == 1) {
    // row-per-warp kernel: MAXC chunks of 32*vec columns per warp
    const int nchunks = (p.d_out + 32 * vec - 1) / (32 * vec);
    // chunks per warp: register budget of the persistent kernel (no spills)
    const int maxc = nchunks <= 2 ? 2 : (nchunks <= 4 || !f32) ? 4 : (nchunks <= 6 ? 6 : 4);
    const int wpt = (nchunks + maxc - 1) / maxc;
    const bool rec4 = (p.ld % 4 == 0) && (p.nk % 4 == 0) &&
                      (reinterpret_cast<uintptr_t>(p.codes) % 16 == 0) &&
                      (reinterpret_cast<uintptr_t>(p.coeff) % 16 == 0);
    const int64_t warps = n * wpt;
    const unsigned grid = (unsigned)((warps * 32 + 255) / 256);
    if (rec4) {
      // persistent row kernel: grid = 2 CTAs per SM; 4 tables' packed rows
      // in flight per lane (the f32 6-chunk case keeps 4 x 6 x 16 B)
      const unsigned pg = (unsigned)std::min<int64_t>(int64_t(c->num_sms) * 2, (warps * 32 + 255) / 256);
      // (MAXC 2 for bf16 -- 2x the column parts, half the bytes in flight per
      // warp -- measured slower: c3 1.39 vs 1.22 ms, c4 2.47 vs 2.07 ms)
      const int pmaxc = f32 ? maxc : (nchunks <= 2 ? 2 : nchunks <= 3 ? 3 : 4);
      const int pwpt = (nchunks + pmaxc - 1) / pmaxc;
      const int64_t pwarps = n * pwpt;
      if (pwpt > 1) p.reverse_odd_rounds = 0;
      const int gsms = c->gather_sms > 0 ? std::min(c->gather_sms, c->num_sms) : c->num_sms;
      const unsigned pgrid = (unsigned)std::min<int64_t>(int64_t(gsms) * 2, (pwarps * 32 + 255) / 256);
      (void)pg;
      // fewer (token, part) items than resident warp slots: split the table
      // walk over S warps per item (gather_split_kernel), S the largest of
      // 8/4/2 that keeps n*parts*S within the slots
      const int64_t slots = int64_t(c->num_sms) * 16;
      int S = 1;
      if (c->gather_variant == 0) {
        for (int s : {8, 4, 2})
          if (pwarps * s <= slots && p.nk % (4 * s) == 0) { S = s; break; }
      }
      if (S > 1) {
        const unsigned sgrid = (unsigned)((pwarps * S + 7) / 8);
#define LFFN_SPLIT(TT, M)                                                                   \
  if (S == 8) gather_split_kernel<TT, M, 4, 8><<<sgrid, 256, 0, st>>>(p, pwpt);             \
  else if (S == 4) gather_split_kernel<TT, M, 4, 4><<<sgrid, 256, 0, st>>>(p, pwpt);        \
  else gather_split_kernel<TT, M, 4, 2><<<sgrid, 256, 0, st>>>(p, pwpt);
        if (f32) {
          if (pmaxc == 2) { LFFN_SPLIT(float, 2) } else if (pmaxc == 4) { LFFN_SPLIT(float, 4) }
          else { LFFN_SPLIT(float, 6) }
        } else {
          if (pmaxc == 2) { LFFN_SPLIT(__nv_bfloat16, 2) } else if (pmaxc == 3) { LFFN_SPLIT(__nv_bfloat16, 3) }
          else { LFFN_SPLIT(__nv_bfloat16, 4) }
        }
#undef LFFN_SPLIT
        ++c->launches;
        LFFN_CUDA(cudaGetLastError());
        return LFFN_OK;
      }
      // (K3s, table tiles staged in shared memory for 1024 tokens x 32
      // columns -- tools/experiments/staged_gather.cuh -- measured slower:
      // c2 1.06-1.18 ms with cp.async and a CTA barrier per table, 0.759 ms
      // with TMA tiles and producer / consumer mbarriers, vs 0.641 ms)
      // (a narrow part-major walk -- one 16-byte chunk per lane, so a round
      // of resident warps touches 1/nchunks of every row and c3's 268 MB
      // stack fits L2 per part -- measured slower everywhere, with 8 tables
      // in flight at 3-4 CTAs per SM (c3 1.39 vs 1.08 ms, c4 2.59 vs 1.76)
      // and with 16 at 2 CTAs per SM (c3 1.46 vs 1.11, c4 2.72 vs 1.84,
      // c2 bf16 0.49 vs 0.36, c2 0.84 vs 0.64): four times the record loads
      // and address work per gathered byte)
      // (measured at c2 fp32: one warp per token with 6 chunks and 2 CTAs/SM
      // beats 2-3 warps per token at 3-4 CTAs/SM, 0.641 vs 0.698-0.942 ms;
      // L2 evict_last/evict_first splits of the table stack: 0.68-0.81 ms)
      // (c2 fp32 with 2 column parts of 3 chunks, part-major, 4 or 8 tables in
      // flight: 0.676 / 0.701 ms vs 0.641 ms one warp per token;
      // c3 with 2 column parts and 8 tables in flight per lane measured
      // 1.27 ms vs 1.22 ms; packed FFMA2 accumulation measured slower for
      // bf16 -- c4 2.31 vs 2.07 ms, c2 bf16 0.407 vs 0.393 ms)
      // several warps per token: part-major item order (gather_kernels.cuh)
#define LFFN_PROW(TT, M, TIF)                                                      \
  if (pwpt > 1) gather_row_persistent_kernel<TT, M, TIF, 2, true><<<pgrid, 256, 0, st>>>(p, pwpt); \
  else gather_row_persistent_kernel<TT, M, TIF, 2, false><<<pgrid, 256, 0, st>>>(p, pwpt);
      if (f32) {
        if (pmaxc == 2) { LFFN_PROW(float, 2, 4) } else if (pmaxc == 4) { LFFN_PROW(float, 4, 4) }
        else { LFFN_PROW(float, 6, 4) }
      } else {
        if (pmaxc == 2) { LFFN_PROW(__nv_bfloat16, 2, 4) } else if (pmaxc == 3) { LFFN_PROW(__nv_bfloat16, 3, 4) } else { LFFN_PROW(__nv_bfloat16, 4, 4) }
      }
#undef LFFN_PROW
      ++c->launches;
      LFFN_CUDA(cudaGetLastError());
      return LFFN_OK;
    }
#define LFFN_ROW(TT, V, M)                                                               \
  if (rec4) gather_row_kernel<TT, V, M, true><<<grid, 256, 0, st>>>(p, wpt);             \
  else gather_row_kernel<TT, V, M, false><<<grid, 256, 0, st>>>(p, wpt);
    if (f32) {
      if (maxc == 2) { LFFN_ROW(float, 4, 2) } else if (maxc == 4) { LFFN_ROW(float, 4, 4) }
      else { LFFN_ROW(float, 4, 6) }
    } else {
      if (maxc == 2) { LFFN_ROW(__nv_bfloat16, 8, 2) } else { LFFN_ROW(__nv_bfloat16, 8, 4) }
    }
#undef LFFN_ROW
    ++c->launches;
    LFFN_CUDA(cudaGetLastError());
    return LFFN_OK;
  }
  constexpr int NTOK = 4;
  const int64_t chunks = (p.d_out + 32 * vec - 1) / (32 * vec);
  const int64_t warps = ((n + NTOK - 1) / NTOK) * chunks;
  const unsigned grid = (unsigned)((warps * 32 + 255) / 256);
  if (f32 && vec == 4) gather_direct_kernel<float, 4, NTOK><<<grid, 256, 0, st>>>(p);
  else if (f32) gather_direct_kernel<float, 1, NTOK><<<grid, 256, 0, st>>>(p);
  else if (vec == 8) gather_direct_kernel<__nv_bfloat16, 8, NTOK><<<grid, 256, 0, st>>>(p);
  else gather_direct_kernel<__nv_bfloat16, 1, NTOK><<<grid, 256, 0, st>>>(p);
  ++c->launches;
  LFFN_CUDA(cudaGetLastError());
  return LFFN_OK;
}

// Tables larger than L2 are walked in groups of at most ~table_group_bytes
// (all tokens finish group g before group g+1 starts), so each table row is
// fetched from HBM about once per forward instead of once per wave of
// resident tokens; y is accumulated across groups (it stays L2-resident).
int launch_gather(lffn_ctx* c, const uint32_t* codes, const float* coeff, int64_t n, float* y,
                  int accumulate, cudaStream_t st) {
  if (n == 0) return LFFN_OK;
  if (!c->d_T) return fail(LFFN_ERR_USAGE, "lookup forward: tables not uploaded");
  if (c->h_loc == 0) {
    if (!accumulate)
      LFFN_CUDA(cudaMemsetAsync(y, 0, size_t(n) * size_t(c->cfg.d_out) * sizeof(float), st));
    return LFFN_OK;
  }
  const size_t esz = c->t_dtype == LFFN_F32 ? 4 : 2;
  const size_t table_bytes = size_t(c->rows) * size_t(c->cfg.d_out) * esz;
  // (a persisting-L2 access window over the first 16-96 MB of the stack
  // measured slower: c3 1.13-1.84 vs 1.11 ms; c2 and c2 bf16 within 2 %)
  int64_t per = c->h_loc;
  if (c->table_group_bytes > 0 && table_bytes * size_t(c->h_loc) > c->table_group_bytes) {
    per = std::max<int64_t>(1, int64_t(c->table_group_bytes / table_bytes));
    if (per >= 4) per &= ~int64_t(3);  // keep the 4-table record loads
    const int64_t groups = (c->h_loc + per - 1) / per;
    per = (c->h_loc + groups - 1) / groups;  // balance the groups
    if (per >= 4) per = (per + 3) & ~int64_t(3);
  }
  for (int64_t k0 = 0; k0 < c->h_loc; k0 += per) {
    const int64_t nk = std::min(per, c->h_loc - k0);
    if (int rc = launch_gather_group(c, codes, coeff, n, y, (k0 > 0) ? 1 : accumulate, k0, nk, st))
      return rc;
  }
  return LFFN_OK;
}

// K5 (small_kernels.cuh): the whole forward of a small batch in one launch,
// grid (token, table group); signflip at D = 2048, top-1, 16-byte rows.
bool small_eligible(const lffn_ctx* c, int64_t n) {
  if (n < 1 || n > std::min<int64_t>(c->small_max, lffn_ctx::kSmallTokens)) return false;
  if (c->proj.kind != LFFN_PROJ_SIGNFLIP || c->n_transforms != 3 || c->logD != 11 || c->nc != 1) return false;
  const int vec = c->t_dtype == LFFN_F32 ? 4 : 8;
  return c->h_loc > 0 && c->cfg.d_out % vec == 0 && c->cfg.d_out / vec <= 2 * kSmallThreads;
}

int launch_small(lffn_ctx* c, const float* d_x, int64_t n, float* d_y, int accumulate, cudaStream_t st) {
  SmallParams q{};
  q.x = d_x;
  q.n = n;
  q.d_in = int(c->cfg.d_in);
  q.code_width = int(c->code_width);
  q.tau = int(c->cfg.code_bits);
  q.kb = int(c->kb);
  q.ke = int(c->ke);
  q.scaled = (c->cfg.variant == LFFN_SCALED || c->cfg.variant == LFFN_GELU_TAU1) ? 1 : 0;
  // G CTAs per token (a cluster): about two CTAs per SM in total, a power of
  // two <= 16 (<= 8 above four tokens: clusters of 16 measured slower
  // there), and at most 256 tables per group.  More CTAs per token cut the
  // rows each CTA walks but repeat the hash: four CTAs per SM measured
  // slower at n = 32 / 64 (26.6 / 24.6 vs 15.3 / 18.4 us).
  const int gmax = n <= 4 ? kSmallMaxGroups : kSmallMaxGroups / 2;
  int G = 1;
  while (G < gmax && int64_t(2 * G) * n <= int64_t(c->num_sms) * 2) G *= 2;
  while (G < kSmallMaxGroups && (c->h_loc + G - 1) / G > kSmallMaxTpg) G *= 2;
  if ((c->h_loc + G - 1) / G > kSmallMaxTpg)
    return fail(LFFN_ERR_USAGE, "small forward: more than 4096 tables");
  q.tpg = int((c->h_loc + G - 1) / G);
  q.groups = G;
  q.signmask = c->d_signmask;
  q.T = c->d_T;
  q.rows = int(c->rows);
  q.d_out = int(c->cfg.d_out);
  q.y = d_y;
  q.accumulate = accumulate;
  q.flag = c->d_flag;
  const bool f32 = c->t_dtype == LFFN_F32;
  const int nch = int(c->cfg.d_out / (f32 ? 4 : 8));
  using SK = void (*)(SmallParams);
  SK fn = f32 ? (nch <= kSmallThreads ? &forward_small_kernel<float, 1> : &forward_small_kernel<float, 2>)
              : (nch <= kSmallThreads ? &forward_small_kernel<__nv_bfloat16, 1>
                                      : &forward_small_kernel<__nv_bfloat16, 2>);
  {
    // clusters of 16 are non-portable: allowed per kernel, per device
    static std::mutex mu;
    static bool done[64] = {};
    std::lock_guard<std::mutex> lock(mu);
    if (c->device < 64 && !done[c->device]) {
      for (SK k : {&forward_small_kernel<float, 1>, &forward_small_kernel<float, 2>,
                   &forward_small_kernel<__nv_bfloat16, 1>, &forward_small_kernel<__nv_bfloat16, 2>})
        cudaFuncSetAttribute(reinterpret_cast<const void*>(k), cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      done[c->device] = true;
    }
  }
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(unsigned(G), unsigned(n));
  lc.blockDim = dim3(kSmallThreads);
  lc.dynamicSmemBytes = 0;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = unsigned(G);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  LFFN_CUDA(cudaLaunchKernelEx(&lc, fn, q));
  ++c->launches;
  LFFN_CUDA(cudaGetLastError());
  return LFFN_OK;
}

int forward_impl(lffn_ctx* c, const float* d_x, int64_t n, float* d_y, cudaStream_t st) {
  const bool tm = c->timing;
  if (tm) LFFN_CUDA(cudaEventRecord(c->ev_t0, st));
  if (small_eligible(c, n)) {
    // one launch: reported as the gather stage
    if (tm) LFFN_CUDA(cudaEventRecord(c->ev_t1, st));
    if (int rc = launch_small(c, d_x, n, d_y, 0, st)) return rc;
    if (tm) {
      LFFN_CUDA(cudaEventRecord(c->ev_t2, st));
      c->timed = true;
    }
    return LFFN_OK;
  }
  if (int rc = launch_hash(c, d_x, n, c->d_codes, c->d_coeff, nullptr, st)) return rc;
  if (tm) LFFN_CUDA(cudaEventRecord(c->ev_t1, st));
  if (int rc = launch_gather(c, c->d_codes, c->d_coeff, n, d_y, 0, st)) return rc;
  if (tm) {
    LFFN_CUDA(cudaEventRecord(c->ev_t2, st));
    c->timed = true;
  }
  return LFFN_OK;
}

// Wait for everything queued on `st` and report the non-finite flag.  With
// the flag word mapped into the device's address space a one-thread kernel
// publishes (and resets) it in stream order and the host polls the word --
// no copy, no driver-side synchronisation latency (~10 us per call); a queue
// that does not drain within a few milliseconds falls back to the driver's
// synchronise.
int poll_flag(lffn_ctx* c, cudaStream_t st) {
  volatile int* hf = c->h_flag;
  for (int64_t spin = 0; *hf == -1; ++spin) {
    if (spin > (int64_t(1) << 22)) {
      LFFN_CUDA(cudaStreamSynchronize(st));
      if (*hf == -1) return fail(LFFN_ERR_RUNTIME, "flag not published");
    }
  }
  return flag_message(*hf);
}

int read_flag(lffn_ctx* c, cudaStream_t st) {
  if (c->host_direct && c->h_flag_dev) {
    *static_cast<volatile int*>(c->h_flag) = -1;
    flag_to_host_kernel<<<1, 1, 0, st>>>(c->d_flag, c->h_flag_dev);
    LFFN_CUDA(cudaGetLastError());
    return poll_flag(c, st);
  }
  LFFN_CUDA(cudaMemcpyAsync(c->h_flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  LFFN_CUDA(cudaMemsetAsync(c->d_flag, 0, sizeof(int), st));
  LFFN_CUDA(cudaStreamSynchronize(st));
  return flag_message(*c->h_flag);
}

uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return uint16_t((u >> 16) | 0x40);  // NaN stays NaN
  const uint32_t rounding = 0x7fffu + ((u >> 16) & 1u);
  return uint16_t((u + rounding) >> 16);
}

// double -> bf16 with a single round-to-nearest-even: round to float with
// round-to-odd first (truncate, then set the sticky LSB when inexact), which
// keeps the second rounding to bf16 exact.
uint16_t f64_to_bf16_rne(double d) {
  if (d != d) return 0x7fc0;
  float f = float(d);
  if (std::isinf(f)) return f32_to_bf16_rne(f);
  if (std::fabs(double(f)) > std::fabs(d)) f = std::nextafter(f, 0.0f);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if (double(f) != d) u |= 1u;
  std::memcpy(&f, &u, 4);
  return f32_to_bf16_rne(f);
}

float bf16_to_f32(uint16_t b) {
  uint32_t u = uint32_t(b) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

}  // namespace

namespace lffn_gpu {

// Converts host tables [k0, k0+nk) of the context's slice (host points at
// table k0) to store_dtype and copies them to the device; (re)allocates the
// device slice when needed.
int tables_upload_range(lffn_ctx* c, const void* host, int host_dtype, int store_dtype, int64_t k0,
                        int64_t nk) {
  if (store_dtype != LFFN_F32 && store_dtype != LFFN_BF16)
    return fail(LFFN_ERR_USAGE, "tables upload: store dtype must be f32 or bf16");
  if (host_dtype < LFFN_F32 || host_dtype > LFFN_F64)
    return fail(LFFN_ERR_USAGE, "tables upload: unknown host dtype");
  if (k0 < 0 || nk < 0 || k0 + nk > c->h_loc)
    return fail(LFFN_ERR_USAGE, "tables upload: table range outside the context's slice");
  DeviceGuard g(c->device);
  const size_t per_table = size_t(c->rows) * size_t(c->cfg.d_out);
  const size_t esz = store_dtype == LFFN_F32 ? 4 : 2;
  if (!c->d_T_owned || c->t_dtype != store_dtype || c->d_T != c->d_T_owned) {
    if (c->d_T_owned) cudaFree(c->d_T_owned);
    c->d_T_owned = nullptr;
    void* d = nullptr;
    LFFN_CUDA(cudaMalloc(&d, std::max<size_t>(per_table * size_t(c->h_loc) * esz, 16)));
    c->d_T_owned = d;
    c->d_T = d;
    c->t_dtype = store_dtype;
  }
  const size_t count = per_table * size_t(nk);
  std::vector<unsigned char> staging(count * esz);
  auto convert = [&](size_t b, size_t e) {
    for (size_t i = b; i < e; ++i) {
      if (store_dtype == LFFN_F32) {
        float f;
        if (host_dtype == LFFN_F64) f = float(static_cast<const double*>(host)[i]);
        else if (host_dtype == LFFN_F32) f = static_cast<const float*>(host)[i];
        else f = bf16_to_f32(static_cast<const uint16_t*>(host)[i]);
        std::memcpy(&staging[i * 4], &f, 4);
      } else {
        const uint16_t b16 = host_dtype == LFFN_BF16 ? static_cast<const uint16_t*>(host)[i]
                             : host_dtype == LFFN_F64
                                 ? f64_to_bf16_rne(static_cast<const double*>(host)[i])
                                 : f32_to_bf16_rne(static_cast<const float*>(host)[i]);
        std::memcpy(&staging[i * 2], &b16, 2);
      }
    }
  };
  // the conversion is the cost of an upload (c4: 537 M elements): host threads
  const unsigned nth = count < (size_t(1) << 20) ? 1u
                       : std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  if (nth == 1) {
    convert(0, count);
  } else {
    std::vector<std::thread> pool;
    for (unsigned q = 0; q < nth; ++q) pool.emplace_back(convert, count * q / nth, count * (q + 1) / nth);
    for (auto& th : pool) th.join();
  }
  LFFN_CUDA(cudaMemcpy(static_cast<char*>(c->d_T_owned) + size_t(k0) * per_table * esz,
                       staging.data(), staging.size(), cudaMemcpyHostToDevice));
  return LFFN_OK;
}

}  // namespace lffn_gpu

extern "C" {

const char* lffn_last_error(void) { return g_last_error.c_str(); }

int lffn_last_error_class(void) { return g_last_class; }

const char* lffn_version(void) { return "lffn_gpu 0.1 sm_100a"; }

int lffn_ctx_create_shard(lffn_ctx** out, int device, int64_t max_tokens, const lffn_cfg* cfg,
                          const lffn_proj* proj, int64_t table_begin, int64_t table_end) {
  if (!out) return fail(LFFN_ERR_USAGE, "ctx_create: null output");
  *out = nullptr;
  if (int rc = validate_cfg(cfg)) return rc;
  if (int rc = validate_proj(proj)) return rc;
  if (!proj->blob) return fail(LFFN_ERR_USAGE, "projection: blob required");
  // check_shapes (lookup.cpp:173-182)
  if (proj->d_in != cfg->d_in || proj->d_out != cfg->tables * cfg->code_bits)
    return fail(LFFN_ERR_USAGE, "lookup forward: projection must map d_in to h*tau");
  if (cfg->neighbor_count < 1 || cfg->neighbor_count > 256)
    return fail(LFFN_ERR_USAGE,
                "lookup forward: the device path supports neighbor_count 1 .. 256");
  if (max_tokens < 0) return fail(LFFN_ERR_USAGE, "ctx_create: negative max_tokens");
  if (table_end == 0 && table_begin == 0) table_end = cfg->tables;
  if (table_begin < 0 || table_end > cfg->tables || table_begin > table_end)
    return fail(LFFN_ERR_USAGE, "ctx_create: table range outside [0, h]");
  const int64_t D = transform_width(proj);
  if (D > 16384) return fail(LFFN_ERR_USAGE, "lookup forward: transform width above 16384 is not supported on the device");

  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(LFFN_ERR_RUNTIME, std::string("no CUDA device: ") + cudaGetErrorString(e));
  if (device < 0 || device >= ndev) return fail(LFFN_ERR_USAGE, "ctx_create: bad device ordinal");
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major < 10)
    return fail(LFFN_ERR_RUNTIME, "lffn_gpu is built for sm_100a (B200); device is sm_" +
                                      std::to_string(prop.major) + std::to_string(prop.minor));

  DeviceGuard g(device);
  lffn_ctx* c = new lffn_ctx();
  c->device = device;
  c->max_tokens = max_tokens;
  c->cfg = *cfg;
  c->proj = *proj;
  c->proj.blob = nullptr;
  c->D = D;
  c->logD = ilog2(D);
  c->code_width = cfg->tables * cfg->code_bits;
  c->rows = int64_t(1) << cfg->code_bits;
  c->kb = table_begin;
  c->ke = table_end;
  c->h_loc = table_end - table_begin;
  c->nc = cfg->neighbor_count;

  auto bail = [&](int rc) {
    destroy_ctx(c);
    return rc;
  };
#define CK(call)                                                                           \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return bail(fail(LFFN_ERR_RUNTIME, std::string(#call) + ": " + cudaGetErrorString(e_))); \
  } while (0)

  // projection parameters
  const double* blob = proj->blob;
  if (proj->kind == LFFN_PROJ_SIGNFLIP) {
    c->n_transforms = 3;
    const int64_t words = (D + 31) / 32;
    std::vector<uint32_t> mask(size_t(3 * words), 0u);
    for (int64_t s = 0; s < 3; ++s)
      for (int64_t j = 0; j < D; ++j) {
        const double v = blob[s * D + j];
        if (v != 1.0 && v != -1.0)
          return bail(fail(LFFN_ERR_USAGE, "signflip projection: sign vectors must hold +-1"));
        if (v == -1.0) mask[size_t(s * words + j / 32)] |= 1u << (j % 32);
      }
    CK(cudaMalloc(&c->d_signmask, mask.size() * sizeof(uint32_t)));
    CK(cudaMemcpy(c->d_signmask, mask.data(), mask.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    if (D == 2048 || D == 4096) {
      // K1f sign masks in its register layouts (hash_sf_kernel.cuh): thread
      // t, register r holds index sf_layout_index(log2 D, tr, t, r) at the
      // start of transform tr
      const int64_t tpt = D / 64;
      std::vector<unsigned long long> sf(size_t(3 * tpt), 0ull);
      for (int64_t tr = 0; tr < 3; ++tr)
        for (int64_t t = 0; t < tpt; ++t)
          for (int64_t r = 0; r < 64; ++r) {
            const int64_t j = sf_layout_index(D == 2048 ? 11 : 12, int(tr), int(t), int(r));
            if (blob[tr * D + j] == -1.0) sf[size_t(tr * tpt + t)] |= 1ull << r;
          }
      CK(cudaMalloc(&c->d_sfmask, sf.size() * sizeof(unsigned long long)));
      CK(cudaMemcpy(c->d_sfmask, sf.data(), sf.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice));
    }
  } else if (proj->kind == LFFN_PROJ_ACDC) {
    c->n_transforms = int(2 * proj->depth);
    CK(cudaMalloc(&c->d_diag, size_t(2 * proj->depth * D) * sizeof(double)));
    CK(cudaMemcpy(c->d_diag, blob, size_t(2 * proj->depth * D) * sizeof(double), cudaMemcpyHostToDevice));
  } else if (proj->kind == LFFN_PROJ_BH) {
    c->n_transforms = int(proj->stages);
    const size_t nb = size_t(blob_size(proj));
    CK(cudaMalloc(&c->d_bh, nb * sizeof(double)));
    CK(cudaMemcpy(c->d_bh, blob, nb * sizeof(double), cudaMemcpyHostToDevice));
  } else if (proj->kind == LFFN_PROJ_DENSE) {
    c->n_transforms = 0;
    const size_t nw = size_t(proj->d_in * proj->d_out);
    CK(cudaMalloc(&c->d_W, nw * sizeof(double)));
    CK(cudaMemcpy(c->d_W, blob, nw * sizeof(double), cudaMemcpyHostToDevice));
    CK(cudaMalloc(&c->d_zbuf, size_t(std::max<int64_t>(max_tokens, 1)) * c->code_width * sizeof(double)));
    // tcgen05 path: N tile = largest multiple of lcm(tau, 16) <= 256
    int64_t l = 16;
    while (l % cfg->code_bits != 0) l += 16;
    const int64_t ncols = c->h_loc * cfg->code_bits;
    if (l <= 128 && ncols > 0 && proj->d_in % 4 == 0 && proj->d_in <= 6144) {
      // N <= 128 so the kSegs K-segment accumulators fit kTmemCols (two CTAs per SM)
      c->dense_ntile = int((128 / l) * l);
      // operand split: bf16 x3 when the bf16 TMA rows allow it (d_in % 8 == 0;
      // 25% fewer operand bytes, c2 dense hash 0.312 vs 0.336 ms), else tf32
      // hi / lo (LFFN_DENSE_SPLIT=tf32 forces it)
      c->dense_split = proj->d_in % 8 == 0 ? kSplitBf16x3 : kSplitTf32;
      const bool bf = c->dense_split != kSplitTf32;
      const int P = bf ? 3 : 2;
      const size_t eb = bf ? 2 : 4;
      const uint32_t box = uint32_t(64 / eb);
      const size_t nw = size_t(ncols) * size_t(proj->d_in);
      for (int q = 0; q < P; ++q) CK(cudaMalloc(&c->d_wp[q], nw * eb));
      CK(cudaMalloc(&c->d_wt64, nw * sizeof(double)));
      if (bf)
        dense_split_weights_bf16x3_kernel<<<unsigned((nw + 255) / 256), 256>>>(
            c->d_W, int(proj->d_in), int(c->code_width), int(c->kb * cfg->code_bits), int(ncols),
            static_cast<__nv_bfloat16*>(c->d_wp[0]), static_cast<__nv_bfloat16*>(c->d_wp[1]),
            static_cast<__nv_bfloat16*>(c->d_wp[2]), c->d_wt64);
      else
        dense_split_weights_kernel<<<unsigned((nw + 255) / 256), 256>>>(
            c->d_W, int(proj->d_in), int(c->code_width), int(c->kb * cfg->code_bits), int(ncols),
            static_cast<float*>(c->d_wp[0]), static_cast<float*>(c->d_wp[1]), c->d_wt64);
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
      for (int q = 0; q < P && c->dense_ntile > 0; ++q)
        if (make_tma_map(&c->dense_maps.w[q], c->d_wp[q], uint64_t(proj->d_in), uint64_t(ncols), box,
                         uint32_t(c->dense_ntile), bf))
          c->dense_ntile = 0;  // no TMA encoder: exact float64 path
      if (c->dense_ntile > 0) {
        const size_t nx = size_t(std::max<int64_t>(max_tokens, 1)) * size_t(proj->d_in);
        for (int q = 0; q < P; ++q) CK(cudaMalloc(&c->d_xp[q], nx * eb));
        // the fixup band holds ~1e-3 of the z for Gaussian-like projections
        // (c2: ~1.5 per token); 4M entries (32 MB) before the kernel falls
        // back to inline recomputation
        c->fix_cap = 1 << 22;
        CK(cudaMalloc(&c->d_xnorm, nx / size_t(proj->d_in) * sizeof(float)));
        {
          std::vector<float> wn(static_cast<size_t>(ncols));
          for (int64_t col = 0; col < ncols; ++col) {
            double ss = 0.0;
            for (int64_t k = 0; k < proj->d_in; ++k) {
              const double wv = blob[size_t(k * c->code_width + c->kb * cfg->code_bits + col)];
              ss += wv * wv;
            }
            wn[size_t(col)] = float(std::sqrt(ss) * (1.0 + 1e-12));
            if (double(wn[size_t(col)]) < std::sqrt(ss)) wn[size_t(col)] = std::nextafter(wn[size_t(col)], 1e30f);
          }
          CK(cudaMalloc(&c->d_wnorm, wn.size() * sizeof(float)));
          CK(cudaMemcpy(c->d_wnorm, wn.data(), wn.size() * sizeof(float), cudaMemcpyHostToDevice));
        }
        CK(cudaMalloc(&c->d_fix_list, size_t(c->fix_cap) * sizeof(uint2)));
        CK(cudaMalloc(&c->d_fix_count, sizeof(int)));
        CK(cudaMemset(c->d_fix_count, 0, sizeof(int)));
        for (int q = 0; q < P && c->dense_ntile > 0; ++q)
          if (make_tma_map(&c->dense_maps.x[q], c->d_xp[q], uint64_t(proj->d_in),
                           uint64_t(std::max<int64_t>(max_tokens, 1)), box, umma::BM, bf))
            c->dense_ntile = 0;
      }
    }
  }

  const size_t mt = size_t(std::max<int64_t>(max_tokens, 1));
  CK(cudaMalloc(&c->d_codes, mt * size_t(std::max<int64_t>(c->h_loc * c->nc, 1)) * sizeof(uint32_t)));
  CK(cudaMalloc(&c->d_coeff, mt * size_t(std::max<int64_t>(c->h_loc * c->nc, 1)) * sizeof(float)));
  if (c->nc > 1 && !c->d_zbuf)  // float64 z for the neighbour enumeration
    CK(cudaMalloc(&c->d_zbuf, mt * size_t(c->code_width) * sizeof(double)));
  CK(cudaMalloc(&c->d_flag, sizeof(int)));
  CK(cudaMemset(c->d_flag, 0, sizeof(int)));
  // lffn_forward_host staging (no allocation on any forward path)
  CK(cudaMalloc(&c->d_xbuf, mt * size_t(cfg->d_in) * sizeof(float)));
  CK(cudaMalloc(&c->d_ybuf, mt * size_t(cfg->d_out) * sizeof(float)));
  CK(cudaMallocHost(&c->h_flag, sizeof(int)));
  {
    void* hfd = nullptr;
    if (cudaHostGetDevicePointer(&hfd, c->h_flag, 0) == cudaSuccess) c->h_flag_dev = static_cast<int*>(hfd);
    else cudaGetLastError();
  }
  CK(cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&c->s_comp, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&c->s_comp2, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking));
  for (int i = 0; i < lffn_ctx::kChunks; ++i) {
    CK(cudaEventCreateWithFlags(&c->ev_h2d[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_comp[i], cudaEventDisableTiming));
  }
  CK(cudaEventCreate(&c->ev_t0));
  CK(cudaEventCreate(&c->ev_t1));
  CK(cudaEventCreate(&c->ev_t2));
  c->num_sms = prop.multiProcessorCount;
#undef CK
  *out = c;
  return LFFN_OK;
}

int lffn_ctx_create(lffn_ctx** out, int device, int64_t max_tokens, const lffn_cfg* cfg,
                    const lffn_proj* proj) {
  return lffn_ctx_create_shard(out, device, max_tokens, cfg, proj, 0, cfg ? cfg->tables : 0);
}

int lffn_ctx_destroy(lffn_ctx* ctx) {
  destroy_ctx(ctx);
  return LFFN_OK;
}

int lffn_ctx_table_range(const lffn_ctx* ctx, int64_t* begin, int64_t* end) {
  if (!ctx) return fail(LFFN_ERR_USAGE, "null context");
  if (begin) *begin = ctx->kb;
  if (end) *end = ctx->ke;
  return LFFN_OK;
}

int64_t lffn_ctx_launch_count(const lffn_ctx* ctx) { return ctx ? ctx->launches : -1; }

int lffn_tables_upload(lffn_ctx* c, const void* host_T, int host_dtype, int store_dtype) {
  if (!c || !host_T) return fail(LFFN_ERR_USAGE, "tables upload: null argument");
  const size_t per_table = size_t(c->rows) * size_t(c->cfg.d_out);
  const size_t hsz = host_dtype == LFFN_F64 ? 8 : host_dtype == LFFN_F32 ? 4 : 2;
  const char* first = static_cast<const char*>(host_T) + size_t(c->kb) * per_table * hsz;
  // bounded staging: convert and copy ~64 MB of host tables at a time
  const int64_t chunk = std::max<int64_t>(1, int64_t((size_t(64) << 20) / (per_table * hsz)));
  for (int64_t k0 = 0; k0 < c->h_loc; k0 += chunk) {
    const int64_t nk = std::min(chunk, c->h_loc - k0);
    if (int rc = tables_upload_range(c, first + size_t(k0) * per_table * hsz, host_dtype,
                                     store_dtype, k0, nk))
      return rc;
  }
  return LFFN_OK;
}

int lffn_tables_upload_slice(lffn_ctx* c, const void* host_slice, int host_dtype, int store_dtype) {
  if (!c || !host_slice) return fail(LFFN_ERR_USAGE, "tables upload: null argument");
  const size_t per_table = size_t(c->rows) * size_t(c->cfg.d_out);
  const size_t hsz = host_dtype == LFFN_F64 ? 8 : host_dtype == LFFN_F32 ? 4 : 2;
  const int64_t chunk = std::max<int64_t>(1, int64_t((size_t(64) << 20) / (per_table * hsz)));
  for (int64_t k0 = 0; k0 < c->h_loc; k0 += chunk) {
    const int64_t nk = std::min(chunk, c->h_loc - k0);
    if (int rc = tables_upload_range(c, static_cast<const char*>(host_slice) + size_t(k0) * per_table * hsz,
                                     host_dtype, store_dtype, k0, nk))
      return rc;
  }
  return LFFN_OK;
}

int lffn_convert(const void* src, int src_dtype, void* dst, int dst_dtype, int64_t n) {
  if ((!src || !dst) && n > 0) return fail(LFFN_ERR_USAGE, "convert: null buffer");
  for (int64_t i = 0; i < n; ++i) {
    double d;
    if (src_dtype == LFFN_F64) d = static_cast<const double*>(src)[i];
    else if (src_dtype == LFFN_F32) d = static_cast<const float*>(src)[i];
    else if (src_dtype == LFFN_BF16) d = bf16_to_f32(static_cast<const uint16_t*>(src)[i]);
    else return fail(LFFN_ERR_USAGE, "convert: unknown dtype");
    if (dst_dtype == LFFN_F64) static_cast<double*>(dst)[i] = d;
    else if (dst_dtype == LFFN_F32) static_cast<float*>(dst)[i] = float(d);
    else if (dst_dtype == LFFN_BF16)
      static_cast<uint16_t*>(dst)[i] = src_dtype == LFFN_F64 ? f64_to_bf16_rne(d) : f32_to_bf16_rne(float(d));
    else return fail(LFFN_ERR_USAGE, "convert: unknown dtype");
  }
  return LFFN_OK;
}

int lffn_tables_attach(lffn_ctx* c, const void* d_T, int dtype) {
  if (!c || !d_T) return fail(LFFN_ERR_USAGE, "tables attach: null argument");
  if (dtype != LFFN_F32 && dtype != LFFN_BF16)
    return fail(LFFN_ERR_USAGE, "tables attach: dtype must be f32 or bf16");
  if (reinterpret_cast<uintptr_t>(d_T) % 16 != 0)
    return fail(LFFN_ERR_USAGE, "tables attach: device buffer must be 16-byte aligned");
  c->d_T = d_T;
  c->t_dtype = dtype;
  return LFFN_OK;
}

int lffn_hash(lffn_ctx* c, const float* d_x, int64_t n, uint32_t* d_codes, float* d_coeff,
              double* d_z, void* stream) {
  if (!c) return fail(LFFN_ERR_USAGE, "null context");
  if (int rc = check_n(c, n)) return rc;
  if (n > 0 && (!d_x || !d_codes || !d_coeff)) return fail(LFFN_ERR_USAGE, "hash: null buffer");
  DeviceGuard g(c->device);
  return launch_hash(c, d_x, n, d_codes, d_coeff, d_z, static_cast<cudaStream_t>(stream));
}

int lffn_lookup_accumulate(lffn_ctx* c, const uint32_t* d_codes, const float* d_coeff, int64_t n,
                           float* d_y, int accumulate, void* stream) {
  if (!c) return fail(LFFN_ERR_USAGE, "null context");
  if (n < 0) return fail(LFFN_ERR_USAGE, "lookup accumulate: negative row count");
  if (n > 0 && (!d_codes || !d_coeff || !d_y))
    return fail(LFFN_ERR_USAGE, "lookup accumulate: null buffer");
  DeviceGuard g(c->device);
  return launch_gather(c, d_codes, d_coeff, n, d_y, accumulate ? 1 : 0,
                       static_cast<cudaStream_t>(stream));
}

int lffn_forward(lffn_ctx* c, const float* d_x, int64_t n, float* d_y, void* stream) {
  if (!c) return fail(LFFN_ERR_USAGE, "null context");
  if (int rc = check_n(c, n)) return rc;
  if (n > 0 && (!d_x || !d_y)) return fail(LFFN_ERR_USAGE, "forward: null buffer");
  if (!c->d_T) return fail(LFFN_ERR_USAGE, "lookup forward: tables not uploaded");
  DeviceGuard g(c->device);
  return forward_impl(c, d_x, n, d_y, static_cast<cudaStream_t>(stream));
}

}  // extern "C"

namespace {

// pinned (page-locked) host memory; *dev = the address the device uses for it
bool is_pinned(const void* p, void** dev = nullptr) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (dev) *dev = a.devicePointer;
  return a.type == cudaMemoryTypeHost;
}

// Small batches through the host path without copy-engine transfers of y or
// the flag: K5 writes y straight into the caller's pinned buffer (each
// element once), a one-thread kernel publishes the flag, and the host polls
// it -- no copy nodes, no driver-side synchronisation latency.  x is read in
// place for n <= 4 (every CTA of a token's cluster re-reads its row: 16 x 3 KB
// over PCIe per token is cheap for a few tokens only) and copied otherwise.
int forward_host_direct(lffn_ctx* c, const float* h_x, const float* dx, int64_t n, float* dy) {
  cudaStream_t st = c->s_comp;
  const float* xs = dx;
  if (n > 4) {
    LFFN_CUDA(cudaMemcpyAsync(c->d_xbuf, h_x, size_t(n) * size_t(c->cfg.d_in) * sizeof(float),
                              cudaMemcpyHostToDevice, st));
    xs = c->d_xbuf;
  }
  volatile int* hf = c->h_flag;
  *hf = -1;
  if (small_eligible(c, n)) {
    if (int rc = launch_small(c, xs, n, dy, 0, st)) return rc;
  } else {
    // medium batches: the two-kernel forward, the gather writing y in place
    if (int rc = launch_hash(c, xs, n, c->d_codes, c->d_coeff, nullptr, st)) return rc;
    if (int rc = launch_gather(c, c->d_codes, c->d_coeff, n, dy, 0, st)) return rc;
  }
  flag_to_host_kernel<<<1, 1, 0, st>>>(c->d_flag, c->h_flag_dev);
  LFFN_CUDA(cudaGetLastError());
  return poll_flag(c, st);
}

// Small batches through the host path: the whole call (x in, K5, y out, the
// non-finite flag read and reset) is one CUDA graph per batch size, built on
// first use; later calls patch the two host pointers and launch it.
int forward_host_graph(lffn_ctx* c, const float* h_x, int64_t n, float* h_y) {
  lffn_ctx::HostGraph& hg = c->host_graph[n];
  const size_t xb = size_t(n) * size_t(c->cfg.d_in) * sizeof(float);
  const size_t yb = size_t(n) * size_t(c->cfg.d_out) * sizeof(float);
  cudaStream_t st = c->s_comp;
  if (!hg.exec) {
    cudaGraph_t graph = nullptr;
    const int64_t launches0 = c->launches;  // the capture launches nothing
    LFFN_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    cudaMemcpyAsync(c->d_xbuf, h_x, xb, cudaMemcpyHostToDevice, st);
    const int rc = launch_small(c, c->d_xbuf, n, c->d_ybuf, 0, st);
    cudaMemcpyAsync(h_y, c->d_ybuf, yb, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(c->h_flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaMemsetAsync(c->d_flag, 0, sizeof(int), st);
    const cudaError_t ce = cudaStreamEndCapture(st, &graph);
    c->launches = launches0;
    if (rc != LFFN_OK) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    if (ce != cudaSuccess) return fail(LFFN_ERR_RUNTIME, std::string("host graph capture: ") + cudaGetErrorString(ce));
    size_t nn = 0;
    cudaGraphGetNodes(graph, nullptr, &nn);
    std::vector<cudaGraphNode_t> nodes(nn);
    cudaGraphGetNodes(graph, nodes.data(), &nn);
    for (cudaGraphNode_t nd : nodes) {
      cudaGraphNodeType ty;
      cudaGraphNodeGetType(nd, &ty);
      if (ty != cudaGraphNodeTypeMemcpy) continue;
      cudaMemcpy3DParms mp{};
      cudaGraphMemcpyNodeGetParams(nd, &mp);
      if (mp.kind == cudaMemcpyHostToDevice) hg.h2d = nd;
      else if (mp.dstPtr.ptr == static_cast<void*>(h_y)) hg.d2h = nd;
    }
    cudaGraphExec_t exec = nullptr;
    const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
    if (ie != cudaSuccess || !hg.h2d || !hg.d2h) {
      if (exec) cudaGraphExecDestroy(exec);
      cudaGraphDestroy(graph);
      hg = lffn_ctx::HostGraph{};
      return fail(LFFN_ERR_RUNTIME, "host graph: instantiation failed");
    }
    hg.exec = exec;
    hg.graph = graph;  // kept: its node handles address the exec's copies
    // the captured copies were not executed: run this call through the graph
  }
  // this call's host pointers into the two copies (nodes of the kept graph)
  LFFN_CUDA(cudaGraphExecMemcpyNodeSetParams1D(hg.exec, hg.h2d, c->d_xbuf, h_x, xb, cudaMemcpyHostToDevice));
  LFFN_CUDA(cudaGraphExecMemcpyNodeSetParams1D(hg.exec, hg.d2h, h_y, c->d_ybuf, yb, cudaMemcpyDeviceToHost));
  ++c->launches;  // K5 inside the graph
  LFFN_CUDA(cudaGraphLaunch(hg.exec, st));
  LFFN_CUDA(cudaStreamSynchronize(st));
  return flag_message(*c->h_flag);
}

}  // namespace

extern "C" {

int lffn_forward_host(lffn_ctx* c, const float* h_x, int64_t n, float* h_y) {
  if (!c) return fail(LFFN_ERR_USAGE, "null context");
  if (int rc = check_n(c, n)) return rc;
  if (n > 0 && (!h_x || !h_y)) return fail(LFFN_ERR_USAGE, "forward: null buffer");
  if (!c->d_T) return fail(LFFN_ERR_USAGE, "lookup forward: tables not uploaded");
  DeviceGuard g(c->device);
  if (n == 0) return LFFN_OK;
  void *dx = nullptr, *dy = nullptr;
  const bool pinned = is_pinned(h_x, &dx) && is_pinned(h_y, &dy);
  if (small_eligible(c, n) && pinned) {
    if (c->host_direct && dx && dy && c->h_flag_dev)
      return forward_host_direct(c, h_x, static_cast<const float*>(dx), n, static_cast<float*>(dy));
    return forward_host_graph(c, h_x, n, h_y);
  }
  if (pinned && c->host_direct && n <= c->host_direct_max && dx && dy && c->h_flag_dev && c->nc == 1 &&
      c->proj.kind != LFFN_PROJ_DENSE)
    return forward_host_direct(c, h_x, static_cast<const float*>(dx), n, static_cast<float*>(dy));
  const int64_t d_in = c->cfg.d_in, d_out = c->cfg.d_out;
  // Chunked pipeline: H2D(chunk i+1) || compute(chunk i) || D2H(chunk i-1).
  // Structured projections use no context scratch, so consecutive chunks
  // alternate between two compute streams and their kernels overlap (one
  // chunk alone does not fill the GPU); the dense kind keeps one stream (its
  // split-x / fixup scratch is per context).
  int nch = int(std::min<int64_t>(std::min(c->host_chunks, lffn_ctx::kChunks), std::max<int64_t>(1, n / 512)));
  const bool dual = c->proj.kind != LFFN_PROJ_DENSE && c->nc == 1;
  // (Zero-copy variants -- the hash reading x from the mapped pinned host
  // memory and / or the gather writing y to it, no copy-engine transfer --
  // measured slower at c2: 2.48 ms (x), 1.84-2.04 ms (y), 2.40 ms (both)
  // against 1.35 ms for the copy engines.)
  const int zc = 0;
  const int64_t per = (n + nch - 1) / nch;
  for (int i = 0; i < nch; ++i) {
    const int64_t r0 = i * per, r1 = std::min(n, r0 + per);
    if (r0 >= r1) break;
    cudaStream_t sc = (dual && (i & 1)) ? c->s_comp2 : c->s_comp;
    const float* xs = c->d_xbuf + r0 * d_in;
    if (zc & 1) {
      xs = h_x + r0 * d_in;
    } else {
      LFFN_CUDA(cudaMemcpyAsync(c->d_xbuf + r0 * d_in, h_x + r0 * d_in,
                                size_t(r1 - r0) * d_in * sizeof(float), cudaMemcpyHostToDevice, c->s_h2d));
      LFFN_CUDA(cudaEventRecord(c->ev_h2d[i], c->s_h2d));
      LFFN_CUDA(cudaStreamWaitEvent(sc, c->ev_h2d[i], 0));
    }
    float* ys = (zc & 2) ? h_y + r0 * d_out : c->d_ybuf + r0 * d_out;
    const int64_t rec = r0 * c->h_loc * c->nc;
    if (small_eligible(c, r1 - r0)) {
      if (int rc = launch_small(c, xs, r1 - r0, ys, 0, sc)) return rc;
    } else {
      if (int rc = launch_hash(c, xs, r1 - r0, c->d_codes + rec, c->d_coeff + rec, nullptr, sc)) return rc;
      if (int rc = launch_gather(c, c->d_codes + rec, c->d_coeff + rec, r1 - r0, ys, 0, sc)) return rc;
    }
    LFFN_CUDA(cudaEventRecord(c->ev_comp[i], sc));
    LFFN_CUDA(cudaStreamWaitEvent(c->s_d2h, c->ev_comp[i], 0));
    if (!(zc & 2))
      LFFN_CUDA(cudaMemcpyAsync(h_y + r0 * d_out, c->d_ybuf + r0 * d_out,
                                size_t(r1 - r0) * d_out * sizeof(float), cudaMemcpyDeviceToHost, c->s_d2h));
  }
  return read_flag(c, c->s_d2h);
}

namespace lffn_gpu {

// Backward scratch, allocated once per context on first use.
int ensure_backward_scratch(lffn_ctx* c) {
  const size_t mt = size_t(std::max<int64_t>(c->max_tokens, 1));
  if (!c->d_zbuf) LFFN_CUDA(cudaMalloc(&c->d_zbuf, mt * size_t(c->code_width) * sizeof(double)));
  if (!c->d_gzbuf) LFFN_CUDA(cudaMalloc(&c->d_gzbuf, mt * size_t(c->code_width) * sizeof(double)));
  const size_t bins = size_t(std::max<int64_t>(c->h_loc, 1)) * size_t(c->rows);
  if (!c->d_bwd_offs) {
    LFFN_CUDA(cudaMalloc(&c->d_bwd_offs, (bins + 1) * sizeof(uint32_t)));
    LFFN_CUDA(cudaMalloc(&c->d_bwd_hist, bins * kBwdBlocks * sizeof(uint32_t)));
    LFFN_CUDA(cudaMalloc(&c->d_bwd_list, mt * size_t(std::max<int64_t>(c->h_loc * c->nc, 1)) * sizeof(uint32_t)));
    LFFN_CUDA(cudaMalloc(&c->d_bwd_rank, mt * size_t(std::max<int64_t>(c->h_loc * c->nc, 1)) * sizeof(uint32_t)));
    LFFN_CUDA(cudaMalloc(&c->d_bwd_gdot, mt * size_t(std::max<int64_t>(c->h_loc * c->nc, 1)) * sizeof(double)));
  }
  if (c->proj.kind == LFFN_PROJ_SIGNFLIP && !c->d_bwd_mask) {
    const int64_t words = (c->D + 31) / 32;
    LFFN_CUDA(cudaMalloc(&c->d_bwd_mask, size_t(3 * words) * sizeof(uint32_t)));
    LFFN_CUDA(cudaMemset(c->d_bwd_mask, 0, size_t(words) * sizeof(uint32_t)));
    LFFN_CUDA(cudaMemcpy(c->d_bwd_mask + words, c->d_signmask + 2 * words, size_t(words) * sizeof(uint32_t),
                         cudaMemcpyDeviceToDevice));
    LFFN_CUDA(cudaMemcpy(c->d_bwd_mask + 2 * words, c->d_signmask + words, size_t(words) * sizeof(uint32_t),
                         cudaMemcpyDeviceToDevice));
  }
  return LFFN_OK;
}

// In-place FWHT of n rows of a [n x D] float64 array.
int launch_rows_fwht(lffn_ctx* c, double* V, int64_t n, cudaStream_t st) {
  HashParams p{};
  p.n = n;
  p.D = int(c->D);
  p.logD = int(c->logD);
  p.flag = c->d_flag;
  const int loge = c->logD >= kMaxLogE ? kMaxLogE : int(c->logD);
  const int tpt = int(c->D >> loge);
  // D = 2048: compile-time geometry, 128-thread CTAs, 3 per SM (as K1)
  const bool fixed = loge == 6 && c->logD == 11;
  const int block = std::max(tpt, ((fixed ? 128 : 256) / tpt) * tpt);
  const int tpb = block / tpt;
  p.tokens_per_block = tpb;
  p.threads_per_token = tpt;
  const size_t smem = size_t(tpb) * size_t(padded_len(int(c->D))) * sizeof(double);
  const unsigned grid = unsigned((n + tpb - 1) / tpb);
  auto go = [&](auto kernel) {
    set_smem(reinterpret_cast<const void*>(kernel), int(smem));
    kernel<<<grid, block, smem, st>>>(p, V);
  };
  if (fixed) {
    go(rows_fwht_kernel<6, 128, 3, 11>);
    ++c->launches;
    LFFN_CUDA(cudaGetLastError());
    return LFFN_OK;
  }
  switch (loge) {
    case 0: go(rows_fwht_kernel<0>); break;
    case 1: go(rows_fwht_kernel<1>); break;
    case 2: go(rows_fwht_kernel<2>); break;
    case 3: go(rows_fwht_kernel<3>); break;
    case 4: go(rows_fwht_kernel<4>); break;
    case 5: go(rows_fwht_kernel<5>); break;
    default: go(rows_fwht_kernel<6>); break;
  }
  ++c->launches;
  return LFFN_OK;
}

// acdc / bh projection backward, stage by stage over [n x D] float64 arrays
// (projection.cpp:322-360): the forward's stage inputs are recomputed, then
// the stages run backwards; parameter gradients sum over the tokens in order.
int launch_proj_backward_stagewise(lffn_ctx* c, const float* d_x, const double* gz, int64_t n,
                                   double* d_grad_x, double* d_grad_proj, cudaStream_t st) {
  const int64_t D = c->D;
  const bool acdc = c->proj.kind == LFFN_PROJ_ACDC;
  const int nst = acdc ? int(2 * c->proj.depth) : int(c->proj.stages);
  const size_t mt = size_t(std::max<int64_t>(c->max_tokens, 1));
  const size_t rows = mt * size_t(D);
  if (!c->d_bwd_rows) LFFN_CUDA(cudaMalloc(&c->d_bwd_rows, size_t(2 + nst) * rows * sizeof(double)));
  double* V = c->d_bwd_rows;
  double* G = V + rows;
  double* S = G + rows;
  const size_t bytes = size_t(n) * size_t(D) * sizeof(double);
  const unsigned ge = unsigned(std::min<int64_t>(int64_t(c->num_sms) * 16, (n * D + 255) / 256));
  const int b = int(c->proj.block == 0 ? D : c->proj.block);
  const int64_t stage_size = (D / b) * b * b;
  if (!acdc && !c->d_bhT) {
    const int64_t total = int64_t(nst) * stage_size;
    LFFN_CUDA(cudaMalloc(&c->d_bhT, size_t(total) * sizeof(double)));
    blocks_transpose_kernel<<<unsigned(std::min<int64_t>(int64_t(c->num_sms) * 8, (total + 255) / 256)), 256, 0,
                              st>>>(c->d_bh, c->d_bhT, total / (int64_t(b) * b), b);
    ++c->launches;
  }
  // forward: the stage inputs (projection.cpp:216-245)
  rows_pad_kernel<<<ge, 256, 0, st>>>(d_x, n, int(c->cfg.d_in), int(D), V);
  ++c->launches;
  for (int s = 0; s < (acdc ? nst / 2 : nst); ++s) {
    if (acdc) {
      const double* a = c->d_diag + 2 * s * D;
      LFFN_CUDA(cudaMemcpyAsync(S + size_t(2 * s) * rows, V, bytes, cudaMemcpyDeviceToDevice, st));
      rows_scale_kernel<<<ge, 256, 0, st>>>(V, n, int(D), a);
      if (int rc = launch_rows_fwht(c, V, n, st)) return rc;
      LFFN_CUDA(cudaMemcpyAsync(S + size_t(2 * s + 1) * rows, V, bytes, cudaMemcpyDeviceToDevice, st));
      rows_scale_kernel<<<ge, 256, 0, st>>>(V, n, int(D), a + D);
      if (int rc = launch_rows_fwht(c, V, n, st)) return rc;
      c->launches += 2;
    } else {
      LFFN_CUDA(cudaMemcpyAsync(S + size_t(s) * rows, V, bytes, cudaMemcpyDeviceToDevice, st));
      rows_blockdiag_kernel<false><<<ge, 256, 0, st>>>(V, G, n, int(D), b, c->d_bh + s * stage_size);
      std::swap(V, G);
      if (int rc = launch_rows_fwht(c, V, n, st)) return rc;
      ++c->launches;
    }
  }
  // backward (projection.cpp:322-360)
  rows_load_kernel<<<ge, 256, 0, st>>>(gz, n, int(c->code_width), int(D), G, c->d_flag);
  ++c->launches;
  for (int s = (acdc ? nst / 2 : nst) - 1; s >= 0; --s) {
    if (acdc) {
      const double* a = c->d_diag + 2 * s * D;
      if (int rc = launch_rows_fwht(c, G, n, st)) return rc;
      if (d_grad_proj) {
        colsum_prod_kernel<<<unsigned((D + 31) / 32), 32, 0, st>>>(S + size_t(2 * s + 1) * rows, G, n, int(D),
                                                                        d_grad_proj + (2 * s + 1) * D);
        ++c->launches;
      }
      rows_scale_kernel<<<ge, 256, 0, st>>>(G, n, int(D), a + D);
      if (int rc = launch_rows_fwht(c, G, n, st)) return rc;
      if (d_grad_proj) {
        colsum_prod_kernel<<<unsigned((D + 31) / 32), 32, 0, st>>>(S + size_t(2 * s) * rows, G, n, int(D),
                                                                        d_grad_proj + 2 * s * D);
        ++c->launches;
      }
      rows_scale_kernel<<<ge, 256, 0, st>>>(G, n, int(D), a);
      c->launches += 2;
    } else {
      if (int rc = launch_rows_fwht(c, G, n, st)) return rc;
      if (d_grad_proj) {
        // grad_B_s[g][r][c] = sum_i src_i[g*b + r] * g_i[g*b + c], tokens ascending
        dim3 grid(unsigned((b + 31) / 32), unsigned((b + 31) / 32), unsigned(D / b));
        gemm_f64_exact4_kernel<double, true, false><<<grid, 64, 0, st>>>(
            S + size_t(s) * rows, int(D), G, int(D), d_grad_proj + s * stage_size, b, b, b, int(n),
            c->d_flag, b, b, int64_t(b) * b);
        ++c->launches;
      }
      // x B_g^T through the transposed copy: the coalesced (non-transposed)
      // row kernel, same products and the same summation order
      rows_blockdiag_kernel<false><<<ge, 256, 0, st>>>(G, V, n, int(D), b, c->d_bhT + s * stage_size);
      std::swap(V, G);
      ++c->launches;
    }
  }
  if (d_grad_x) {
    rows_store_kernel<<<ge, 256, 0, st>>>(G, n, int(c->cfg.d_in), int(D), d_grad_x, c->d_flag);
    ++c->launches;
  }
  LFFN_CUDA(cudaGetLastError());
  return LFFN_OK;
}

// Projection::backward (projection.cpp:279-386) on device grad_z.
int launch_proj_backward(lffn_ctx* c, const float* d_x, const double* gz, int64_t n, double* d_grad_x,
                         double* d_grad_proj, cudaStream_t st) {
  const int d_in = int(c->cfg.d_in), cw = int(c->code_width);
  if (c->proj.kind == LFFN_PROJ_DENSE) {
    if (d_grad_x) {
      dim3 grid(unsigned((d_in + 63) / 64), unsigned((n + 63) / 64));
      gemm_f64_exact8_kernel<double, false, true><<<grid, 64, 0, st>>>(gz, cw, c->d_W, cw, d_grad_x, d_in,
                                                                      int(n), d_in, cw, c->d_flag);
      ++c->launches;
    }
    if (d_grad_proj) {
      // grad_W = x^T g: its K (tokens) must stay sequential, so the output
      // tiles are all the parallelism -- 32 x 32 tiles when 64 x 64 ones
      // would not fill the SMs a few times over
      const int64_t tiles64 = int64_t((cw + 63) / 64) * ((d_in + 63) / 64);
      if (tiles64 < int64_t(c->num_sms) * 8) {
        dim3 grid(unsigned((cw + 31) / 32), unsigned((d_in + 31) / 32));
        gemm_f64_exact4_kernel<float, true, false><<<grid, 64, 0, st>>>(d_x, d_in, gz, cw, d_grad_proj, cw,
                                                                       d_in, cw, int(n), c->d_flag);
      } else {
        dim3 grid(unsigned((cw + 63) / 64), unsigned((d_in + 63) / 64));
        gemm_f64_exact8_kernel<float, true, false><<<grid, 64, 0, st>>>(d_x, d_in, gz, cw, d_grad_proj, cw,
                                                                       d_in, cw, int(n), c->d_flag);
      }
      ++c->launches;
    }
    LFFN_CUDA(cudaGetLastError());
    return LFFN_OK;
  }
  if (c->proj.kind == LFFN_PROJ_ACDC || c->proj.kind == LFFN_PROJ_BH)
    return launch_proj_backward_stagewise(c, d_x, gz, n, d_grad_x, d_grad_proj, st);
  // signflip: grad_x only (the signs carry no gradient, param_count 0)
  if (!d_grad_x) return LFFN_OK;
  HashParams p{};
  p.n = n;
  p.d_in = d_in;
  p.D = int(c->D);
  p.logD = int(c->logD);
  p.code_width = cw;
  p.n_transforms = 3;
  p.signmask = c->d_bwd_mask;
  p.flag = c->d_flag;
  const int loge = c->logD >= kMaxLogE ? kMaxLogE : int(c->logD);
  const int tpt = int(c->D >> loge);
  // D = 2048 / 4096: compile-time geometry, 128-thread CTAs, 3 per SM (as K1)
  const bool fixed = loge == 6 && (c->logD == 11 || c->logD == 12);
  const int nt = fixed ? 128 : 256;
  const int block = std::max(tpt, (nt / tpt) * tpt);
  const int tpb = block / tpt;
  p.tokens_per_block = tpb;
  p.threads_per_token = tpt;
  const size_t smem = size_t(tpb) * size_t(padded_len(int(c->D))) * sizeof(double);
  const unsigned grid = unsigned((n + tpb - 1) / tpb);
  auto go = [&](auto kernel) {
    set_smem(reinterpret_cast<const void*>(kernel), int(smem));
    kernel<<<grid, block, smem, st>>>(p, gz, c->d_signmask, d_grad_x);
  };
  if (fixed) {
    if (c->logD == 11) go(proj_bwd_signflip_kernel<6, 128, 3, 11>);
    else go(proj_bwd_signflip_kernel<6, 128, 3, 12>);
    ++c->launches;
    LFFN_CUDA(cudaGetLastError());
    return LFFN_OK;
  }
  switch (loge) {
    case 0: go(proj_bwd_signflip_kernel<0>); break;
    case 1: go(proj_bwd_signflip_kernel<1>); break;
    case 2: go(proj_bwd_signflip_kernel<2>); break;
    case 3: go(proj_bwd_signflip_kernel<3>); break;
    case 4: go(proj_bwd_signflip_kernel<4>); break;
    case 5: go(proj_bwd_signflip_kernel<5>); break;
    default: go(proj_bwd_signflip_kernel<6>); break;
  }
  ++c->launches;
  LFFN_CUDA(cudaGetLastError());
  return LFFN_OK;
}

int check_backward_kind(const lffn_ctx*) { return LFFN_OK; }  // every projection kind

}  // namespace lffn_gpu

int lffn_proj_backward(lffn_ctx* c, const float* d_x, const double* d_grad_z, int64_t n,
                       double* d_grad_x, double* d_grad_proj, void* stream) {
  if (!c) return fail(LFFN_ERR_USAGE, "null context");
  if (int rc = check_n(c, n)) return rc;
  if (int rc = check_backward_kind(c)) return rc;
  if (n > 0 && (!d_x || !d_grad_z)) return fail(LFFN_ERR_USAGE, "projection backward: null buffer");
  if (n == 0) return LFFN_OK;
  DeviceGuard g(c->device);
  if (int rc = ensure_backward_scratch(c)) return rc;
  return launch_proj_backward(c, d_x, d_grad_z, n, d_grad_x, d_grad_proj,
                              static_cast<cudaStream_t>(stream));
}

int lffn_backward(lffn_ctx* c, const float* d_x, const float* d_grad_y, int64_t n, double* d_grad_x,
                  float* d_grad_tables, double* d_grad_proj, void* stream) {
  if (!c) return fail(LFFN_ERR_USAGE, "null context");
  if (int rc = check_n(c, n)) return rc;
  if (int rc = check_backward_kind(c)) return rc;
  if (n > 0 && (!d_x || !d_grad_y)) return fail(LFFN_ERR_USAGE, "lookup backward: null buffer");
  if (!c->d_T) return fail(LFFN_ERR_USAGE, "lookup forward: tables not uploaded");
  const int64_t bins = c->h_loc * c->rows;
  if (n * c->h_loc * c->nc > int64_t(0xffffffffu) || bins > (int64_t(1) << 28))
    return fail(LFFN_ERR_USAGE, "lookup backward: record or row count above the device limit");
  DeviceGuard g(c->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (int rc = ensure_backward_scratch(c)) return rc;
  const size_t esz = c->t_dtype == LFFN_F32 ? 4 : 2;
  if (n > 0) {
    // the forward's z (float64, exact), records and coefficients
    if (c->nc == 1) {
      if (int rc = launch_hash_top1(c, d_x, n, c->d_codes, c->d_coeff, c->d_zbuf, st, true)) return rc;
    } else if (int rc = launch_hash(c, d_x, n, c->d_codes, c->d_coeff, c->d_zbuf, st)) {
      return rc;
    }
    BwdParams p{};
    p.z = c->d_zbuf;
    p.codes = c->d_codes;
    p.coeff = c->d_coeff;
    p.gy = d_grad_y;
    p.T = c->d_T;
    p.n = n;
    p.d_out = int(c->cfg.d_out);
    p.code_width = int(c->code_width);
    p.tau = int(c->cfg.code_bits);
    p.kb = int(c->kb);
    p.hl = int(c->h_loc);
    p.nc = int(c->nc);
    p.rows = int(c->rows);
    p.scaled = (c->cfg.variant == LFFN_SCALED || c->cfg.variant == LFFN_GELU_TAU1) ? 1 : 0;
    p.gz = c->d_gzbuf;
    p.offs = c->d_bwd_offs;
    p.list = c->d_bwd_list;
    p.gT = d_grad_tables;
    p.flag = c->d_flag;
    LFFN_CUDA(cudaMemsetAsync(c->d_gzbuf, 0, size_t(n) * size_t(c->code_width) * sizeof(double), st));
    if (c->h_loc > 0) {
      const unsigned g1 = unsigned((n * 32 + 255) / 256);
      const bool v4 = c->cfg.d_out % 4 == 0;
      // bf16 rows with d_out % 8 == 0: 8 columns per lane per chunk (16-byte
      // loads); otherwise 4 (fp32 16-byte / bf16 8-byte loads)
      const bool v8 = esz == 2 && c->cfg.d_out % 8 == 0;
      const int mc = int((c->cfg.d_out + (v8 ? 255 : 127)) / (v8 ? 256 : 128));  // chunks per lane
      if (v4 && mc <= (v8 ? 4 : 8) && c->cfg.code_bits <= 24 && !c->bwd_one_pass) {
        // KB1a gdot per record (many rows in flight), KB1b gz per (token, table)
        const unsigned gg = unsigned(std::min<int64_t>(int64_t(c->num_sms) * 2, (n * 32 + 255) / 256));
#define LFFN_GDOT(TT, M, V) \
  bwd_gdot_kernel<TT, M, ((M) * (V) >= 32 ? 1 : (M) * (V) >= 24 ? 2 : 4), V><<<gg, 256, 0, st>>>(p, c->d_bwd_gdot)
        if (esz == 4) {
          if (mc <= 2) LFFN_GDOT(float, 2, 4); else if (mc <= 4) LFFN_GDOT(float, 4, 4);
          else if (mc <= 6) LFFN_GDOT(float, 6, 4); else LFFN_GDOT(float, 8, 4);
        } else if (v8) {
          // packed rows in flight: TIF 4 / 2 at 2 / 4 chunks
          if (mc <= 2) bwd_gdot_kernel<__nv_bfloat16, 2, 4, 8><<<gg, 256, 0, st>>>(p, c->d_bwd_gdot);
          else bwd_gdot_kernel<__nv_bfloat16, 4, 2, 8><<<gg, 256, 0, st>>>(p, c->d_bwd_gdot);
        } else {
          if (mc <= 2) LFFN_GDOT(__nv_bfloat16, 2, 4); else if (mc <= 4) LFFN_GDOT(__nv_bfloat16, 4, 4);
          else if (mc <= 6) LFFN_GDOT(__nv_bfloat16, 6, 4); else LFFN_GDOT(__nv_bfloat16, 8, 4);
        }
#undef LFFN_GDOT
        const unsigned gz = unsigned((n * c->h_loc + 255) / 256);
        if (c->cfg.code_bits == 8) bwd_gz_kernel<8><<<gz, 256, 0, st>>>(p, c->d_bwd_gdot);
        else if (c->cfg.code_bits == 10) bwd_gz_kernel<10><<<gz, 256, 0, st>>>(p, c->d_bwd_gdot);
        else bwd_gz_kernel<0><<<gz, 256, 0, st>>>(p, c->d_bwd_gdot);
        c->launches += 2;
      } else {
        if (esz == 4 && v4) bwd_gradz_kernel<float, 4><<<g1, 256, 0, st>>>(p);
        else if (esz == 4) bwd_gradz_kernel<float, 1><<<g1, 256, 0, st>>>(p);
        else if (v8) bwd_gradz_kernel<__nv_bfloat16, 8><<<g1, 256, 0, st>>>(p);
        else if (v4) bwd_gradz_kernel<__nv_bfloat16, 4><<<g1, 256, 0, st>>>(p);
        else bwd_gradz_kernel<__nv_bfloat16, 1><<<g1, 256, 0, st>>>(p);
        ++c->launches;
      }
    }
    if (d_grad_tables && c->h_loc > 0) {
      // deterministic buckets: ranks per token block, block offsets, row
      // starts, stable placement, one warp per row
      const int64_t hb = c->h_loc * kBwdBlocks;
      LFFN_CUDA(cudaMemsetAsync(c->d_bwd_hist, 0, size_t(hb) * size_t(c->rows) * sizeof(uint32_t), st));
      bwd_rank_kernel<<<unsigned((hb + 127) / 128), 128, 0, st>>>(p, c->d_bwd_hist, c->d_bwd_rank);
      bwd_block_offsets_kernel<<<unsigned((bins * 32 + 255) / 256), 256, 0, st>>>(p, c->d_bwd_hist);
      bwd_scan_kernel<<<1, 1024, 0, st>>>(p);
      const unsigned gr = unsigned(std::min<int64_t>(int64_t(c->num_sms) * 8, (n * c->h_loc * c->nc + 255) / 256));
      bwd_place_kernel<<<gr, 256, 0, st>>>(p, c->d_bwd_hist, c->d_bwd_rank);
      const unsigned gt = unsigned((bins * 32 + 255) / 256);
      const int mc4 = int((c->cfg.d_out + 127) / 128);
      if (c->cfg.d_out % 4 == 0) {
        if (mc4 <= 2) bwd_gradT4_kernel<2><<<gt, 256, 0, st>>>(p, 1);
        else if (mc4 <= 4) bwd_gradT4_kernel<4><<<gt, 256, 0, st>>>(p, 1);
        else if (mc4 <= 6) bwd_gradT4_kernel<6><<<gt, 256, 0, st>>>(p, 1);
        else {
          const int parts = (mc4 + 3) / 4;
          bwd_gradT4_kernel<4><<<unsigned((bins * parts * 32 + 255) / 256), 256, 0, st>>>(p, parts);
        }
      } else {
        bwd_gradT_kernel<<<gt, 256, 0, st>>>(p);
      }
      c->launches += 5;
    }
    LFFN_CUDA(cudaGetLastError());
  } else if (d_grad_tables && c->h_loc > 0) {
    LFFN_CUDA(cudaMemsetAsync(d_grad_tables, 0, size_t(bins) * size_t(c->cfg.d_out) * sizeof(float), st));
  }
  if (n > 0 && (d_grad_x || d_grad_proj))
    return launch_proj_backward(c, d_x, c->d_gzbuf, n, d_grad_x, d_grad_proj, st);
  if (n == 0 && d_grad_proj && c->proj.kind != LFFN_PROJ_SIGNFLIP)
    LFFN_CUDA(cudaMemsetAsync(d_grad_proj, 0, size_t(blob_size(&c->proj)) * sizeof(double), st));
  return LFFN_OK;
}

int lffn_sync(lffn_ctx* c, void* stream) {
  if (!c) return fail(LFFN_ERR_USAGE, "null context");
  DeviceGuard g(c->device);
  return read_flag(c, static_cast<cudaStream_t>(stream));
}

int lffn_ctx_set_option(lffn_ctx* c, int option, int64_t value) {
  if (!c) return fail(LFFN_ERR_USAGE, "null context");
  switch (option) {
    case LFFN_OPT_DENSE_EXACT:
      c->dense_exact = value != 0;
      return LFFN_OK;
    case LFFN_OPT_GATHER_VARIANT:
      if (value != 0 && value != -1)
        return fail(LFFN_ERR_USAGE, "option: no such gather variant " + std::to_string(value));
      c->gather_variant = value;
      return LFFN_OK;
    case LFFN_OPT_BWD_ONE_PASS:
      c->bwd_one_pass = value != 0;
      return LFFN_OK;
    case LFFN_OPT_HASH_EXACT:
      c->hash_exact = value != 0;
      return LFFN_OK;
    case LFFN_OPT_GATHER_SMS:
      if (value < 0) return fail(LFFN_ERR_USAGE, "option: negative SM count");
      c->gather_sms = int(value);
      return LFFN_OK;
    case LFFN_OPT_SMALL_MAX_TOKENS:
      if (value < 0) return fail(LFFN_ERR_USAGE, "option: negative small-batch limit");
      c->small_max = int(std::min<int64_t>(value, lffn_ctx::kSmallTokens));
      return LFFN_OK;
    case LFFN_OPT_HOST_CHUNKS:
      if (value < 1 || value > lffn_ctx::kChunks)
        return fail(LFFN_ERR_USAGE, "option: host chunks must be 1 .. 16");
      c->host_chunks = int(value);
      return LFFN_OK;
    case LFFN_OPT_HOST_DIRECT:
      c->host_direct = value != 0;
      c->host_direct_max = value > 1 ? value : 128;
      return LFFN_OK;
    case LFFN_OPT_BF16_COEFF_FMA:
      c->bf16w = value != 0;
      return LFFN_OK;
    case LFFN_OPT_TABLE_GROUP_BYTES:
      if (value < 0) return fail(LFFN_ERR_USAGE, "option: negative table group size");
      c->table_group_bytes = size_t(value);
      return LFFN_OK;
  }
  return fail(LFFN_ERR_USAGE, "option: unknown option " + std::to_string(option));
}

int lffn_ctx_set_timing(lffn_ctx* c, int enable) {
  if (!c) return fail(LFFN_ERR_USAGE, "null context");
  c->timing = enable != 0;
  c->timed = false;
  return LFFN_OK;
}

int lffn_ctx_stage_ms(lffn_ctx* c, float* hash_ms, float* gather_ms) {
  if (!c) return fail(LFFN_ERR_USAGE, "null context");
  if (!c->timed) {
    if (hash_ms) *hash_ms = 0.f;
    if (gather_ms) *gather_ms = 0.f;
    return LFFN_OK;
  }
  DeviceGuard g(c->device);
  LFFN_CUDA(cudaEventSynchronize(c->ev_t2));
  float a = 0.f, b = 0.f;
  LFFN_CUDA(cudaEventElapsedTime(&a, c->ev_t0, c->ev_t1));
  LFFN_CUDA(cudaEventElapsedTime(&b, c->ev_t1, c->ev_t2));
  if (hash_ms) *hash_ms = a;
  if (gather_ms) *gather_ms = b;
  return LFFN_OK;
}

}  // extern "C"
