// group.cu -- lffn_group: one rank of a table-sharded LookupFFN forward over
// an NCCL communicator the group owns (lffn_forward_sharded;
// BASELINE north star: tables split over GPUs, partial sums combined by an
// NCCL reduce-scatter or all-reduce over NVLink).
//
// The reference is single-process ("rows independent;
// embarrassingly parallel"); this is the multi-GPU mirror of
// paper_2403_07221_b200/sharded.py without torch:
//   1. hash: rank r hashes only its token block split_range(n, P, r) for ALL
//      tables (a table-less context) -- the hash is not table-separable;
//   2. records: one grouped NCCL send/recv exchange delivers to every rank
//      the (code, coefficient) records of ITS tables for all n tokens, in
//      the order the gather consumes them (for the reduce-scatter, chunk c of
//      every rank's row block is contiguous, so one gather launch per chunk
//      fills the whole staging buffer of that chunk's collective);
//   3. gather + combine: per token chunk, the rank's gather writes the fp32
//      partial over its tables, and NCCL reduces it on the group's stream
//      while the next chunk is gathered (two staging buffers).
// NCCL is loaded at run time (dlopen "libnccl.so.2": the same library torch
// loads, if it is already in the process); no NCCL symbol is linked.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>

#include "lffn_gpu.h"
#include "checked.cuh"
#include "lffn_internal.h"

using lffn_gpu::fail;

namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
  std::string error;
};

const NcclApi* nccl() {
  static NcclApi api{};
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.error = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return;
    }
#define LFFN_SYM(field, name)                                              \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));      \
  if (!api.field) {                                                        \
    api.error = std::string("libnccl.so.2 lacks ") + name;                 \
    return;                                                                \
  }
    LFFN_SYM(GetUniqueId, "ncclGetUniqueId")
    LFFN_SYM(CommInitRank, "ncclCommInitRank")
    LFFN_SYM(CommDestroy, "ncclCommDestroy")
    LFFN_SYM(GroupStart, "ncclGroupStart")
    LFFN_SYM(GroupEnd, "ncclGroupEnd")
    LFFN_SYM(Send, "ncclSend")
    LFFN_SYM(Recv, "ncclRecv")
    LFFN_SYM(AllReduce, "ncclAllReduce")
    LFFN_SYM(ReduceScatter, "ncclReduceScatter")
    LFFN_SYM(GetErrorString, "ncclGetErrorString")
#undef LFFN_SYM
  });
  return api.error.empty() ? &api : nullptr;
}

int nccl_missing() {
  static NcclApi probe{};
  (void)probe;
  return fail(LFFN_ERR_RUNTIME, "NCCL unavailable (dlopen libnccl.so.2)");
}

// even split of [0, total) into parts; the first total % parts get one more
// (sharded.py split_range)
void split_range(int64_t total, int64_t parts, int64_t index, int64_t* b, int64_t* e) {
  const int64_t base = total / parts, extra = total % parts;
  *b = index * base + std::min(index, extra);
  *e = *b + base + (index < extra ? 1 : 0);
}

// owner rank of table k under split_range(h, P, .)
__device__ __forceinline__ int owner_of(int k, int h, int P) {
  const int base = h / P, extra = h % P;
  const int big = extra * (base + 1);
  return k < big ? k / (base + 1) : extra + (k - big) / base;
}

// hasher output [m x h] -> per-destination blocks: destination q's block is
// [m x hq] at offset m * kq0 (the tables of q, token-major)
__global__ void pack_records_kernel(const uint32_t* __restrict__ codes, const float* __restrict__ coeff,
                                    int64_t m, int h, int P, uint32_t* __restrict__ scodes,
                                    float* __restrict__ scoeff) {
  const int64_t total = m * h;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / h;
    const int k = int(e - i * h);
    const int q = owner_of(k, h, P);
    const int base = h / P, extra = h % P;
    const int kq0 = q * base + min(q, extra);
    const int hq = base + (q < extra ? 1 : 0);
    const int64_t dst = m * kq0 + i * hq + (k - kq0);
    LFFN_DCHECK(dst >= 0 && dst < total && k - kq0 < hq);
    scodes[dst] = codes[e];
    scoeff[dst] = coeff[e];
  }
}

}  // namespace

struct lffn_group {
  int device = 0, rank = 0, world = 1;
  int64_t max_tokens = 0, h = 0, d_in = 0, d_out = 0, kb = 0, ke = 0;
  lffn_ctx* shard = nullptr;   // tables [kb, ke)
  lffn_ctx* hasher = nullptr;  // all tables, the rank's token block
  ncclComm_t comm = nullptr;
  cudaStream_t s_comm = nullptr;
  static constexpr int kMaxChunks = 8;
  cudaEvent_t ev_ready = nullptr, ev_recv = nullptr;
  cudaEvent_t ev_gather[kMaxChunks] = {}, ev_comm[kMaxChunks] = {};
  uint32_t* hcodes = nullptr;  // [mmax x h]
  float* hcoeff = nullptr;
  uint32_t* scodes = nullptr;  // [mmax x h] packed by destination
  float* scoeff = nullptr;
  uint32_t* rcodes = nullptr;  // [max_tokens x h_r] in gather order
  float* rcoeff = nullptr;
  float* part[2] = {nullptr, nullptr};  // reduce-scatter staging [max_tokens / chunks x d_out]
  int chunks = 4;
};

namespace {

int nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return LFFN_OK;
  const NcclApi* api = nccl();
  return fail(LFFN_ERR_RUNTIME, std::string(what) + ": " + (api ? api->GetErrorString(r) : "nccl"));
}

#define LFFN_CUDA_G(call)                                                                  \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail(LFFN_ERR_RUNTIME, std::string(#call) + ": " + cudaGetErrorString(e_));   \
  } while (0)

void destroy_group(lffn_group* g) {
  if (!g) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(g->device);
  if (g->comm && nccl()) nccl()->CommDestroy(g->comm);
  if (g->shard) lffn_ctx_destroy(g->shard);
  if (g->hasher) lffn_ctx_destroy(g->hasher);
  if (g->s_comm) cudaStreamDestroy(g->s_comm);
  if (g->ev_ready) cudaEventDestroy(g->ev_ready);
  if (g->ev_recv) cudaEventDestroy(g->ev_recv);
  for (int i = 0; i < lffn_group::kMaxChunks; ++i) {
    if (g->ev_gather[i]) cudaEventDestroy(g->ev_gather[i]);
    if (g->ev_comm[i]) cudaEventDestroy(g->ev_comm[i]);
  }
  cudaFree(g->hcodes);
  cudaFree(g->hcoeff);
  cudaFree(g->scodes);
  cudaFree(g->scoeff);
  cudaFree(g->rcodes);
  cudaFree(g->rcoeff);
  cudaFree(g->part[0]);
  cudaFree(g->part[1]);
  cudaSetDevice(prev);
  delete g;
}

}  // namespace

extern "C" {

int lffn_nccl_unique_id(void* out, int64_t len) {
  if (!out || len < NCCL_UNIQUE_ID_BYTES) return fail(LFFN_ERR_USAGE, "nccl unique id: buffer below 128 bytes");
  const NcclApi* api = nccl();
  if (!api) return nccl_missing();
  ncclUniqueId id;
  if (int rc = nccl_check(api->GetUniqueId(&id), "ncclGetUniqueId")) return rc;
  std::memcpy(out, &id, NCCL_UNIQUE_ID_BYTES);
  return LFFN_OK;
}

int lffn_group_create(lffn_group** out, int device, int64_t max_tokens, const lffn_cfg* cfg,
                      const lffn_proj* proj, const void* nccl_id, int rank, int world) {
  if (!out) return fail(LFFN_ERR_USAGE, "group create: null output");
  *out = nullptr;
  if (!cfg || !proj || !nccl_id) return fail(LFFN_ERR_USAGE, "group create: null argument");
  if (world < 1 || rank < 0 || rank >= world) return fail(LFFN_ERR_USAGE, "group create: bad rank / world");
  if (cfg->neighbor_count != 1)
    return fail(LFFN_ERR_USAGE, "group create: the sharded forward serves neighbor_count 1");
  if (max_tokens < 0) return fail(LFFN_ERR_USAGE, "group create: negative max_tokens");
  const NcclApi* api = nccl();
  if (!api) return nccl_missing();
  lffn_group* g = new lffn_group();
  g->device = device;
  g->rank = rank;
  g->world = world;
  g->max_tokens = max_tokens;
  g->h = cfg->tables;
  g->d_in = cfg->d_in;
  g->d_out = cfg->d_out;
  split_range(cfg->tables, world, rank, &g->kb, &g->ke);
  auto bail = [&](int rc) {
    destroy_group(g);
    return rc;
  };
  const int64_t mmax = (max_tokens + world - 1) / world;
  if (int rc = lffn_ctx_create_shard(&g->shard, device, max_tokens, cfg, proj, g->kb, g->ke)) return bail(rc);
  if (int rc = lffn_ctx_create_shard(&g->hasher, device, std::max<int64_t>(mmax, 1), cfg, proj, 0, cfg->tables))
    return bail(rc);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  auto restore = [&](int rc) {
    cudaSetDevice(prev);
    return rc;
  };
#define CKG(call)                                                                                     \
  do {                                                                                                \
    cudaError_t e_ = (call);                                                                          \
    if (e_ != cudaSuccess)                                                                            \
      return restore(bail(fail(LFFN_ERR_RUNTIME, std::string(#call) + ": " + cudaGetErrorString(e_)))); \
  } while (0)
  const size_t mm = size_t(std::max<int64_t>(mmax, 1)) * size_t(g->h);
  const size_t rr = size_t(std::max<int64_t>(max_tokens, 1)) * size_t(std::max<int64_t>(g->ke - g->kb, 1));
  CKG(cudaMalloc(&g->hcodes, mm * 4));
  CKG(cudaMalloc(&g->hcoeff, mm * 4));
  CKG(cudaMalloc(&g->scodes, mm * 4));
  CKG(cudaMalloc(&g->scoeff, mm * 4));
  CKG(cudaMalloc(&g->rcodes, rr * 4));
  CKG(cudaMalloc(&g->rcoeff, rr * 4));
  const size_t pb = size_t(std::max<int64_t>(max_tokens, 1)) * size_t(g->d_out) * sizeof(float);
  CKG(cudaMalloc(&g->part[0], pb));  // a chunk needs n / chunks rows; sized for chunks >= 1
  CKG(cudaMalloc(&g->part[1], pb));
  CKG(cudaStreamCreateWithFlags(&g->s_comm, cudaStreamNonBlocking));
  CKG(cudaEventCreateWithFlags(&g->ev_ready, cudaEventDisableTiming));
  CKG(cudaEventCreateWithFlags(&g->ev_recv, cudaEventDisableTiming));
  for (int i = 0; i < lffn_group::kMaxChunks; ++i) {
    CKG(cudaEventCreateWithFlags(&g->ev_gather[i], cudaEventDisableTiming));
    CKG(cudaEventCreateWithFlags(&g->ev_comm[i], cudaEventDisableTiming));
  }
#undef CKG
  ncclUniqueId id;
  std::memcpy(&id, nccl_id, NCCL_UNIQUE_ID_BYTES);
  if (int rc = nccl_check(api->CommInitRank(&g->comm, world, id, rank), "ncclCommInitRank"))
    return restore(bail(rc));
  *out = g;
  return restore(LFFN_OK);
}

int lffn_group_destroy(lffn_group* g) {
  destroy_group(g);
  return LFFN_OK;
}

lffn_ctx* lffn_group_shard(lffn_group* g) { return g ? g->shard : nullptr; }

int lffn_group_set_chunks(lffn_group* g, int chunks) {
  if (!g) return fail(LFFN_ERR_USAGE, "null group");
  if (chunks < 1 || chunks > lffn_group::kMaxChunks) return fail(LFFN_ERR_USAGE, "group: chunks must be 1 .. 8");
  g->chunks = chunks;
  return LFFN_OK;
}

int lffn_forward_sharded(lffn_group* g, const float* d_x, int64_t n, float* d_y, int combine,
                         void* stream) {
  if (!g) return fail(LFFN_ERR_USAGE, "null group");
  if (combine != LFFN_COMBINE_REDUCE_SCATTER && combine != LFFN_COMBINE_ALL_REDUCE &&
      combine != LFFN_COMBINE_NONE)
    return fail(LFFN_ERR_USAGE, "forward sharded: unknown combine");
  if (n < 0 || n > g->max_tokens)
    return fail(LFFN_ERR_USAGE, "forward sharded: row count outside [0, max_tokens]");
  if (n > 0 && (!d_x || !d_y)) return fail(LFFN_ERR_USAGE, "forward sharded: null buffer");
  const int P = g->world, r = g->rank;
  int C = g->chunks;
  if (combine == LFFN_COMBINE_REDUCE_SCATTER && n % (int64_t(P) * C) != 0)
    return fail(LFFN_ERR_USAGE, "forward sharded: reduce-scatter needs n a multiple of world * chunks");
  if (n == 0) return LFFN_OK;
  const NcclApi* api = nccl();
  if (!api) return nccl_missing();
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != g->device) cudaSetDevice(g->device);
  struct Restore {
    int dev, prev;
    ~Restore() {
      if (dev != prev) cudaSetDevice(prev);
    }
  } restore{g->device, prev};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t h = g->h, hr = g->ke - g->kb, d = g->d_out;
  int64_t t0, t1;
  split_range(n, P, r, &t0, &t1);
  const int64_t m = t1 - t0;
  // 1. hash of the rank's token block, all tables
  if (m > 0) {
    if (int rc = lffn_hash(g->hasher, d_x + t0 * g->d_in, m, g->hcodes, g->hcoeff, nullptr, st)) return rc;
    const unsigned grid = unsigned(std::min<int64_t>(1184, (m * h + 255) / 256));
    pack_records_kernel<<<grid, 256, 0, st>>>(g->hcodes, g->hcoeff, m, int(h), P, g->scodes, g->scoeff);
    LFFN_CUDA_G(cudaGetLastError());
  }
  LFFN_CUDA_G(cudaEventRecord(g->ev_ready, st));
  LFFN_CUDA_G(cudaStreamWaitEvent(g->s_comm, g->ev_ready, 0));
  // 2. records exchange into gather order
  const bool rs = combine == LFFN_COMBINE_REDUCE_SCATTER;
  const int64_t per_rank = n / P, sub = rs ? per_rank / C : 0;
  auto recv_rows = [&](int q, int c, int64_t* row0, int64_t* rows) {
    // rows of rank q's token block that land in chunk c, and where
    if (rs) {
      *row0 = int64_t(c) * P * sub + int64_t(q) * sub;
      *rows = sub;
    } else {
      int64_t a, b;
      split_range(n, P, q, &a, &b);
      *row0 = a;
      *rows = b - a;
    }
  };
  const int pieces = rs ? C : 1;
  if (int rc = nccl_check(api->GroupStart(), "ncclGroupStart")) return rc;
  for (int q = 0; q < P; ++q) {
    int64_t kq0, kq1, tq0, tq1;
    split_range(h, P, q, &kq0, &kq1);
    split_range(n, P, q, &tq0, &tq1);
    const int64_t hq = kq1 - kq0;
    for (int c = 0; c < pieces; ++c) {
      // send: my block's rows [c*sub, (c+1)*sub) (or all) for q's tables
      const int64_t s0 = rs ? int64_t(c) * sub : 0, sn = rs ? sub : m;
      const uint32_t* sc = g->scodes + m * kq0 + s0 * hq;
      const float* sw = g->scoeff + m * kq0 + s0 * hq;
      // receive: q's rows of chunk c for my tables
      int64_t row0, rows;
      recv_rows(q, c, &row0, &rows);
      uint32_t* rc_ = g->rcodes + row0 * hr;
      float* rw = g->rcoeff + row0 * hr;
      if (q == r) {
        if (sn * hq > 0) {
          LFFN_CUDA_G(cudaMemcpyAsync(rc_, sc, size_t(sn * hq) * 4, cudaMemcpyDeviceToDevice, g->s_comm));
          LFFN_CUDA_G(cudaMemcpyAsync(rw, sw, size_t(sn * hq) * 4, cudaMemcpyDeviceToDevice, g->s_comm));
        }
        continue;
      }
      if (sn * hq > 0) {
        if (int rc = nccl_check(api->Send(sc, size_t(sn * hq), ncclUint32, q, g->comm, g->s_comm), "ncclSend"))
          return rc;
        if (int rc = nccl_check(api->Send(sw, size_t(sn * hq), ncclFloat32, q, g->comm, g->s_comm), "ncclSend"))
          return rc;
      }
      if (rows * hr > 0) {
        if (int rc = nccl_check(api->Recv(rc_, size_t(rows * hr), ncclUint32, q, g->comm, g->s_comm), "ncclRecv"))
          return rc;
        if (int rc = nccl_check(api->Recv(rw, size_t(rows * hr), ncclFloat32, q, g->comm, g->s_comm), "ncclRecv"))
          return rc;
      }
    }
  }
  if (int rc = nccl_check(api->GroupEnd(), "ncclGroupEnd")) return rc;
  LFFN_CUDA_G(cudaEventRecord(g->ev_recv, g->s_comm));
  LFFN_CUDA_G(cudaStreamWaitEvent(st, g->ev_recv, 0));
  // 3. gather + combine per chunk
  if (combine == LFFN_COMBINE_NONE) {
    if (int rc = lffn_lookup_accumulate(g->shard, g->rcodes, g->rcoeff, n, d_y, 0, st)) return rc;
    if (int rc = lffn_sync(g->hasher, st)) return rc;
    return lffn_sync(g->shard, st);
  }
  if (!rs) C = int(std::min<int64_t>(C, n));
  for (int c = 0; c < C; ++c) {
    int64_t row0, rows;
    float* dst;
    if (rs) {
      row0 = int64_t(c) * P * sub;
      rows = int64_t(P) * sub;
      if (c >= 2) LFFN_CUDA_G(cudaStreamWaitEvent(st, g->ev_comm[c - 2], 0));  // staging reuse
      dst = g->part[c & 1];
    } else {
      int64_t a, b;
      split_range(n, C, c, &a, &b);
      row0 = a;
      rows = b - a;
      dst = d_y + row0 * d;
    }
    if (rows > 0)
      if (int rc = lffn_lookup_accumulate(g->shard, g->rcodes + row0 * hr, g->rcoeff + row0 * hr, rows, dst, 0, st))
        return rc;
    LFFN_CUDA_G(cudaEventRecord(g->ev_gather[c], st));
    LFFN_CUDA_G(cudaStreamWaitEvent(g->s_comm, g->ev_gather[c], 0));
    if (rs) {
      if (int rc = nccl_check(api->ReduceScatter(dst, d_y + int64_t(c) * sub * d, size_t(sub * d), ncclFloat32,
                                                 ncclSum, g->comm, g->s_comm),
                              "ncclReduceScatter"))
        return rc;
    } else if (rows > 0) {
      if (int rc = nccl_check(api->AllReduce(dst, dst, size_t(rows * d), ncclFloat32, ncclSum, g->comm, g->s_comm),
                              "ncclAllReduce"))
        return rc;
    }
    LFFN_CUDA_G(cudaEventRecord(g->ev_comm[c], g->s_comm));
  }
  LFFN_CUDA_G(cudaStreamWaitEvent(st, g->ev_comm[C - 1], 0));
  if (int rc = lffn_sync(g->hasher, st)) return rc;
  return lffn_sync(g->shard, st);
}

}  // extern "C"
