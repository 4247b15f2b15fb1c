// neighbor_kernels.cuh -- multi-neighbour codes and coefficients (nc > 1).
//
// Reference (/root/reference/proj/src/lookup.cpp):
//   neighbor_codes   :118-165  the nc codes closest to the sign code, in order
//                              of increasing flip cost sum_{j flipped} |z_j|,
//                              enumerated by a min-heap frontier over the
//                              coordinates sorted by |z| (ties by index)
//   log_denominator  :102-109  sum_j |z_j| + log1p(exp(-2|z_j|))
//   code_dot         :111-116  sum_j (bit j ? z_j : -z_j)
//   forward_impl     :231-262  w = exp(dot - logden); coeff = scaled ? w * dot : w;
//                              records (table k, neighbour c), table-major
//
// The frontier is a std::priority_queue<Node, vector<Node>, greater<Node>>
// that compares costs only, so equal costs are ordered by the heap layout;
// the sift-up / sift-down below follow the libstdc++ push_heap / pop_heap
// algorithm step for step, which makes the neighbour ORDER (and therefore the
// fp32 accumulation order of the gather) identical to the reference even for
// tied costs.  One thread per (token, table); the frontier lives in local
// memory (2 nc + 4 nodes).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace lffn_gpu {

struct NeighborParams {
  const double* z;      // [n x code_width] projection output (all tables)
  int64_t n;
  int code_width;
  int tau;
  int kb, ke;           // tables owned
  int nc;               // neighbour_count (<= NCMAX)
  int scaled;
  uint32_t* codes;      // [n x (ke-kb) x nc]
  float* coeff;         // [n x (ke-kb) x nc]
  int* flag;
};

struct NbNode {
  double cost;
  uint32_t mask;
  uint32_t last;
};

// libstdc++ __push_heap with comp = greater (a "smaller" cost rises)
__device__ __forceinline__ void nb_sift_up(NbNode* h, int hole, int top, NbNode v) {
  int parent = (hole - 1) / 2;
  while (hole > top && h[parent].cost > v.cost) {
    h[hole] = h[parent];
    hole = parent;
    parent = (hole - 1) / 2;
  }
  h[hole] = v;
}

// libstdc++ __adjust_heap: move the hole to a leaf along the smaller child,
// then sift the value up from there
__device__ __forceinline__ void nb_adjust(NbNode* h, int hole, int len, NbNode v) {
  const int top = hole;
  int child = hole;
  while (child < (len - 1) / 2) {
    child = 2 * (child + 1);
    if (h[child].cost > h[child - 1].cost) --child;
    h[hole] = h[child];
    hole = child;
  }
  if ((len & 1) == 0 && child == (len - 2) / 2) {
    child = 2 * (child + 1);
    h[hole] = h[child - 1];
    hole = child - 1;
  }
  nb_sift_up(h, hole, top, v);
}

template <int NCMAX>
__global__ void __launch_bounds__(128) neighbor_kernel(NeighborParams p) {
  const int hl = p.ke - p.kb;
  const int64_t item = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= p.n * hl) return;
  const int64_t token = item / hl;
  const int k = p.kb + int(item - token * hl);
  const int tau = p.tau;
  const double* zk = p.z + token * p.code_width + (int64_t)k * tau;
  uint32_t* out_c = p.codes + item * p.nc;
  float* out_w = p.coeff + item * p.nc;

  double z[24], a[24];
  uint32_t base = 0;
  double logden = 0.0;
  for (int j = 0; j < tau; ++j) {
    z[j] = zk[j];
    a[j] = fabs(z[j]);
    base |= (z[j] >= 0.0 ? 1u : 0u) << j;                   // sign_code (lookup.cpp:74-79)
    logden = logden + (a[j] + log1p(exp(-2.0 * a[j])));    // lookup.cpp:102-109
  }
  // coordinates by (|z|, index) ascending: insertion sort of the indices
  int ord[24];
  for (int j = 0; j < tau; ++j) {
    int i = j;
    while (i > 0 && (a[ord[i - 1]] > a[j] || (a[ord[i - 1]] == a[j] && ord[i - 1] > j))) {
      ord[i] = ord[i - 1];
      --i;
    }
    ord[i] = j;
  }

  auto emit = [&](int slot, uint32_t code) {
    double dot = 0.0;  // code_dot (lookup.cpp:111-116)
    for (int j = 0; j < tau; ++j) dot = dot + (((code >> j) & 1u) ? z[j] : -z[j]);
    const double w = exp(dot - logden);
    out_c[slot] = code;
    out_w[slot] = (float)(p.scaled ? w * dot : w);
  };

  emit(0, base);
  NbNode heap[2 * NCMAX + 4];
  int len = 0;
  int nout = 1;
  heap[len++] = NbNode{a[ord[0]], 1u, 0u};
  while (nout < p.nc && len > 0) {
    // pop_heap + pop_back
    const NbNode node = heap[0];
    if (len > 1) {
      const NbNode v = heap[len - 1];
      heap[len - 1] = heap[0];
      nb_adjust(heap, 0, len - 1, v);
    }
    --len;
    uint32_t code = base;
    for (int q = 0; q < tau; ++q)
      if ((node.mask >> q) & 1u) code ^= 1u << ord[q];
    emit(nout++, code);
    if (int(node.last) + 1 < tau) {
      const uint32_t nx = node.last + 1;
      const NbNode ext{node.cost + a[ord[nx]], node.mask | (1u << nx), nx};
      heap[len] = ext;
      ++len;
      nb_sift_up(heap, len - 1, 0, heap[len - 1]);
      const NbNode swp{node.cost - a[ord[node.last]] + a[ord[nx]],
                       (node.mask ^ (1u << node.last)) | (1u << nx), nx};
      heap[len] = swp;
      ++len;
      nb_sift_up(heap, len - 1, 0, heap[len - 1]);
    }
  }
  if (!isfinite(logden)) atomicOr(p.flag, 2);
}

}  // namespace lffn_gpu
