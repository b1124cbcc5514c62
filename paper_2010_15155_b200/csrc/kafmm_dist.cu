// Multi-GPU support: one process per GPU, the tree split by
// contiguous Morton ranges of points (whole leaves).  Every rank builds the
// same global tree and lists at setup; kafmm_restrict then narrows the plan's
// work lists to the boxes whose subtree holds points of the rank's range:
//   owned leaves                  S2M, UC2UE, L2T, M2T, P2P, scatter_out
//   active boxes (range overlap)  M2M into them, M2L / S2L / DC2DE / L2L targets
// The exchanges between the upward and the downward pass (ghost and shared
// multipoles, source values, outputs) are index lists computed on the host
// from the global tree (paper_2010_15155_b200/dist.py) and carried out with
// torch.distributed (NCCL); the pack/unpack kernels below move the rows.
#include <algorithm>
#include <vector>

#include "kafmm_internal.h"

namespace kafmm {

static inline unsigned nblk(int64_t n, int t = 256) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

template <class T>
static void d2h(Plan& P, std::vector<T>& h, const T* d, int64_t n) {
  h.resize(n);
  if (n) KF_CUDA(cudaMemcpyAsync(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, P.stream));
  KF_CUDA(cudaStreamSynchronize(P.stream));
}

template <class T>
static T* h2d(Plan& P, const std::vector<T>& h) {
  T* d = dalloc<T>(P, std::max<size_t>(1, h.size()));
  if (!h.empty()) KF_CUDA(cudaMemcpyAsync(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, P.stream));
  return d;
}

// M2L (dense) tiles from the V pairs whose target is active; the pairs are
// sorted by (level, offset), so filtering keeps the runs that share an operator.
void build_m2l_batch(Plan& P) {
  free_batch(P, P.g_m2l);
  std::vector<int2> pr;
  std::vector<int32_t> lev, ijk;
  d2h(P, pr, P.d_v_pairs, P.n_v);
  d2h(P, lev, P.d_level, P.nbox);
  d2h(P, ijk, P.d_ijk, 3 * P.nbox);
  std::vector<int2> it;
  std::vector<int> key;
  for (const int2& q : pr) {
    if (!P.box_active.empty() && !P.box_active[q.y]) continue;
    const int ox = ijk[3 * q.x] - ijk[3 * q.y], oy = ijk[3 * q.x + 1] - ijk[3 * q.y + 1],
              oz = ijk[3 * q.x + 2] - ijk[3 * q.y + 2];
    int id = 0, oid = -1;
    for (int a = 0; a < 343 && oid < 0; ++a) {
      const int x = a / 49 - 3, y = (a / 7) % 7 - 3, z = a % 7 - 3;
      if (std::max(std::abs(x), std::max(std::abs(y), std::abs(z))) < 2) continue;
      if (x == ox && y == oy && z == oz) oid = id;
      ++id;
    }
    it.push_back(q);
    key.push_back(lev[q.y] * N_OFFSETS + oid);
  }
  GemmBatch& g = P.g_m2l;
  g.h_tiles.clear();
  size_t e = 0;
  while (e < it.size()) {
    size_t f = e;
    while (f < it.size() && key[f] == key[e]) ++f;
    for (size_t s = e; s < f; s += GEMM_BN)
      g.h_tiles.push_back({key[e] % N_OFFSETS, (int)s, (int)std::min<size_t>(GEMM_BN, f - s), 0,
                           std::ldexp(1.0, key[e] / N_OFFSETS)});
    e = f;
  }
  upload_batch(P, g, it);
}

// compact a CSR list (per job) to the jobs kept
template <class T>
static void compact_csr(const std::vector<int64_t>& off, const std::vector<T>& val, const std::vector<int64_t>& keep,
                        std::vector<int64_t>& noff, std::vector<T>& nval) {
  noff.assign(1, 0);
  nval.clear();
  for (int64_t j : keep) {
    for (int64_t e = off[j]; e < off[j + 1]; ++e) nval.push_back(val[e]);
    noff.push_back((int64_t)nval.size());
  }
}

void restrict_plan(Plan& P, int64_t plo, int64_t phi) {
  if (plo < 0 || phi < plo || phi > P.n) throw Error{KAFMM_EINVAL, "kafmm_restrict: bad point range"};
  if (P.restricted) throw Error{KAFMM_ESTATE, "kafmm_restrict: plan already restricted"};
  std::vector<int64_t> pb, pe;
  std::vector<uint8_t> leaf;
  std::vector<int32_t> lev, leaves;
  d2h(P, pb, P.d_pbeg, P.nbox);
  d2h(P, pe, P.d_pend, P.nbox);
  d2h(P, leaf, P.d_leaf, P.nbox);
  d2h(P, lev, P.d_level, P.nbox);
  d2h(P, leaves, P.d_leaf_ids, P.nleaf);
  P.box_active.assign(P.nbox, 0);
  for (int64_t b = 0; b < P.nbox; ++b) {
    P.box_active[b] = (pb[b] < phi && pe[b] > plo) ? 1 : 0;
    if (P.box_active[b] && leaf[b] && (pb[b] < plo || pe[b] > phi))
      throw Error{KAFMM_EINVAL, "kafmm_restrict: range boundary inside a leaf"};
  }
  Jobs& J = P.J;
  J.plo = plo;
  J.phi = phi;
  // leaf jobs (slot order) and their W lists / P2P ranges
  std::vector<int64_t> keep;
  std::vector<int32_t> lids, s2m;
  for (int64_t s = 0; s < P.nleaf; ++s)
    if (P.box_active[leaves[s]]) {
      keep.push_back(s);
      lids.push_back(leaves[s]);
      if (lev[leaves[s]] >= 2) s2m.push_back(leaves[s]);
    }
  {
    std::vector<int64_t> off, noff;
    std::vector<int32_t> src, nsrc;
    d2h(P, off, P.d_w_off, P.nleaf + 1);
    d2h(P, src, P.d_w_src, P.n_w);
    compact_csr(off, src, keep, noff, nsrc);
    J.w_off = h2d(P, noff);
    J.w_src = h2d(P, nsrc);
    std::vector<int2> rng, nrng;
    d2h(P, off, P.d_u_roff, P.nleaf + 1);
    d2h(P, rng, P.d_u_rng, off.back());
    compact_csr(off, rng, keep, noff, nrng);
    J.u_roff = h2d(P, noff);
    J.u_rng = h2d(P, nrng);
  }
  J.leaf_ids = h2d(P, lids);
  J.nleaf = (int64_t)lids.size();
  J.s2m_ids = h2d(P, s2m);
  J.ns2m = (int64_t)s2m.size();
  // S2L targets
  J.nx = 0;
  if (P.n_xbox > 0) {
    std::vector<int32_t> xt, nxt;
    std::vector<int64_t> off, noff, xkeep;
    std::vector<int2> rng, nrng;
    d2h(P, xt, P.d_x_tgt, P.n_xbox);
    d2h(P, off, P.d_x_roff, P.n_xbox + 1);
    d2h(P, rng, P.d_x_rng, off.back());
    for (int64_t j = 0; j < P.n_xbox; ++j)
      if (P.box_active[xt[j]]) {
        xkeep.push_back(j);
        nxt.push_back(xt[j]);
      }
    compact_csr(off, rng, xkeep, noff, nrng);
    J.x_tgt = h2d(P, nxt);
    J.nx = (int64_t)nxt.size();
    J.x_roff = h2d(P, noff);
    J.x_rng = h2d(P, nrng);
  }
  KF_CUDA(cudaStreamSynchronize(P.stream));
  build_gemm_batches(P);
  if (P.n_v > 0) build_m2l_batch(P);
  build_fft_chunks(P, P.fft_budget);
  P.restricted = true;
  // the work lists, GEMM batches and FFT chunk buffers were rebuilt: a graph captured
  // before must not be replayed (it points at the released lists)
  if (P.gexec) KF_CUDA(cudaGraphExecDestroy(P.gexec));
  P.gexec = nullptr;
  P.g_src = nullptr;
  P.g_out = nullptr;
}

// ---------------------------------------------------------------------------
// row movers for the exchanges
// ---------------------------------------------------------------------------
__global__ void k_pack_boxes(const double* __restrict__ a, int lda, const int32_t* __restrict__ ids, int64_t n,
                             int w, double* __restrict__ buf) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * w) return;
  int64_t j = t / w;
  int c = (int)(t - j * w);
  buf[t] = a[(int64_t)ids[j] * lda + c];
}

__global__ void k_unpack_boxes(double* __restrict__ a, int lda, const int32_t* __restrict__ ids, int64_t n, int w,
                               const double* __restrict__ buf) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * w) return;
  int64_t j = t / w;
  int c = (int)(t - j * w);
  a[(int64_t)ids[j] * lda + c] = buf[t];
}

__global__ void k_gather_rows(const double* __restrict__ src, int ld, const int64_t* __restrict__ idx, int64_t n,
                              double* __restrict__ dst) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * ld) return;
  int64_t j = t / ld;
  int c = (int)(t - j * ld);
  dst[t] = src[idx[j] * ld + c];
}

__global__ void k_scatter_rows(const double* __restrict__ src, int ld, const int64_t* __restrict__ idx, int64_t n,
                               double* __restrict__ dst) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * ld) return;
  int64_t j = t / ld;
  int c = (int)(t - j * ld);
  dst[idx[j] * ld + c] = src[t];
}

void pack_ue(Plan& P, const int32_t* ids, int64_t n, double* buf) {
  if (n <= 0) return;
  k_pack_boxes<<<nblk(n * P.neq), 256, 0, P.stream>>>(P.d_ue, P.ldn, ids, n, P.neq, buf);
  KF_CHECK_LAUNCH();
}
void unpack_ue(Plan& P, const int32_t* ids, int64_t n, const double* buf) {
  if (n <= 0) return;
  k_unpack_boxes<<<nblk(n * P.neq), 256, 0, P.stream>>>(P.d_ue, P.ldn, ids, n, P.neq, buf);
  KF_CHECK_LAUNCH();
}
void gather_rows(Plan& P, const double* src, int ld, const int64_t* idx, int64_t n, double* dst) {
  if (n <= 0) return;
  k_gather_rows<<<nblk(n * ld), 256, 0, P.stream>>>(src, ld, idx, n, dst);
  KF_CHECK_LAUNCH();
}
void scatter_rows(Plan& P, const double* src, int ld, const int64_t* idx, int64_t n, double* dst) {
  if (n <= 0) return;
  k_scatter_rows<<<nblk(n * ld), 256, 0, P.stream>>>(src, ld, idx, n, dst);
  KF_CHECK_LAUNCH();
}

}  // namespace kafmm
