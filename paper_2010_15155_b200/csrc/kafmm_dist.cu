// Multi-GPU evaluation (the paper's MPI domain decomposition,
// PAPER.md:600-603, App. D :918-933): one process per GPU, the tree split into
// contiguous Morton ranges of the sorted points (whole leaves).
//
// Setup (kafmm_setup_dist): the ranks all-gather their points, every rank
// builds the same global tree and lists (deterministic GPU build), cuts the
// sorted points into ranges balancing an estimate of the work, and derives the
// exchange lists of every rank on the host -- the same computation on every
// rank, so nothing about them is communicated.  The rank then compacts its
// plan: heavy per-box rows (UE, CHK, DE, T) only for its active boxes (subtree
// holds owned points), the boxes straddling ranks and its ghost boxes (remote
// V / W sources); source records only for its owned points and the points of
// remote U / X leaves.  Per-rank memory therefore falls with the rank count.
//
// Evaluation (kafmm_eval on such a plan, the caller's rows in and out):
//   E1  all-to-all-v  source values: caller rows -> every rank whose local
//                     points include them (owned + remote U / X leaves)
//       up pass       gather, S2M, UC2UE, M2M; P2P starts on the side stream
//                     (it needs only E1) and overlaps E2, E3 and the down pass
//   E2  all-reduce    UE of the boxes straddling ranks (partial sums)
//   E3  all-to-all-v  ghost UE from each box's owner
//                     (E2 and E3 run on a second stream; S2L, which needs only
//                     the source records, runs meanwhile on the plan's stream)
//       down pass     M2L, DC2DE, L2L, L2T, M2T, join P2P, scatter
//   E4  all-to-all-v  outputs: owner -> caller rows
// The collectives are NCCL (kafmm_comm.cu) on the plan's stream.  The host
// logic follows the reference specification in paper_2010_15155_b200/dist.py
// (point_weights, partition, rank_maps), which the GPU tests compare with.
#include <algorithm>
#include <numeric>
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

// ---------------------------------------------------------------------------
// row movers of the exchanges
// ---------------------------------------------------------------------------
__global__ void k_pack_rows32(const double* __restrict__ a, int lda, const int32_t* __restrict__ rows, int64_t n,
                              int w, double* __restrict__ buf) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * w) return;
  int64_t j = t / w;
  int c = (int)(t - j * w);
  buf[t] = a[(int64_t)rows[j] * lda + c];
}

__global__ void k_unpack_rows32(double* __restrict__ a, int lda, const int32_t* __restrict__ rows, int64_t n, int w,
                                const double* __restrict__ buf) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * w) return;
  int64_t j = t / w;
  int c = (int)(t - j * w);
  a[(int64_t)rows[j] * lda + c] = buf[t];
}

__global__ void k_gather_rows64(const double* __restrict__ src, int ld, const int64_t* __restrict__ idx, int64_t n,
                                double* __restrict__ dst) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * ld) return;
  int64_t j = t / ld;
  int c = (int)(t - j * ld);
  dst[t] = src[idx[j] * ld + c];
}

__global__ void k_scatter_rows64(const double* __restrict__ src, int ld, const int64_t* __restrict__ idx, int64_t n,
                                 double* __restrict__ dst) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * ld) return;
  int64_t j = t / ld;
  int c = (int)(t - j * ld);
  dst[idx[j] * ld + c] = src[t];
}

static void pack_rows(Plan& P, const int32_t* rows, int64_t n, double* buf, cudaStream_t st) {
  if (n <= 0) return;
  k_pack_rows32<<<nblk(n * P.neq), 256, 0, st>>>(P.d_ue, P.ldn, rows, n, P.neq, buf);
  KF_CHECK_LAUNCH();
  P.launches++;
}
static void unpack_rows(Plan& P, const int32_t* rows, int64_t n, const double* buf, cudaStream_t st) {
  if (n <= 0) return;
  k_unpack_rows32<<<nblk(n * P.neq), 256, 0, st>>>(P.d_ue, P.ldn, rows, n, P.neq, buf);
  KF_CHECK_LAUNCH();
  P.launches++;
}

// ---------------------------------------------------------------------------
// host logic of the partition (dist.py: point_weights, partition, _needed, rank_maps)
// ---------------------------------------------------------------------------
namespace {

struct HostTree {
  int64_t nbox = 0, n = 0, nleaf = 0;
  std::vector<int32_t> level, parent, child, leaf_ids;
  std::vector<uint8_t> leaf;
  std::vector<int64_t> pbeg, pend, perm;
  // lists as (target, source) pairs in the order of kafmm_get_list
  std::vector<int32_t> ut, us, vt, vs, wt, ws, xt, xs;
};

void fetch_tree(Plan& P, HostTree& T) {
  T.nbox = P.nbox;
  T.n = P.n;
  T.nleaf = P.nleaf;
  d2h(P, T.level, P.d_level, P.nbox);
  d2h(P, T.parent, P.d_parent, P.nbox);
  d2h(P, T.child, P.d_child, 8 * P.nbox);
  d2h(P, T.leaf, P.d_leaf, P.nbox);
  d2h(P, T.pbeg, P.d_pbeg, P.nbox);
  d2h(P, T.pend, P.d_pend, P.nbox);
  d2h(P, T.perm, P.d_perm, P.n);
  d2h(P, T.leaf_ids, P.d_leaf_ids, P.nleaf);
  std::vector<int64_t> off;
  std::vector<int32_t> src;
  d2h(P, off, P.d_u_off, P.nleaf + 1);
  d2h(P, src, P.d_u_src, P.n_u);
  for (int64_t s = 0; s < P.nleaf; ++s)
    for (int64_t e = off[s]; e < off[s + 1]; ++e) {
      T.ut.push_back(T.leaf_ids[s]);
      T.us.push_back(src[e]);
    }
  std::vector<int2> vp;
  d2h(P, vp, P.d_v_pairs, P.n_v);
  for (const int2& q : vp) {
    T.vt.push_back(q.y);
    T.vs.push_back(q.x);
  }
  d2h(P, off, P.d_w_off, P.nleaf + 1);
  d2h(P, src, P.d_w_src, P.n_w);
  for (int64_t s = 0; s < P.nleaf; ++s)
    for (int64_t e = off[s]; e < off[s + 1]; ++e) {
      T.wt.push_back(T.leaf_ids[s]);
      T.ws.push_back(src[e]);
    }
  if (P.n_xbox > 0) {
    std::vector<int32_t> tg;
    d2h(P, tg, P.d_x_tgt, P.n_xbox);
    d2h(P, off, P.d_x_off, P.n_xbox + 1);
    d2h(P, src, P.d_x_src, P.n_w);
    for (int64_t s = 0; s < P.n_xbox; ++s)
      for (int64_t e = off[s]; e < off[s + 1]; ++e) {
        T.xt.push_back(tg[s]);
        T.xs.push_back(src[e]);
      }
  }
}

// estimated work per sorted point (dist.py point_weights; integer-valued box
// costs, then the same summation order, so the cuts agree with the reference)
std::vector<double> point_weights(const HostTree& T, int M, int kml, int NF) {
  const double c_pair = 30.0;
  std::vector<double> npts(T.nbox), cost(T.nbox, 0.0);
  for (int64_t b = 0; b < T.nbox; ++b) npts[b] = (double)(T.pend[b] - T.pbeg[b]);
  for (size_t e = 0; e < T.ut.size(); ++e) cost[T.ut[e]] += npts[T.ut[e]] * npts[T.us[e]] * c_pair;
  for (size_t e = 0; e < T.wt.size(); ++e) cost[T.wt[e]] += npts[T.wt[e]] * M * c_pair;
  for (size_t e = 0; e < T.xt.size(); ++e) cost[T.xt[e]] += npts[T.xs[e]] * M * c_pair;
  for (int64_t b = 0; b < T.nbox; ++b)
    if (T.leaf[b]) cost[b] += npts[b] * M * c_pair * 2.0;
  const double c_v = 8.0 * kml * kml * std::max(NF, 1);
  for (size_t e = 0; e < T.vt.size(); ++e) cost[T.vt[e]] += c_v;
  std::vector<double> dens(T.nbox), diff(T.n + 1, 0.0);
  for (int64_t b = 0; b < T.nbox; ++b) dens[b] = npts[b] > 0 ? cost[b] / std::max(npts[b], 1.0) : 0.0;
  for (int64_t b = 0; b < T.nbox; ++b) diff[T.pbeg[b]] += dens[b];
  for (int64_t b = 0; b < T.nbox; ++b) diff[T.pend[b]] += -dens[b];
  std::vector<double> w(T.n);
  double acc = 0.0;
  for (int64_t i = 0; i < T.n; ++i) {
    acc += diff[i];
    w[i] = acc;
  }
  return w;
}

// dist.py partition: cuts at leaf starts balancing the prefix sums of w
std::vector<int64_t> partition(const HostTree& T, int world, const std::vector<double>& w) {
  std::vector<int64_t> cuts{0};
  if (world == 1) {
    cuts.push_back(T.n);
    return cuts;
  }
  std::vector<double> cum(T.n + 1, 0.0);
  for (int64_t i = 0; i < T.n; ++i) cum[i + 1] = cum[i] + w[i];
  std::vector<int64_t> bounds;
  for (int64_t b = 0; b < T.nbox; ++b)
    if (T.leaf[b]) bounds.push_back(T.pbeg[b]);
  bounds.push_back(T.n);
  std::sort(bounds.begin(), bounds.end());
  bounds.erase(std::unique(bounds.begin(), bounds.end()), bounds.end());
  std::vector<double> cb(bounds.size());
  for (size_t i = 0; i < bounds.size(); ++i) cb[i] = cum[bounds[i]];
  for (int k = 1; k < world; ++k) {
    const double target = cum[T.n] * k / world;
    const int64_t j = std::lower_bound(cb.begin(), cb.end(), target) - cb.begin();
    const int64_t a = bounds[std::max<int64_t>(j - 1, 0)], b = bounds[std::min<int64_t>(j, bounds.size() - 1)];
    const int64_t c = std::abs(cum[b] - target) < std::abs(cum[a] - target) ? b : a;
    cuts.push_back(std::max(c, cuts.back()));
  }
  cuts.push_back(T.n);
  return cuts;
}

inline int rank_of(const std::vector<int64_t>& cuts, int64_t idx) {
  return (int)(std::upper_bound(cuts.begin(), cuts.end(), idx) - cuts.begin()) - 1;
}

// what rank q needs from the others (dist.py _needed)
struct Needs {
  std::vector<int32_t> ghost;                          // sorted box ids
  std::vector<std::pair<int64_t, int64_t>> ranges;     // sorted disjoint point ranges (owned + remote leaves)
  int64_t npts = 0;
};

}  // namespace

// ---------------------------------------------------------------------------
// setup of one rank
// ---------------------------------------------------------------------------
void setup_dist(Plan& P, const double* d_local_points, int64_t n_local) {
  DistState& D = *P.dist;
  Comm& C = *D.comm;
  D.rank = C.rank;
  D.world = C.world;
  const int world = D.world, me = D.rank;
  cudaStream_t st = P.stream;

  // 1. all points, in caller order (rank 0's rows, then rank 1's, ...)
  const std::vector<int64_t> cnt = C.allgather_count(n_local, st);
  D.caller_off.assign(world + 1, 0);
  for (int q = 0; q < world; ++q) D.caller_off[q + 1] = D.caller_off[q] + cnt[q];
  const int64_t n = D.caller_off[world];
  if (n < 1 || n > INT32_MAX) throw Error{KAFMM_EINVAL, "kafmm_setup_dist: total point count out of range"};
  D.n_global = n;
  D.n_caller = n_local;
  P.n = n;
  double* d_all = nullptr;
  KF_CUDA(cudaMalloc(&d_all, (size_t)n * 24));
  {
    std::vector<int64_t> sd(world, 0), sc(world, 3 * n_local), rd(world), rc(world);
    for (int q = 0; q < world; ++q) {
      rd[q] = 3 * D.caller_off[q];
      rc[q] = 3 * cnt[q];
    }
    C.alltoallv(d_local_points, sd.data(), sc.data(), d_all, rd.data(), rc.data(), st);
    KF_CUDA(cudaStreamSynchronize(st));
  }
  try {
    build_plan_core(P, d_all);
  } catch (...) {
    cudaFree(d_all);
    throw;
  }
  cudaFree(d_all);

  // 2. the partition (identical on every rank)
  HostTree T;
  fetch_tree(P, T);
  const int NF = P.NF;
  const std::vector<double> w = point_weights(T, P.M, P.kml, NF);
  D.cuts = partition(T, world, w);
  const std::vector<int64_t>& cuts = D.cuts;
  std::vector<int> lo(T.nbox), hi(T.nbox);
  for (int64_t b = 0; b < T.nbox; ++b) {
    lo[b] = rank_of(cuts, T.pbeg[b]);
    hi[b] = rank_of(cuts, std::max(T.pend[b] - 1, T.pbeg[b]));
  }
  // box b is active on the ranks whose range overlaps its points: [first, last]
  auto first_active = [&](int64_t b) {
    int r = lo[b];
    while (r < world && !(cuts[r] < T.pend[b] && cuts[r + 1] > T.pbeg[b])) ++r;
    return r;
  };
  std::vector<int> fa(T.nbox), la(T.nbox);
  for (int64_t b = 0; b < T.nbox; ++b) {
    fa[b] = first_active(b);
    la[b] = hi[b];
    while (la[b] >= fa[b] && !(cuts[la[b]] < T.pend[b] && cuts[la[b] + 1] > T.pbeg[b])) --la[b];
  }
  std::vector<uint8_t> shared(T.nbox);
  for (int64_t b = 0; b < T.nbox; ++b) shared[b] = lo[b] != hi[b];

  // 3. needs of every rank: ghost UE boxes (V / W sources of its active boxes,
  //    neither active nor shared) and remote leaves (U / X sources)
  std::vector<std::vector<uint8_t>> needbox(world, std::vector<uint8_t>(T.nbox, 0));
  std::vector<std::vector<uint8_t>> needleaf(world, std::vector<uint8_t>(T.nbox, 0));
  auto mark = [&](std::vector<std::vector<uint8_t>>& m, const std::vector<int32_t>& tg,
                  const std::vector<int32_t>& sr) {
    for (size_t e = 0; e < tg.size(); ++e)
      for (int q = fa[tg[e]]; q <= la[tg[e]]; ++q) m[q][sr[e]] = 1;
  };
  mark(needbox, T.vt, T.vs);
  mark(needbox, T.wt, T.ws);
  mark(needleaf, T.ut, T.us);
  mark(needleaf, T.xt, T.xs);
  std::vector<int64_t> leaves_by_pt;  // leaves in Morton (point) order
  for (int64_t b = 0; b < T.nbox; ++b)
    if (T.leaf[b]) leaves_by_pt.push_back(b);
  std::sort(leaves_by_pt.begin(), leaves_by_pt.end(), [&](int64_t a, int64_t b) { return T.pbeg[a] < T.pbeg[b]; });
  std::vector<Needs> need(world);
  for (int q = 0; q < world; ++q) {
    const int64_t plo = cuts[q], phi = cuts[q + 1];
    Needs& N = need[q];
    for (int64_t b = 0; b < T.nbox; ++b) {
      const bool act = T.pbeg[b] < phi && T.pend[b] > plo;
      if (needbox[q][b] && !act && !shared[b]) N.ghost.push_back((int32_t)b);
    }
    for (int64_t b : leaves_by_pt) {
      const bool own = T.pbeg[b] >= plo && T.pend[b] <= phi;
      const bool remote = needleaf[q][b] && (T.pbeg[b] < plo || T.pend[b] > phi);
      if (!(own || remote) || T.pend[b] == T.pbeg[b]) continue;
      if (!N.ranges.empty() && N.ranges.back().second == T.pbeg[b]) N.ranges.back().second = T.pend[b];
      else N.ranges.push_back({T.pbeg[b], T.pend[b]});
      N.npts += T.pend[b] - T.pbeg[b];
    }
  }
  needbox.clear();
  needleaf.clear();
  auto caller_of = [&](int64_t u) { return rank_of(D.caller_off, u); };

  // 4. this rank's rows and local points
  const int64_t plo = cuts[me], phi = cuts[me + 1];
  P.box_active.assign(T.nbox, 0);
  for (int64_t b = 0; b < T.nbox; ++b) P.box_active[b] = (T.pbeg[b] < phi && T.pend[b] > plo) ? 1 : 0;
  {
    std::vector<uint8_t> hasrow(T.nbox, 0);
    for (int64_t b = 0; b < T.nbox; ++b) hasrow[b] = P.box_active[b] || shared[b];
    for (int32_t b : need[me].ghost) hasrow[b] = 1;
    P.h_row.assign(T.nbox, -1);
    int64_t r = 0;
    for (int64_t b = 0; b < T.nbox; ++b)
      if (hasrow[b]) P.h_row[b] = (int32_t)r++;
    P.nrow = r;
  }
  const Needs& mine = need[me];
  std::vector<int64_t> l2g;  // local point -> global Morton position
  l2g.reserve(mine.npts);
  for (auto& rg : mine.ranges)
    for (int64_t g = rg.first; g < rg.second; ++g) l2g.push_back(g);
  std::vector<int64_t> rstart;  // local start of each range
  {
    int64_t a = 0;
    for (auto& rg : mine.ranges) {
      rstart.push_back(a);
      a += rg.second - rg.first;
    }
  }
  auto loc = [&](int64_t g) -> int64_t {  // local index of a kept global point
    auto it = std::upper_bound(mine.ranges.begin(), mine.ranges.end(), std::make_pair(g, INT64_MAX));
    const int64_t k = (it - mine.ranges.begin()) - 1;
    if (k < 0 || g >= mine.ranges[k].second) throw Error{KAFMM_ECUDA, "partition: point outside the local set"};
    return rstart[k] + (g - mine.ranges[k].first);
  };
  P.nloc = (int64_t)l2g.size();
  D.n_owned = phi - plo;
  D.n_ghost_points = P.nloc - D.n_owned;
  D.n_ghost_boxes = (int64_t)mine.ghost.size();
  const int64_t own0 = D.n_owned > 0 ? loc(plo) : 0;

  // 5. exchange lists
  D.counts.assign(6 * world, 0);
  // E1 values.  Sender r -> q: rows of r's caller values that q's local points need, in q's
  // local order; receiver: local point i reads position (block of its caller) + rank.
  const int ks = P.ks, kt = P.kt;
  std::vector<int64_t> val_idx;
  {
    Exchange& X = D.e1;
    X.scount.assign(world, 0);
    X.sdispl.assign(world, 0);
    X.rcount.assign(world, 0);
    X.rdispl.assign(world, 0);
    for (int q = 0; q < world; ++q) {
      X.sdispl[q] = (int64_t)val_idx.size() * ks;
      for (auto& rg : need[q].ranges)
        for (int64_t g = rg.first; g < rg.second; ++g) {
          const int64_t u = T.perm[g];
          if (caller_of(u) == me) val_idx.push_back(u - D.caller_off[me]);
        }
      X.scount[q] = (int64_t)val_idx.size() * ks - X.sdispl[q];
      D.counts[0 * world + q] = X.scount[q] / ks;
    }
    X.stotal = (int64_t)val_idx.size() * ks;
    std::vector<int64_t> per(world, 0), gperm(P.nloc);
    for (int64_t i = 0; i < P.nloc; ++i) per[caller_of(T.perm[l2g[i]])]++;
    int64_t a = 0;
    for (int q = 0; q < world; ++q) {
      X.rdispl[q] = a * ks;
      X.rcount[q] = per[q] * ks;
      D.counts[1 * world + q] = per[q];
      a += per[q];
    }
    X.rtotal = a * ks;
    std::vector<int64_t> fill(world);
    for (int q = 0; q < world; ++q) fill[q] = X.rdispl[q] / ks;
    for (int64_t i = 0; i < P.nloc; ++i) gperm[i] = fill[caller_of(T.perm[l2g[i]])]++;
    dfree(P, P.d_perm);
    P.d_perm = h2d(P, gperm);  // k_gather: local point i <- row gperm[i] of the E1 receive buffer
  }
  // E3 ghost UE: each ghost from the rank owning all its points
  std::vector<int32_t> ue_send, ue_recv;
  {
    Exchange& X = D.e3;
    X.scount.assign(world, 0);
    X.sdispl.assign(world, 0);
    X.rcount.assign(world, 0);
    X.rdispl.assign(world, 0);
    for (int q = 0; q < world; ++q) {
      X.sdispl[q] = (int64_t)ue_send.size() * P.neq;
      for (int32_t b : need[q].ghost)
        if (lo[b] == me) ue_send.push_back(P.h_row[b]);
      X.scount[q] = (int64_t)ue_send.size() * P.neq - X.sdispl[q];
      D.counts[2 * world + q] = X.scount[q] / P.neq;
    }
    for (int q = 0; q < world; ++q) {
      X.rdispl[q] = (int64_t)ue_recv.size() * P.neq;
      for (int32_t b : mine.ghost)
        if (lo[b] == q) ue_recv.push_back(P.h_row[b]);
      X.rcount[q] = (int64_t)ue_recv.size() * P.neq - X.rdispl[q];
      D.counts[3 * world + q] = X.rcount[q] / P.neq;
    }
    X.stotal = (int64_t)ue_send.size() * P.neq;
    X.rtotal = (int64_t)ue_recv.size() * P.neq;
  }
  // E2 shared boxes (the same list on every rank)
  std::vector<int32_t> shared_rows;
  for (int64_t b = 0; b < T.nbox; ++b)
    if (shared[b]) shared_rows.push_back(P.h_row[b]);
  D.nshared = (int64_t)shared_rows.size();
  // E4 outputs: owner -> caller, rows sorted by user index (so grouped by caller)
  std::vector<int64_t> operm(P.nloc, 0), out_idx;
  {
    Exchange& X = D.e4;
    X.scount.assign(world, 0);
    X.sdispl.assign(world, 0);
    X.rcount.assign(world, 0);
    X.rdispl.assign(world, 0);
    std::vector<int64_t> users(D.n_owned);
    for (int64_t g = plo; g < phi; ++g) users[g - plo] = T.perm[g];
    std::vector<int64_t> order(D.n_owned);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return users[a] < users[b]; });
    for (int64_t k = 0; k < D.n_owned; ++k) {
      operm[own0 + order[k]] = k;  // owned local point own0 + j (global plo + j) -> send row k
      X.scount[caller_of(users[order[k]])] += kt;
    }
    int64_t a = 0;
    for (int q = 0; q < world; ++q) {
      X.sdispl[q] = a;
      a += X.scount[q];
      D.counts[4 * world + q] = X.scount[q] / kt;
    }
    X.stotal = a;
    // receiver: from each owner q the sorted users owned by q whose caller is me
    std::vector<std::vector<int64_t>> from(world);
    std::vector<int64_t> inv(T.n);  // user row -> global Morton position
    for (int64_t g = 0; g < T.n; ++g) inv[T.perm[g]] = g;
    for (int64_t u = D.caller_off[me]; u < D.caller_off[me + 1]; ++u) from[rank_of(cuts, inv[u])].push_back(u);
    a = 0;
    for (int q = 0; q < world; ++q) {
      X.rdispl[q] = a * kt;
      X.rcount[q] = (int64_t)from[q].size() * kt;
      D.counts[5 * world + q] = (int64_t)from[q].size();
      for (int64_t u : from[q]) out_idx.push_back(u - D.caller_off[me]);
      a += (int64_t)from[q].size();
    }
    X.rtotal = a * kt;
  }

  for (size_t e = 0; e < T.vt.size(); ++e) D.n_v_local += P.box_active[T.vt[e]];
  for (size_t e = 0; e < T.ut.size(); ++e)
    if (P.box_active[T.ut[e]])
      D.n_p2p_local += (T.pend[T.ut[e]] - T.pbeg[T.ut[e]]) * (T.pend[T.us[e]] - T.pbeg[T.us[e]]);

  // 6. compacted work lists (local point indices; box ids, mapped to rows by the kernels)
  Jobs& J = P.J;
  J.plo = own0;
  J.phi = own0 + D.n_owned;
  std::vector<int64_t> keep;
  std::vector<int32_t> lids, s2m;
  for (int64_t s = 0; s < T.nleaf; ++s) {
    const int32_t b = T.leaf_ids[s];
    if (P.box_active[b]) {
      keep.push_back(s);
      lids.push_back(b);
      if (T.level[b] >= 2) s2m.push_back(b);
    }
  }
  auto map_ranges = [&](const std::vector<int64_t>& off, const std::vector<int2>& rng, const std::vector<int64_t>& jobs,
                        std::vector<int64_t>& noff, std::vector<int2>& nrng) {
    noff.assign(1, 0);
    nrng.clear();
    for (int64_t j : jobs) {
      for (int64_t e = off[j]; e < off[j + 1]; ++e) {
        const int64_t a = loc(rng[e].x), b = loc(rng[e].y - 1) + 1;
        if (b - a != (int64_t)rng[e].y - rng[e].x) throw Error{KAFMM_ECUDA, "partition: source range not contiguous"};
        nrng.push_back(make_int2((int)a, (int)b));
      }
      noff.push_back((int64_t)nrng.size());
    }
  };
  {
    std::vector<int64_t> off, noff;
    std::vector<int32_t> src, nsrc;
    d2h(P, off, P.d_w_off, P.nleaf + 1);
    d2h(P, src, P.d_w_src, P.n_w);
    noff.assign(1, 0);
    for (int64_t s : keep) {
      for (int64_t e = off[s]; e < off[s + 1]; ++e) nsrc.push_back(src[e]);
      noff.push_back((int64_t)nsrc.size());
    }
    J.w_off = h2d(P, noff);
    J.w_src = h2d(P, nsrc);
    std::vector<int2> rng, nrng;
    d2h(P, off, P.d_u_roff, P.nleaf + 1);
    d2h(P, rng, P.d_u_rng, off.back());
    map_ranges(off, rng, keep, noff, nrng);
    J.u_roff = h2d(P, noff);
    J.u_rng = h2d(P, nrng);
  }
  J.leaf_ids = h2d(P, lids);
  J.nleaf = (int64_t)lids.size();
  J.s2m_ids = h2d(P, s2m);
  J.ns2m = (int64_t)s2m.size();
  J.nx = 0;
  J.x_tgt = nullptr;
  J.x_rng = nullptr;
  J.x_roff = nullptr;
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
    map_ranges(off, rng, xkeep, noff, nrng);
    J.x_tgt = h2d(P, nxt);
    J.nx = (int64_t)nxt.size();
    J.x_roff = h2d(P, noff);
    J.x_rng = h2d(P, nrng);
  }
  // row maps, local point ranges of the kept leaves, local sorted points
  {
    std::vector<int32_t> crow(8 * T.nbox, -1);
    for (int64_t b = 0; b < T.nbox; ++b)
      for (int o = 0; o < 8; ++o) {
        const int32_t c = T.child[8 * b + o];
        if (c >= 0) crow[8 * b + o] = P.h_row[c];
      }
    P.d_row = h2d(P, P.h_row);
    P.d_crow = h2d(P, crow);
    std::vector<int64_t> lpb(T.nbox, 0), lpe(T.nbox, 0);
    for (int64_t b : leaves_by_pt) {
      if (T.pend[b] == T.pbeg[b]) continue;
      auto it = std::upper_bound(mine.ranges.begin(), mine.ranges.end(), std::make_pair(T.pbeg[b], INT64_MAX));
      const int64_t k = (it - mine.ranges.begin()) - 1;
      if (k >= 0 && T.pbeg[b] < mine.ranges[k].second) {
        lpb[b] = loc(T.pbeg[b]);
        lpe[b] = lpb[b] + (T.pend[b] - T.pbeg[b]);
      }
    }
    int64_t* d_l2g = h2d(P, l2g);
    double* pts = dalloc<double>(P, (size_t)std::max<int64_t>(1, P.nloc) * 4);
    if (P.nloc > 0) {
      k_gather_rows64<<<nblk(P.nloc * 4), 256, 0, st>>>(P.d_pts, 4, d_l2g, P.nloc, pts);
      KF_CHECK_LAUNCH();
    }
    KF_CUDA(cudaStreamSynchronize(st));
    dfree(P, d_l2g);
    dfree(P, P.d_pts);
    P.d_pts = pts;
    // the work lists are rebuilt from the global tree first (they read pbeg / pend of
    // no box), then the point ranges switch to local indices
    build_gemm_batches(P);
    if (P.n_v > 0) build_m2l_batch(P);
    build_fft_chunks(P, P.fft_budget);
    dfree(P, P.d_pbeg);
    dfree(P, P.d_pend);
    P.d_pbeg = h2d(P, lpb);
    P.d_pend = h2d(P, lpe);
    P.d_operm = h2d(P, operm);
  }
  // global-size lists the rank no longer uses
  for (void* p : {(void*)P.d_u_off, (void*)P.d_u_src, (void*)P.d_w_off, (void*)P.d_w_src, (void*)P.d_u_rng,
                  (void*)P.d_u_roff, (void*)P.d_x_rng, (void*)P.d_x_roff, (void*)P.d_x_tgt, (void*)P.d_x_off,
                  (void*)P.d_x_src, (void*)P.d_leaf_ids, (void*)P.d_s2m_ids})
    dfree(P, p);
  P.d_u_off = P.d_u_roff = P.d_w_off = P.d_x_roff = P.d_x_off = nullptr;
  P.d_u_src = P.d_w_src = P.d_x_tgt = P.d_x_src = P.d_leaf_ids = P.d_s2m_ids = nullptr;
  P.d_u_rng = P.d_x_rng = nullptr;
  P.restricted = true;

  // 7. workspaces at the rank's size, exchange buffers
  alloc_workspaces(P);
  D.d_val_idx = h2d(P, val_idx);
  D.d_out_idx = h2d(P, out_idx);
  D.d_ue_send_rows = h2d(P, ue_send);
  D.d_ue_recv_rows = h2d(P, ue_recv);
  D.d_shared_rows = h2d(P, shared_rows);
  for (Exchange* X : {&D.e1, &D.e3, &D.e4}) {
    X->d_sbuf = dalloc<double>(P, std::max<int64_t>(1, X->stotal));
    X->d_rbuf = dalloc<double>(P, std::max<int64_t>(1, X->rtotal));
  }
  D.d_shared_buf = dalloc<double>(P, std::max<int64_t>(1, D.nshared * P.neq));
  KF_CUDA(cudaStreamSynchronize(st));
}

// ---------------------------------------------------------------------------
// one partitioned evaluation
// ---------------------------------------------------------------------------
void run_eval_dist(Plan& P, const double* d_src, double* d_out) {
  DistState& D = *P.dist;
  Comm& C = *D.comm;
  cudaStream_t st = P.stream;
  // E1
  const int64_t nv = D.e1.stotal / P.ks;
  if (nv > 0) {
    k_gather_rows64<<<nblk(nv * P.ks), 256, 0, st>>>(d_src, P.ks, D.d_val_idx, nv, D.e1.d_sbuf);
    KF_CHECK_LAUNCH();
  }
  C.alltoallv(D.e1.d_sbuf, D.e1.sdispl.data(), D.e1.scount.data(), D.e1.d_rbuf, D.e1.rdispl.data(),
              D.e1.rcount.data(), st);
  run_eval_up(P, D.e1.d_rbuf);  // P2P now runs on the side stream, overlapping E2 / E3
  int extra = 1;
  // E2 and E3 on the exchange stream once the upward pass is done, while the plan's
  // stream runs S2L (issued first, so that a host-blocking transport still overlaps);
  // stage timing (mode 1) keeps everything on one stream in the original order
  const bool overlap = P.timing != 1;
  cudaStream_t xs = overlap ? P.cstream : st;
  if (overlap) {
    KF_CUDA(cudaEventRecord(P.ev_up, st));
    run_eval_s2l(P);
    KF_CUDA(cudaStreamWaitEvent(xs, P.ev_up, 0));
  }
  // E2
  if (D.nshared > 0) {
    pack_rows(P, D.d_shared_rows, D.nshared, D.d_shared_buf, xs);
    C.allreduce(D.d_shared_buf, D.nshared * P.neq, xs);
    unpack_rows(P, D.d_shared_rows, D.nshared, D.d_shared_buf, xs);
  }
  // E3
  pack_rows(P, D.d_ue_send_rows, D.e3.stotal / P.neq, D.e3.d_sbuf, xs);
  C.alltoallv(D.e3.d_sbuf, D.e3.sdispl.data(), D.e3.scount.data(), D.e3.d_rbuf, D.e3.rdispl.data(),
              D.e3.rcount.data(), xs);
  unpack_rows(P, D.d_ue_recv_rows, D.e3.rtotal / P.neq, D.e3.d_rbuf, xs);
  if (overlap) {
    KF_CUDA(cudaEventRecord(P.ev_ghost, xs));
    KF_CUDA(cudaStreamWaitEvent(st, P.ev_ghost, 0));
  }
  const int up_launches = P.launches;
  run_eval_down(P, D.e4.d_sbuf);
  // E4
  C.alltoallv(D.e4.d_sbuf, D.e4.sdispl.data(), D.e4.scount.data(), D.e4.d_rbuf, D.e4.rdispl.data(),
              D.e4.rcount.data(), st);
  const int64_t no = D.e4.rtotal / P.kt;
  if (no > 0) {
    k_scatter_rows64<<<nblk(no * P.kt), 256, 0, st>>>(D.e4.d_rbuf, P.kt, D.d_out_idx, no, d_out);
    KF_CHECK_LAUNCH();
    ++extra;
  }
  (void)up_launches;
  P.launches += extra;
}

}  // namespace kafmm
