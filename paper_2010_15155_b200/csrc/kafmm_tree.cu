// Setup on the GPU: Morton keys, radix sort, level-by-level octree split,
// U/V/W/X interaction lists, and the GEMM work lists of the evaluation pass.
//
// Tree definition (reading R4): root [0,1)^3,
// q = floor(x 2^21) clamped, a box splits iff count > cap and level < 20,
// only non-empty children are kept, no 2:1 balance.
// Lists (PAPER.md:152-156 + reading R3): adjacency = closed boxes intersect;
//   U(B) leaf: all adjacent leaves incl. B;  V(B): children of the parent's
//   colleagues not adjacent to B;  W(B) leaf: descendants D of B's colleagues
//   with D not adjacent and parent(D) adjacent;  X(B) = {A : B in W(A)}.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "kafmm_internal.h"

namespace kafmm {

// ---------------------------------------------------------------------------
// Morton helpers
// ---------------------------------------------------------------------------
__host__ __device__ inline uint64_t spread3(uint32_t v) {
  uint64_t x = v & 0x1fffff;
  x = (x | x << 32) & 0x1f00000000ffffULL;
  x = (x | x << 16) & 0x1f0000ff0000ffULL;
  x = (x | x << 8) & 0x100f00f00f00f00fULL;
  x = (x | x << 4) & 0x10c30c30c30c30c3ULL;
  x = (x | x << 2) & 0x1249249249249249ULL;
  return x;
}
__host__ __device__ inline uint32_t compact3(uint64_t x) {
  x &= 0x1249249249249249ULL;
  x = (x ^ (x >> 2)) & 0x10c30c30c30c30c3ULL;
  x = (x ^ (x >> 4)) & 0x100f00f00f00f00fULL;
  x = (x ^ (x >> 8)) & 0x1f0000ff0000ffULL;
  x = (x ^ (x >> 16)) & 0x1f00000000ffffULL;
  x = (x ^ (x >> 32)) & 0x1fffffULL;
  return (uint32_t)x;
}
__host__ __device__ inline uint64_t morton3(uint32_t i, uint32_t j, uint32_t k) {
  return (spread3(i) << 2) | (spread3(j) << 1) | spread3(k);
}

__global__ void k_validate_keys(const double* __restrict__ pts, int64_t n, uint64_t* keys,
                                int64_t* idx, int* flag) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t q[3];
  for (int a = 0; a < 3; ++a) {
    double x = pts[3 * i + a];
    if (!isfinite(x)) {
      atomicOr(flag, 2);
      x = 0.0;
    } else if (!(x >= 0.0 && x < 1.0)) {
      atomicOr(flag, 1);
      x = 0.0;
    }
    double s = floor(x * (double)(1 << QBITS));
    s = fmin(fmax(s, 0.0), (double)((1 << QBITS) - 1));
    q[a] = (uint32_t)s;
  }
  keys[i] = morton3(q[0], q[1], q[2]);
  idx[i] = i;
}

__global__ void k_sorted_points(const double* __restrict__ pts, const int64_t* __restrict__ perm,
                                int64_t n, double* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t u = perm[i];
  out[4 * i + 0] = pts[3 * u + 0];
  out[4 * i + 1] = pts[3 * u + 1];
  out[4 * i + 2] = pts[3 * u + 2];
  out[4 * i + 3] = 0.0;
}

// per box of level l: child counts by binary search of the sorted keys
__global__ void k_split(const uint64_t* __restrict__ keys, int64_t nb, const uint64_t* __restrict__ bkey,
                        const int64_t* __restrict__ pb, const int64_t* __restrict__ pe, int level, int cap,
                        int64_t* ccnt, int64_t* cbeg) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= nb) return;
  int64_t lo = pb[b], hi = pe[b];
  bool split = (hi - lo > cap) && level < MAX_LEVEL;
  int shift = 3 * (QBITS - 1 - level);
  int64_t prev = lo;
  for (int o = 0; o < 8; ++o) {
    int64_t end;
    if (!split) {
      end = lo;
    } else if (o == 7) {
      end = hi;
    } else {
      uint64_t bound = ((bkey[b] << 3) | (uint64_t)(o + 1)) << shift;
      int64_t a = prev, c = hi;  // first index with key >= bound
      while (a < c) {
        int64_t m = (a + c) >> 1;
        if (keys[m] < bound) a = m + 1; else c = m;
      }
      end = a;
    }
    ccnt[8 * b + o] = split ? end - prev : 0;
    cbeg[8 * b + o] = prev;
    prev = end;
  }
}

__global__ void k_nz_flags(const int64_t* c, int64_t* f, int64_t m) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < m) f[t] = c[t] > 0 ? 1 : 0;
  if (t == m) f[t] = 0;
}

__global__ void k_emit_children(int64_t nb, int64_t base_this, int64_t base_next, const uint64_t* __restrict__ bkey,
                                const int64_t* __restrict__ ccnt, const int64_t* __restrict__ cbeg,
                                const int64_t* __restrict__ cpos, uint64_t* nkey, int64_t* npb, int64_t* npe,
                                int32_t* npar, int32_t* child_of_this) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= 8 * nb) return;
  int64_t b = t >> 3;
  int o = (int)(t & 7);
  if (ccnt[t] > 0) {
    int64_t c = cpos[t];
    nkey[c] = (bkey[b] << 3) | (uint64_t)o;
    npb[c] = cbeg[t];
    npe[c] = cbeg[t] + ccnt[t];
    npar[c] = (int32_t)(base_this + b);
    child_of_this[t] = (int32_t)(base_next + c);
  } else {
    child_of_this[t] = -1;
  }
}

__global__ void k_box_geometry(int64_t nbox, const uint64_t* __restrict__ key, const int32_t* __restrict__ level,
                               const int32_t* __restrict__ child, int32_t* ijk, uint8_t* leaf) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= nbox) return;
  uint64_t k = key[b];
  ijk[3 * b + 0] = (int32_t)compact3(k >> 2);
  ijk[3 * b + 1] = (int32_t)compact3(k >> 1);
  ijk[3 * b + 2] = (int32_t)compact3(k);
  bool lf = true;
  for (int o = 0; o < 8; ++o) lf &= child[8 * b + o] < 0;
  leaf[b] = lf ? 1 : 0;
  (void)level;
}

// ---------------------------------------------------------------------------
// list construction
// ---------------------------------------------------------------------------
struct TreeView {
  const int32_t* level;
  const int32_t* ijk;
  const int32_t* parent;
  const int32_t* child;
  const uint8_t* leaf;
  const uint64_t* key;
  const int64_t* lbeg;  // per level begin (depth+2 entries)
  int depth;
};

__device__ inline int32_t find_box(const TreeView& T, int l, int i, int j, int k) {
  if (l > T.depth) return -1;
  int n = 1 << l;
  if (i < 0 || j < 0 || k < 0 || i >= n || j >= n || k >= n) return -1;
  uint64_t key = morton3((uint32_t)i, (uint32_t)j, (uint32_t)k);
  int64_t a = T.lbeg[l], c = T.lbeg[l + 1];
  while (a < c) {
    int64_t m = (a + c) >> 1;
    if (T.key[m] < key) a = m + 1; else c = m;
  }
  if (a < T.lbeg[l + 1] && T.key[a] == key) return (int32_t)a;
  return -1;
}

// closed boxes A (finer or equal level) and B intersect
__device__ inline bool adjacent(const TreeView& T, int32_t a, int32_t b) {
  int la = T.level[a], lb = T.level[b];
  if (la < lb) { int32_t t = a; a = b; b = t; int tl = la; la = lb; lb = tl; }
  int s = la - lb;
  for (int d = 0; d < 3; ++d) {
    int ia = T.ijk[3 * a + d];
    int lo = T.ijk[3 * b + d] << s, hi = (T.ijk[3 * b + d] + 1) << s;
    if (ia > hi || ia + 1 < lo) return false;
  }
  return true;
}

// U and W of one leaf.  When out arrays are null only counts are produced.
__device__ void leaf_lists(const TreeView& T, int32_t B, int64_t* nu, int64_t* nw, int32_t* u_out,
                           int32_t* w_out) {
  int l = T.level[B];
  int bi = T.ijk[3 * B], bj = T.ijk[3 * B + 1], bk = T.ijk[3 * B + 2];
  int64_t cu = 0, cw = 0;
  if (u_out) u_out[cu] = B;
  cu++;
  int32_t stack[8 * (MAX_LEVEL + 2)];
  for (int d = 0; d < 27; ++d) {
    if (d == 13) continue;
    int dx = d / 9 - 1, dy = (d / 3) % 3 - 1, dz = d % 3 - 1;
    int ci = bi + dx, cj = bj + dy, ck = bk + dz;
    int n = 1 << l;
    if (ci < 0 || cj < 0 || ck < 0 || ci >= n || cj >= n || ck >= n) continue;
    for (int lp = l; lp >= 0; --lp) {
      int s = l - lp;
      int32_t b2 = find_box(T, lp, ci >> s, cj >> s, ck >> s);
      if (b2 < 0) continue;
      if (T.leaf[b2]) {
        bool first = true;  // a coarser leaf containing several neighbour cells: emit once
        if (lp < l) {
          for (int e = 0; e < d && first; ++e) {
            if (e == 13) continue;
            int ei = bi + e / 9 - 1, ej = bj + (e / 3) % 3 - 1, ek = bk + e % 3 - 1;
            if (ei < 0 || ej < 0 || ek < 0 || ei >= n || ej >= n || ek >= n) continue;
            if ((ei >> s) == (ci >> s) && (ej >> s) == (cj >> s) && (ek >> s) == (ck >> s)) first = false;
          }
        }
        if (first) {
          if (u_out) u_out[cu] = b2;
          cu++;
        }
      } else if (lp == l) {
        // non-leaf colleague: descend through boxes adjacent to B
        int sp = 0;
        stack[sp++] = b2;
        while (sp > 0) {
          int32_t c = stack[--sp];
          for (int o = 0; o < 8; ++o) {
            int32_t D = T.child[8 * c + o];
            if (D < 0) continue;
            if (adjacent(T, D, B)) {
              if (T.leaf[D]) {
                if (u_out) u_out[cu] = D;
                cu++;
              } else {
                stack[sp++] = D;
              }
            } else {
              if (w_out) w_out[cw] = D;
              cw++;
            }
          }
        }
      }
      break;  // the deepest existing box containing the cell decides
    }
  }
  *nu = cu;
  *nw = cw;
}

__global__ void k_leaf_lists(TreeView T, const int32_t* __restrict__ leaves, int64_t nleaf, int64_t* ucnt,
                             int64_t* wcnt, const int64_t* __restrict__ uoff, const int64_t* __restrict__ woff,
                             int32_t* usrc, int32_t* wsrc) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= nleaf) return;
  int64_t nu, nw;
  if (usrc == nullptr) {
    leaf_lists(T, leaves[s], &nu, &nw, nullptr, nullptr);
    ucnt[s] = nu;
    wcnt[s] = nw;
  } else {
    leaf_lists(T, leaves[s], &nu, &nw, usrc + uoff[s], wsrc + woff[s]);
  }
}

__constant__ int16_t c_offset_id[343];

__global__ void k_v_lists(TreeView T, int64_t b0, int64_t b1, int64_t* vcnt, const int64_t* __restrict__ voff,
                          int2* pairs, int32_t* keys) {
  int64_t B = b0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (B >= b1) return;
  int l = T.level[B];
  int bi = T.ijk[3 * B], bj = T.ijk[3 * B + 1], bk = T.ijk[3 * B + 2];
  int64_t c = 0;
  int64_t base = pairs ? voff[B - b0] : 0;
  for (int d = 0; d < 27; ++d) {
    if (d == 13) continue;
    int32_t Q = find_box(T, l - 1, (bi >> 1) + d / 9 - 1, (bj >> 1) + (d / 3) % 3 - 1, (bk >> 1) + d % 3 - 1);
    if (Q < 0) continue;
    for (int o = 0; o < 8; ++o) {
      int32_t C = T.child[8 * Q + o];
      if (C < 0) continue;
      int ox = T.ijk[3 * C] - bi, oy = T.ijk[3 * C + 1] - bj, oz = T.ijk[3 * C + 2] - bk;
      int m = max(abs(ox), max(abs(oy), abs(oz)));
      if (m < 2) continue;  // adjacent
      if (pairs) {
        pairs[base + c] = make_int2(C, (int32_t)B);
        keys[base + c] = l * N_OFFSETS + c_offset_id[(ox + 3) * 49 + (oy + 3) * 7 + (oz + 3)];
      }
      c++;
    }
  }
  if (!pairs) vcnt[B - b0] = c;
}

__global__ void k_x_pairs(const int32_t* __restrict__ leaves, int64_t nleaf, const int64_t* __restrict__ woff,
                          const int32_t* __restrict__ wsrc, int32_t* xkey, int32_t* xval) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= nleaf) return;
  for (int64_t e = woff[s]; e < woff[s + 1]; ++e) {
    xkey[e] = wsrc[e];   // target box D of S2L
    xval[e] = leaves[s]; // source leaf A
  }
}

// ---------------------------------------------------------------------------
// host orchestration
// ---------------------------------------------------------------------------
static inline unsigned nblk(int64_t n, int t = 256) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

template <class T>
static void to_host(Plan& P, std::vector<T>& h, const T* d, int64_t n) {
  h.resize(n);
  if (n) KF_CUDA(cudaMemcpyAsync(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, P.stream));
  KF_CUDA(cudaStreamSynchronize(P.stream));
}

static void exclusive_scan(Plan& P, const int64_t* in, int64_t* out, int64_t n) {
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, P.stream);
  void* d_tmp = nullptr;
  KF_CUDA(cudaMallocAsync(&d_tmp, tmp + 8, P.stream));
  cub::DeviceScan::ExclusiveSum(d_tmp, tmp, in, out, n, P.stream);
  KF_CUDA(cudaFreeAsync(d_tmp, P.stream));
}

// per job s: the point ranges [pbeg, pend) of boxes src[off[s] .. off[s+1]),
// sorted and merged where they touch
static void merged_ranges(const std::vector<int64_t>& off, const std::vector<int32_t>& src,
                          const std::vector<int64_t>& pb, const std::vector<int64_t>& pe, int64_t njobs,
                          std::vector<int2>& rng, std::vector<int64_t>& roff) {
  rng.clear();
  roff.assign(1, 0);
  std::vector<int2> tmp;
  for (int64_t s = 0; s < njobs; ++s) {
    tmp.clear();
    for (int64_t e = off[s]; e < off[s + 1]; ++e) {
      const int32_t b = src[e];
      if (pe[b] > pb[b]) tmp.push_back(make_int2((int)pb[b], (int)pe[b]));
    }
    std::sort(tmp.begin(), tmp.end(), [](int2 a, int2 b) { return a.x < b.x; });
    for (size_t i = 0; i < tmp.size(); ++i) {
      if (i > 0 && rng.back().y == tmp[i].x) rng.back().y = tmp[i].y;
      else rng.push_back(tmp[i]);
    }
    roff.push_back((int64_t)rng.size());
  }
}

void build_tree_and_lists(Plan& P, const double* d_points) {
  const int64_t n = P.n;
  cudaStream_t st = P.stream;
  // 1. validate + Morton keys + sort --------------------------------------
  uint64_t *d_k0, *d_k1;
  int64_t *d_i0;
  KF_CUDA(cudaMallocAsync(&d_k0, n * 8, st));
  KF_CUDA(cudaMallocAsync(&d_k1, n * 8, st));
  KF_CUDA(cudaMallocAsync(&d_i0, n * 8, st));
  P.d_perm = dalloc<int64_t>(P, n);
  P.d_flag = dalloc<int>(P, 4);
  k_validate_keys<<<nblk(n), 256, 0, st>>>(d_points, n, d_k0, d_i0, P.d_flag);
  KF_CHECK_LAUNCH();
  int hflag = 0;
  KF_CUDA(cudaMemcpyAsync(&hflag, P.d_flag, 4, cudaMemcpyDeviceToHost, st));
  KF_CUDA(cudaStreamSynchronize(st));
  if (hflag & 2) throw Error{KAFMM_ENONFINITE, "non-finite point coordinate"};
  if (hflag & 1) throw Error{KAFMM_EDOMAIN, "point outside [0,1)^3"};
  {
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, d_k0, d_k1, d_i0, P.d_perm, n, 0, 63, st);
    void* d_tmp;
    KF_CUDA(cudaMallocAsync(&d_tmp, tmp + 8, st));
    cub::DeviceRadixSort::SortPairs(d_tmp, tmp, d_k0, d_k1, d_i0, P.d_perm, n, 0, 63, st);
    KF_CUDA(cudaFreeAsync(d_tmp, st));
  }
  P.d_pts = dalloc<double>(P, 4 * n);
  k_sorted_points<<<nblk(n), 256, 0, st>>>(d_points, P.d_perm, n, P.d_pts);
  KF_CHECK_LAUNCH();

  // 2. level-by-level split -------------------------------------------------
  struct LevelBufs {
    uint64_t* key;
    int64_t *pb, *pe;
    int32_t *par, *child;
    int64_t nb;
  };
  std::vector<LevelBufs> L;
  {
    LevelBufs r;
    r.nb = 1;
    KF_CUDA(cudaMallocAsync(&r.key, 8, st));
    KF_CUDA(cudaMallocAsync(&r.pb, 8, st));
    KF_CUDA(cudaMallocAsync(&r.pe, 8, st));
    KF_CUDA(cudaMallocAsync(&r.par, 4, st));
    uint64_t z = 0;
    int64_t zb = 0;
    int32_t mp = -1;
    KF_CUDA(cudaMemcpyAsync(r.key, &z, 8, cudaMemcpyHostToDevice, st));
    KF_CUDA(cudaMemcpyAsync(r.pb, &zb, 8, cudaMemcpyHostToDevice, st));
    KF_CUDA(cudaMemcpyAsync(r.pe, &n, 8, cudaMemcpyHostToDevice, st));
    KF_CUDA(cudaMemcpyAsync(r.par, &mp, 4, cudaMemcpyHostToDevice, st));
    KF_CUDA(cudaStreamSynchronize(st));
    L.push_back(r);
  }
  int64_t base = 0;
  for (int l = 0;; ++l) {
    LevelBufs& cur = L[l];
    KF_CUDA(cudaMallocAsync(&cur.child, cur.nb * 8 * 4, st));
    int64_t *ccnt, *cbeg, *cpos, *nzf;
    KF_CUDA(cudaMallocAsync(&ccnt, cur.nb * 8 * 8, st));
    KF_CUDA(cudaMallocAsync(&cbeg, cur.nb * 8 * 8, st));
    KF_CUDA(cudaMallocAsync(&cpos, (cur.nb * 8 + 1) * 8, st));
    KF_CUDA(cudaMallocAsync(&nzf, (cur.nb * 8 + 1) * 8, st));
    k_split<<<nblk(cur.nb), 256, 0, st>>>(d_k1, cur.nb, cur.key, cur.pb, cur.pe, l, P.cap, ccnt, cbeg);
    KF_CHECK_LAUNCH();
    k_nz_flags<<<nblk(cur.nb * 8 + 1), 256, 0, st>>>(ccnt, nzf, cur.nb * 8);
    KF_CHECK_LAUNCH();
    exclusive_scan(P, nzf, cpos, cur.nb * 8 + 1);
    int64_t nnext = 0;
    KF_CUDA(cudaMemcpyAsync(&nnext, cpos + cur.nb * 8, 8, cudaMemcpyDeviceToHost, st));
    KF_CUDA(cudaStreamSynchronize(st));
    LevelBufs nx;
    nx.nb = nnext;
    nx.key = nullptr;
    if (nnext > 0) {
      KF_CUDA(cudaMallocAsync(&nx.key, nnext * 8, st));
      KF_CUDA(cudaMallocAsync(&nx.pb, nnext * 8, st));
      KF_CUDA(cudaMallocAsync(&nx.pe, nnext * 8, st));
      KF_CUDA(cudaMallocAsync(&nx.par, nnext * 4, st));
    }
    k_emit_children<<<nblk(cur.nb * 8), 256, 0, st>>>(cur.nb, base, base + cur.nb, cur.key, ccnt, cbeg, cpos, nx.key,
                                                     nx.pb, nx.pe, nx.par, cur.child);
    KF_CHECK_LAUNCH();
    KF_CUDA(cudaFreeAsync(ccnt, st));
    KF_CUDA(cudaFreeAsync(cbeg, st));
    KF_CUDA(cudaFreeAsync(cpos, st));
    KF_CUDA(cudaFreeAsync(nzf, st));
    base += cur.nb;
    if (nnext == 0) break;
    L.push_back(nx);
  }
  P.depth = (int)L.size() - 1;
  P.nbox = base;
  P.levels.clear();
  int64_t off = 0;
  for (auto& lv : L) {
    P.levels.push_back({off, off + lv.nb});
    off += lv.nb;
  }
  // 3. concatenate levels -----------------------------------------------------
  P.d_key = dalloc<uint64_t>(P, P.nbox);
  P.d_pbeg = dalloc<int64_t>(P, P.nbox);
  P.d_pend = dalloc<int64_t>(P, P.nbox);
  P.d_parent = dalloc<int32_t>(P, P.nbox);
  P.d_child = dalloc<int32_t>(P, 8 * P.nbox);
  P.d_level = dalloc<int32_t>(P, P.nbox);
  P.d_ijk = dalloc<int32_t>(P, 3 * P.nbox);
  P.d_leaf = dalloc<uint8_t>(P, P.nbox);
  {
    std::vector<int32_t> hlev(P.nbox);
    for (int l = 0; l <= P.depth; ++l) {
      int64_t o = P.levels[l].begin, m = L[l].nb;
      KF_CUDA(cudaMemcpyAsync(P.d_key + o, L[l].key, m * 8, cudaMemcpyDeviceToDevice, st));
      KF_CUDA(cudaMemcpyAsync(P.d_pbeg + o, L[l].pb, m * 8, cudaMemcpyDeviceToDevice, st));
      KF_CUDA(cudaMemcpyAsync(P.d_pend + o, L[l].pe, m * 8, cudaMemcpyDeviceToDevice, st));
      KF_CUDA(cudaMemcpyAsync(P.d_parent + o, L[l].par, m * 4, cudaMemcpyDeviceToDevice, st));
      KF_CUDA(cudaMemcpyAsync(P.d_child + 8 * o, L[l].child, m * 32, cudaMemcpyDeviceToDevice, st));
      for (int64_t b = 0; b < m; ++b) hlev[o + b] = l;
    }
    KF_CUDA(cudaMemcpyAsync(P.d_level, hlev.data(), P.nbox * 4, cudaMemcpyHostToDevice, st));
    KF_CUDA(cudaStreamSynchronize(st));
    for (auto& lv : L) {
      KF_CUDA(cudaFreeAsync(lv.key, st));
      KF_CUDA(cudaFreeAsync(lv.pb, st));
      KF_CUDA(cudaFreeAsync(lv.pe, st));
      KF_CUDA(cudaFreeAsync(lv.par, st));
      KF_CUDA(cudaFreeAsync(lv.child, st));
    }
  }
  k_box_geometry<<<nblk(P.nbox), 256, 0, st>>>(P.nbox, P.d_key, P.d_level, P.d_child, P.d_ijk, P.d_leaf);
  KF_CHECK_LAUNCH();
  KF_CUDA(cudaFreeAsync(d_k0, st));
  KF_CUDA(cudaFreeAsync(d_k1, st));
  KF_CUDA(cudaFreeAsync(d_i0, st));

  // 4. lists ------------------------------------------------------------------
  std::vector<uint8_t> hleaf;
  to_host(P, hleaf, P.d_leaf, P.nbox);
  std::vector<int32_t> hlevel;
  to_host(P, hlevel, P.d_level, P.nbox);
  std::vector<int32_t> leaves, s2m;
  for (int64_t b = 0; b < P.nbox; ++b)
    if (hleaf[b]) {
      leaves.push_back((int32_t)b);
      if (hlevel[b] >= 2) s2m.push_back((int32_t)b);
    }
  P.nleaf = (int64_t)leaves.size();
  P.n_s2m = (int64_t)s2m.size();
  P.d_leaf_ids = dalloc<int32_t>(P, P.nleaf);
  P.d_s2m_ids = dalloc<int32_t>(P, P.n_s2m);
  KF_CUDA(cudaMemcpyAsync(P.d_leaf_ids, leaves.data(), P.nleaf * 4, cudaMemcpyHostToDevice, st));
  if (P.n_s2m) KF_CUDA(cudaMemcpyAsync(P.d_s2m_ids, s2m.data(), P.n_s2m * 4, cudaMemcpyHostToDevice, st));

  std::vector<int64_t> hlbeg(P.depth + 2);
  for (int l = 0; l <= P.depth; ++l) hlbeg[l] = P.levels[l].begin;
  hlbeg[P.depth + 1] = P.nbox;
  int64_t* d_lbeg = dalloc<int64_t>(P, P.depth + 2);
  KF_CUDA(cudaMemcpyAsync(d_lbeg, hlbeg.data(), (P.depth + 2) * 8, cudaMemcpyHostToDevice, st));
  TreeView T{P.d_level, P.d_ijk, P.d_parent, P.d_child, P.d_leaf, P.d_key, d_lbeg, P.depth};

  // U / W
  {
    int64_t *ucnt, *wcnt;
    KF_CUDA(cudaMallocAsync(&ucnt, (P.nleaf + 1) * 8, st));
    KF_CUDA(cudaMallocAsync(&wcnt, (P.nleaf + 1) * 8, st));
    KF_CUDA(cudaMemsetAsync(ucnt, 0, (P.nleaf + 1) * 8, st));
    KF_CUDA(cudaMemsetAsync(wcnt, 0, (P.nleaf + 1) * 8, st));
    k_leaf_lists<<<nblk(P.nleaf, 128), 128, 0, st>>>(T, P.d_leaf_ids, P.nleaf, ucnt, wcnt, nullptr, nullptr, nullptr,
                                                     nullptr);
    KF_CHECK_LAUNCH();
    P.d_u_off = dalloc<int64_t>(P, P.nleaf + 1);
    P.d_w_off = dalloc<int64_t>(P, P.nleaf + 1);
    exclusive_scan(P, ucnt, P.d_u_off, P.nleaf + 1);
    exclusive_scan(P, wcnt, P.d_w_off, P.nleaf + 1);
    KF_CUDA(cudaMemcpyAsync(&P.n_u, P.d_u_off + P.nleaf, 8, cudaMemcpyDeviceToHost, st));
    KF_CUDA(cudaMemcpyAsync(&P.n_w, P.d_w_off + P.nleaf, 8, cudaMemcpyDeviceToHost, st));
    KF_CUDA(cudaStreamSynchronize(st));
    P.d_u_src = dalloc<int32_t>(P, P.n_u);
    P.d_w_src = dalloc<int32_t>(P, P.n_w);
    k_leaf_lists<<<nblk(P.nleaf, 128), 128, 0, st>>>(T, P.d_leaf_ids, P.nleaf, nullptr, nullptr, P.d_u_off,
                                                     P.d_w_off, P.d_u_src, P.d_w_src);
    KF_CHECK_LAUNCH();
    KF_CUDA(cudaFreeAsync(ucnt, st));
    KF_CUDA(cudaFreeAsync(wcnt, st));
  }
  // X = transpose of W, grouped by target box
  {
    P.n_xbox = 0;
    if (P.n_w > 0) {
      int32_t *xk, *xv, *xk2;
      KF_CUDA(cudaMallocAsync(&xk, P.n_w * 4, st));
      KF_CUDA(cudaMallocAsync(&xv, P.n_w * 4, st));
      KF_CUDA(cudaMallocAsync(&xk2, P.n_w * 4, st));
      P.d_x_src = dalloc<int32_t>(P, P.n_w);
      k_x_pairs<<<nblk(P.nleaf), 256, 0, st>>>(P.d_leaf_ids, P.nleaf, P.d_w_off, P.d_w_src, xk, xv);
      KF_CHECK_LAUNCH();
      size_t tmp = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, tmp, xk, xk2, xv, P.d_x_src, P.n_w, 0, 32, st);
      void* d_tmp;
      KF_CUDA(cudaMallocAsync(&d_tmp, tmp + 8, st));
      cub::DeviceRadixSort::SortPairs(d_tmp, tmp, xk, xk2, xv, P.d_x_src, P.n_w, 0, 32, st);
      KF_CUDA(cudaFreeAsync(d_tmp, st));
      std::vector<int32_t> hk;
      to_host(P, hk, xk2, P.n_w);
      std::vector<int32_t> tg;
      std::vector<int64_t> of;
      for (int64_t e = 0; e < P.n_w; ++e)
        if (e == 0 || hk[e] != hk[e - 1]) {
          tg.push_back(hk[e]);
          of.push_back(e);
        }
      of.push_back(P.n_w);
      P.n_xbox = (int64_t)tg.size();
      P.d_x_tgt = dalloc<int32_t>(P, P.n_xbox);
      P.d_x_off = dalloc<int64_t>(P, P.n_xbox + 1);
      KF_CUDA(cudaMemcpyAsync(P.d_x_tgt, tg.data(), P.n_xbox * 4, cudaMemcpyHostToDevice, st));
      KF_CUDA(cudaMemcpyAsync(P.d_x_off, of.data(), (P.n_xbox + 1) * 8, cudaMemcpyHostToDevice, st));
      KF_CUDA(cudaFreeAsync(xk, st));
      KF_CUDA(cudaFreeAsync(xv, st));
      KF_CUDA(cudaFreeAsync(xk2, st));
      KF_CUDA(cudaStreamSynchronize(st));
    }
  }
  // V pairs for boxes at level >= 2, sorted by (level, offset)
  {
    int16_t tab[343];
    int id = 0;
    for (int a = 0; a < 343; ++a) {
      int ox = a / 49 - 3, oy = (a / 7) % 7 - 3, oz = a % 7 - 3;
      tab[a] = (std::max(std::abs(ox), std::max(std::abs(oy), std::abs(oz))) >= 2) ? (int16_t)id++ : (int16_t)-1;
    }
    KF_CUDA(cudaMemcpyToSymbol(c_offset_id, tab, sizeof(tab)));
    P.n_v = 0;
    if (P.depth >= 2) {
      int64_t b0 = P.levels[2].begin, b1 = P.nbox, nb = b1 - b0;
      int64_t *vcnt, *voff;
      KF_CUDA(cudaMallocAsync(&vcnt, (nb + 1) * 8, st));
      KF_CUDA(cudaMallocAsync(&voff, (nb + 1) * 8, st));
      KF_CUDA(cudaMemsetAsync(vcnt, 0, (nb + 1) * 8, st));
      k_v_lists<<<nblk(nb), 256, 0, st>>>(T, b0, b1, vcnt, nullptr, nullptr, nullptr);
      KF_CHECK_LAUNCH();
      exclusive_scan(P, vcnt, voff, nb + 1);
      KF_CUDA(cudaMemcpyAsync(&P.n_v, voff + nb, 8, cudaMemcpyDeviceToHost, st));
      KF_CUDA(cudaStreamSynchronize(st));
      if (P.n_v > 0) {
        int2* pr;
        int32_t *ky, *ky2;
        KF_CUDA(cudaMallocAsync(&pr, P.n_v * 8, st));
        KF_CUDA(cudaMallocAsync(&ky, P.n_v * 4, st));
        KF_CUDA(cudaMallocAsync(&ky2, P.n_v * 4, st));
        P.d_v_pairs = dalloc<int2>(P, P.n_v);
        k_v_lists<<<nblk(nb), 256, 0, st>>>(T, b0, b1, nullptr, voff, pr, ky);
        KF_CHECK_LAUNCH();
        size_t tmp = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tmp, ky, ky2, (uint64_t*)pr, (uint64_t*)P.d_v_pairs, P.n_v, 0, 32,
                                        st);
        void* d_tmp;
        KF_CUDA(cudaMallocAsync(&d_tmp, tmp + 8, st));
        cub::DeviceRadixSort::SortPairs(d_tmp, tmp, ky, ky2, (uint64_t*)pr, (uint64_t*)P.d_v_pairs, P.n_v, 0, 32, st);
        KF_CUDA(cudaFreeAsync(d_tmp, st));
        std::vector<int32_t> hk;
        to_host(P, hk, ky2, P.n_v);
        // M2L tiles: runs of equal (level, offset), chunked by GEMM_BN
        GemmBatch& g = P.g_m2l;
        g.h_tiles.clear();
        int64_t e = 0;
        while (e < P.n_v) {
          int64_t f = e;
          while (f < P.n_v && hk[f] == hk[e]) ++f;
          int lev = hk[e] / N_OFFSETS, off = hk[e] % N_OFFSETS;
          for (int64_t s = e; s < f; s += GEMM_BN)
            g.h_tiles.push_back({off, (int)s, (int)std::min<int64_t>(GEMM_BN, f - s), 0, std::ldexp(1.0, lev)});
          e = f;
        }
        g.n_items = P.n_v;
        g.d_items = P.d_v_pairs;
        g.owns_items = false;
        g.d_tiles = dalloc<GemmTile>(P, g.h_tiles.size());
        KF_CUDA(cudaMemcpyAsync(g.d_tiles, g.h_tiles.data(), g.h_tiles.size() * sizeof(GemmTile),
                                cudaMemcpyHostToDevice, st));
        KF_CUDA(cudaFreeAsync(pr, st));
        KF_CUDA(cudaFreeAsync(ky, st));
        KF_CUDA(cudaFreeAsync(ky2, st));
        KF_CUDA(cudaStreamSynchronize(st));
      }
      KF_CUDA(cudaFreeAsync(vcnt, st));
      KF_CUDA(cudaFreeAsync(voff, st));
    }
  }
  // P2P interaction count (for the flop accounting)
  {
    std::vector<int64_t> uoff, pb, pe;
    std::vector<int32_t> usrc;
    to_host(P, uoff, P.d_u_off, P.nleaf + 1);
    to_host(P, usrc, P.d_u_src, P.n_u);
    to_host(P, pb, P.d_pbeg, P.nbox);
    to_host(P, pe, P.d_pend, P.nbox);
    int64_t tot = 0;
    for (int64_t s = 0; s < P.nleaf; ++s) {
      int64_t nt = pe[leaves[s]] - pb[leaves[s]];
      int64_t ns = 0;
      for (int64_t e = uoff[s]; e < uoff[s + 1]; ++e) ns += pe[usrc[e]] - pb[usrc[e]];
      tot += nt * ns;
    }
    P.n_p2p = tot;
    // merged source point ranges of the P2P (U) and S2L (X) streams: the
    // sources of adjacent Morton leaves are contiguous in the sorted points
    std::vector<int2> rng;
    std::vector<int64_t> roff;
    merged_ranges(uoff, usrc, pb, pe, P.nleaf, rng, roff);
    P.d_u_rng = dalloc<int2>(P, std::max<size_t>(1, rng.size()));
    P.d_u_roff = dalloc<int64_t>(P, roff.size());
    if (!rng.empty()) KF_CUDA(cudaMemcpyAsync(P.d_u_rng, rng.data(), rng.size() * 8, cudaMemcpyHostToDevice, st));
    KF_CUDA(cudaMemcpyAsync(P.d_u_roff, roff.data(), roff.size() * 8, cudaMemcpyHostToDevice, st));
    KF_CUDA(cudaStreamSynchronize(st));
    if (P.n_xbox > 0) {
      std::vector<int64_t> xoff;
      std::vector<int32_t> xsrc;
      to_host(P, xoff, P.d_x_off, P.n_xbox + 1);
      to_host(P, xsrc, P.d_x_src, P.n_w);
      merged_ranges(xoff, xsrc, pb, pe, P.n_xbox, rng, roff);
      P.d_x_rng = dalloc<int2>(P, std::max<size_t>(1, rng.size()));
      P.d_x_roff = dalloc<int64_t>(P, roff.size());
      if (!rng.empty()) KF_CUDA(cudaMemcpyAsync(P.d_x_rng, rng.data(), rng.size() * 8, cudaMemcpyHostToDevice, st));
      KF_CUDA(cudaMemcpyAsync(P.d_x_roff, roff.data(), roff.size() * 8, cudaMemcpyHostToDevice, st));
      KF_CUDA(cudaStreamSynchronize(st));
    }
  }
  // the evaluation runs over every box until kafmm_restrict narrows it
  Jobs& J = P.J;
  J.plo = 0;
  J.phi = P.n;
  J.leaf_ids = P.d_leaf_ids;
  J.nleaf = P.nleaf;
  J.w_off = P.d_w_off;
  J.w_src = P.d_w_src;
  J.u_roff = P.d_u_roff;
  J.u_rng = P.d_u_rng;
  J.s2m_ids = P.d_s2m_ids;
  J.ns2m = P.n_s2m;
  J.x_tgt = P.d_x_tgt;
  J.nx = P.n_xbox;
  J.x_roff = P.d_x_roff;
  J.x_rng = P.d_x_rng;
}

// GEMM work lists of the per-box translations -----------------------------
// items are (input box, output box); on a partitioned plan they become heavy rows
void upload_batch(Plan& P, GemmBatch& g, const std::vector<int2>& box_items) {
  std::vector<int2> mapped;
  if (!P.h_row.empty()) {
    mapped.reserve(box_items.size());
    for (const int2& it : box_items) {
      const int2 r = make_int2(P.h_row[it.x], P.h_row[it.y]);
      if (r.x < 0 || r.y < 0) throw Error{KAFMM_ECUDA, "GEMM item on a box without a row (partition bookkeeping)"};
      mapped.push_back(r);
    }
  }
  const std::vector<int2>& items = P.h_row.empty() ? box_items : mapped;
  g.n_items = (int64_t)items.size();
  g.d_items = dalloc<int2>(P, std::max<size_t>(1, items.size()));
  if (!items.empty())
    KF_CUDA(cudaMemcpyAsync(g.d_items, items.data(), items.size() * sizeof(int2), cudaMemcpyHostToDevice, P.stream));
  g.d_tiles = dalloc<GemmTile>(P, std::max<size_t>(1, g.h_tiles.size()));
  if (!g.h_tiles.empty())
    KF_CUDA(cudaMemcpyAsync(g.d_tiles, g.h_tiles.data(), g.h_tiles.size() * sizeof(GemmTile), cudaMemcpyHostToDevice,
                            P.stream));
  KF_CUDA(cudaStreamSynchronize(P.stream));
}

// groups: consecutive runs of items sharing (op, alpha)
static void tiles_for_runs(GemmBatch& g, const std::vector<int2>& items, const std::vector<int>& op,
                           const std::vector<double>& alpha) {
  g.h_tiles.clear();
  size_t e = 0;
  while (e < items.size()) {
    size_t f = e;
    while (f < items.size() && op[f] == op[e] && alpha[f] == alpha[e]) ++f;
    for (size_t s = e; s < f; s += GEMM_BN)
      g.h_tiles.push_back({op[e], (int)s, (int)std::min<size_t>(GEMM_BN, f - s), 0, alpha[e]});
    e = f;
  }
}

void build_gemm_batches(Plan& P) {
  // re-planning (kafmm_restrict): release the previous batches' device lists
  free_batch(P, P.g_uc2ue_1);
  free_batch(P, P.g_uc2ue_2);
  for (auto* v : {&P.g_m2m, &P.g_dc2de_1, &P.g_dc2de_2, &P.g_l2l})
    for (GemmBatch& g : *v) free_batch(P, g);
  std::vector<int32_t> hlevel, hparent, hijk, hleaf_ids, hs2m;
  std::vector<uint8_t> hleaf;
  to_host(P, hlevel, P.d_level, P.nbox);
  to_host(P, hparent, P.d_parent, P.nbox);
  to_host(P, hijk, P.d_ijk, 3 * P.nbox);
  to_host(P, hs2m, P.J.s2m_ids, P.J.ns2m);
  auto oct = [&](int64_t b) { return 4 * (hijk[3 * b] & 1) + 2 * (hijk[3 * b + 1] & 1) + (hijk[3 * b + 2] & 1); };
  auto act = [&](int64_t b) { return P.box_active.empty() || P.box_active[b] != 0; };
  // UC2UE on the S2M leaves (level >= 2), level-major so alpha = 2^-l forms runs
  {
    std::vector<int2> it;
    std::vector<int> op;
    std::vector<double> a1, a2;
    for (int32_t b : hs2m) {
      it.push_back(make_int2(b, b));
      op.push_back(0);
      a1.push_back(1.0);
      a2.push_back(std::ldexp(1.0, -hlevel[b]));
    }
    tiles_for_runs(P.g_uc2ue_1, it, op, a1);
    upload_batch(P, P.g_uc2ue_1, it);
    tiles_for_runs(P.g_uc2ue_2, it, op, a2);
    upload_batch(P, P.g_uc2ue_2, it);
  }
  // M2M per parent level l = depth-1 .. 2: items (child -> parent) grouped by octant
  P.g_m2m.clear();
  for (int l = P.depth - 1; l >= 2; --l) {
    std::vector<std::vector<int2>> by(8);
    for (int64_t c = P.levels[l + 1].begin; c < P.levels[l + 1].end; ++c)
      if (act(c)) by[oct(c)].push_back(make_int2((int)c, hparent[c]));
    std::vector<int2> it;
    std::vector<int> op;
    std::vector<double> al;
    for (int o = 0; o < 8; ++o)
      for (auto& x : by[o]) {
        it.push_back(x);
        op.push_back(o);
        al.push_back(1.0);
      }
    GemmBatch g;
    tiles_for_runs(g, it, op, al);
    upload_batch(P, g, it);
    P.g_m2m.push_back(g);
  }
  // DC2DE and L2L per level 2..depth
  P.g_dc2de_1.clear();
  P.g_dc2de_2.clear();
  P.g_l2l.clear();
  for (int l = 2; l <= P.depth; ++l) {
    std::vector<int2> it;
    std::vector<int> op;
    std::vector<double> a1, a2;
    for (int64_t b = P.levels[l].begin; b < P.levels[l].end; ++b) {
      if (!act(b)) continue;
      it.push_back(make_int2((int)b, (int)b));
      op.push_back(0);
      a1.push_back(1.0);
      a2.push_back(std::ldexp(1.0, -l));
    }
    GemmBatch g1, g2;
    tiles_for_runs(g1, it, op, a1);
    upload_batch(P, g1, it);
    tiles_for_runs(g2, it, op, a2);
    upload_batch(P, g2, it);
    P.g_dc2de_1.push_back(g1);
    P.g_dc2de_2.push_back(g2);
    GemmBatch g3;
    if (l >= 3) {
      std::vector<std::vector<int2>> by(8);
      for (int64_t b = P.levels[l].begin; b < P.levels[l].end; ++b)
        if (act(b)) by[oct(b)].push_back(make_int2(hparent[b], (int)b));
      std::vector<int2> it3;
      std::vector<int> op3;
      std::vector<double> al3;
      for (int o = 0; o < 8; ++o)
        for (auto& x : by[o]) {
          it3.push_back(x);
          op3.push_back(o);
          al3.push_back(1.0);
        }
      tiles_for_runs(g3, it3, op3, al3);
      upload_batch(P, g3, it3);
    }
    P.g_l2l.push_back(g3);
  }
}

}  // namespace kafmm
