// The evaluation pass (hot path), SURVEY.md §8(a) rows a1-a12:
//   a1 gather_src     permute source values into Morton order, fused with the
//                     sorted coordinates into 32/64-byte source records
//   a2 S2M            leaf sources -> upward check surface (S-row kernel)
//   a3 UC2UE          two-factor check->equivalent            (kafmm_gemm.cu)
//   a4 M2M            composed, bottom-up                       (kafmm_gemm.cu)
//   a5 M2L            V list, raw kernel matrices               (kafmm_gemm.cu)
//   a6 S2L            X list, sources -> downward check surface (S-row kernel)
//   a7 DC2DE          two-factor, per level                     (kafmm_gemm.cu)
//   a8 L2L            composed, top-down                        (kafmm_gemm.cu)
//   a9/a10 L2T + M2T  downward equivalents of the leaf and W-list upward
//                     equivalents -> targets (T-column kernel)
//   a11 P2P           U list direct sum (S2T kernel)
//   a12 scatter_out   un-permute, apply 1/(4 pi) or 1/(8 pi)
// Kernel tables: PAPER.md Table I (158-171), Table IV (292-305), Table V (337-349).
#include <cmath>

#include "kafmm_internal.h"
#include "kafmm_kernels.cuh"

namespace kafmm {

constexpr int PT_THREADS = 128;  // pointwise kernels

__device__ __forceinline__ void box_geom(const int32_t* __restrict__ level, const int32_t* __restrict__ ijk, int b,
                                         double& cx, double& cy, double& cz, double& h) {
  int l = level[b];
  h = ldexp(0.5, -l);  // half-width 2^-(l+1); centre (ijk + 1/2) 2^-l, exact in fp64
  double w = 2.0 * h;
  cx = (ijk[3 * b] + 0.5) * w;
  cy = (ijk[3 * b + 1] + 0.5) * w;
  cz = (ijk[3 * b + 2] + 0.5) * w;
}

// a1 ------------------------------------------------------------------------
__global__ void k_gather(const double* __restrict__ vals, const double* __restrict__ pts,
                         const int64_t* __restrict__ perm, int64_t n, int ks, int srec, int sqcol,
                         double* __restrict__ rec, int* __restrict__ nonfinite) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t u = perm[i];
  double r[12];
  r[0] = pts[4 * i];
  r[1] = pts[4 * i + 1];
  r[2] = pts[4 * i + 2];
#pragma unroll
  for (int c = 3; c < 12; ++c) r[c] = 0.0;
  bool bad = false;
  for (int c = 0; c < ks; ++c) {
    r[3 + c] = vals[u * ks + c];
    bad |= !isfinite(r[3 + c]);
  }
  if (sqcol >= 0) bad |= r[3 + sqcol] < 0.0;
  if (bad) atomicOr(nonfinite, 1);  // sticky; reported by kafmm_sync / kafmm_eval_host (ENONFINITE)
  // the radius b (RPY) or blob size eps (regularised kernels) enters every pair only
  // squared: the record carries the square, formed once per source here
  if (sqcol >= 0) r[3 + sqcol] *= r[3 + sqcol];
  double2* o = reinterpret_cast<double2*>(rec + (int64_t)srec * i);
#pragma unroll
  for (int c = 0; c < 6; ++c)
    if (2 * c < srec) o[c] = make_double2(r[2 * c], r[2 * c + 1]);
}

// Source streaming shared by the pointwise kernels: the CTA walks a list of
// point ranges (or generated surface points), copies them into one shared
// chunk of CH records and runs the pair loop once per full chunk, so a
// __syncthreads pair is paid per CH sources instead of per source leaf.
constexpr int STREAM_DOUBLES = 2048;  // 16 KB of shared memory per CTA

// copy `take` records of SREC doubles from rec[a ..] to chunk slot `fill`
template <int SREC>
__device__ __forceinline__ void copy_records(double* __restrict__ ss, int fill, const double* __restrict__ rec,
                                             int64_t a, int take) {
  const double2* g = reinterpret_cast<const double2*>(rec + a * SREC);
  double2* s = reinterpret_cast<double2*>(ss + fill * SREC);
  for (int idx = threadIdx.x; idx < take * (SREC / 2); idx += blockDim.x) s[idx] = g[idx];
}

// a2 / a6: points -> check surface of a box ------------------------------------
// jobs[j] = target box; sources = the box's own points (roff == nullptr, S2M)
// or the merged point ranges rng[roff[j] .. roff[j+1]) of its X list (S2L).
// TQ check points per thread (TQ * PT_THREADS >= M).
template <class K, int SREC, int TQ, bool ADD, int NTH>
__global__ void __launch_bounds__(NTH)
    k_points_to_surface(const int32_t* __restrict__ jobs, const int64_t* __restrict__ roff,
                        const int2* __restrict__ rng, const int32_t* __restrict__ level,
                        const int32_t* __restrict__ ijk, const int64_t* __restrict__ pbeg,
                        const int64_t* __restrict__ pend, const double* __restrict__ rec,
                        const double* __restrict__ surf, int M, double alpha, double* __restrict__ out, int ldn,
                        const int32_t* __restrict__ row) {
  constexpr int CH = STREAM_DOUBLES / SREC;
  __shared__ __align__(16) double ss[CH * SREC];
  const int job = blockIdx.x, tid = threadIdx.x;
  const int b = jobs[job];
  double cx, cy, cz, h;
  box_geom(level, ijk, b, cx, cy, cz, h);
  const double sc = alpha * h;
  double tx[TQ], ty[TQ], tz[TQ], acc[TQ][K::KT];
#pragma unroll
  for (int q = 0; q < TQ; ++q) {
    int i = min(tid + NTH * q, M - 1);
    tx[q] = cx + sc * surf[3 * i];
    ty[q] = cy + sc * surf[3 * i + 1];
    tz[q] = cz + sc * surf[3 * i + 2];
#pragma unroll
    for (int a = 0; a < K::KT; ++a) acc[q][a] = 0.0;
  }
  auto run = [&](int cnt) {
    __syncthreads();
    for (int j = 0; j < cnt; ++j) {
      const double* sr = ss + j * SREC;
      const double sx = sr[0], sy = sr[1], sz = sr[2];
#pragma unroll
      for (int q = 0; q < TQ; ++q) K::acc(tx[q] - sx, ty[q] - sy, tz[q] - sz, sr + 3, acc[q]);
    }
    __syncthreads();
  };
  const int64_t r0 = roff ? roff[job] : 0, r1 = roff ? roff[job + 1] : 1;
  int fill = 0;
  for (int64_t r = r0; r < r1; ++r) {
    int64_t a, e;
    if (roff) {
      const int2 g = rng[r];
      a = g.x;
      e = g.y;
    } else {
      a = pbeg[b];
      e = pend[b];
    }
    while (a < e) {
      const int take = (int)min((int64_t)(CH - fill), e - a);
      copy_records<SREC>(ss, fill, rec, a, take);
      fill += take;
      a += take;
      if (fill == CH) {
        run(CH);
        fill = 0;
      }
    }
  }
  if (fill) run(fill);
  double* o = out + (int64_t)(row ? row[b] : b) * ldn;
#pragma unroll
  for (int q = 0; q < TQ; ++q) {
    int i = tid + NTH * q;
    if (i < M) {
#pragma unroll
      for (int a = 0; a < K::KT; ++a) {
        if (ADD) o[i * K::KT + a] += acc[q][a];
        else o[i * K::KT + a] = acc[q][a];
      }
    }
  }
}

// Target/source mapping of the leaf kernels: a pass covers up to TP x 128
// targets; every thread holds TP targets (t = i NTT + tt, i < TP) and walks
// source slice sl of S, so ceil(nt / TP) x S threads are busy (>= 94% for
// leaves of 30-128 points at TP = 4) and each shared-memory source read
// feeds TP pairs.
// TP = 4 for kernels with up to 4 outputs, 2 above (registers)
template <class K>
struct TPof {
  static constexpr int v = K::KT <= 4 ? 4 : 2;
};

template <int TP>
struct Tile {
  int nt, NTT, S, tt, sl;
  bool act;
  __device__ Tile(int n) {
    nt = n;
    NTT = (n + TP - 1) / TP;
    S = PT_THREADS / max(NTT, 1);
    tt = threadIdx.x % max(NTT, 1);
    sl = threadIdx.x / max(NTT, 1);
    act = sl < S;
  }
};

// sum the slices of every target (shared fp64 atomics into the free source
// chunk, one target slot i at a time) and store / add to dst[t * KT + a]
template <int TP, int KT>
__device__ __forceinline__ void tile_reduce_store(const Tile<TP>& z, double (&acc)[TP][KT], double* red, double* dst,
                                                  bool add) {
  for (int i = 0; i < TP; ++i) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < z.NTT * KT; idx += PT_THREADS) red[idx] = 0.0;
    __syncthreads();
    if (z.act && i * z.NTT + z.tt < z.nt) {
#pragma unroll
      for (int a = 0; a < KT; ++a) atomicAdd(&red[z.tt * KT + a], acc[i][a]);
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < z.NTT * KT; idx += PT_THREADS) {
      if (i * z.NTT + idx / KT < z.nt) {
        double* d = dst + (int64_t)i * z.NTT * KT + idx;
        if (add) *d += red[idx];
        else *d = red[idx];
      }
    }
  }
  __syncthreads();  // red aliases the source chunk the next pass refills
}

// pair loop over a chunk of cnt staged sources (SSTR doubles each); with one
// target per thread two interleaved accumulator sets give independent chains
template <class K, int SSTR, int TP>
__device__ __forceinline__ void tile_pairs(const Tile<TP>& z, const double* ss, int cnt, const double (&tx)[TP],
                                           const double (&ty)[TP], const double (&tz)[TP], double (&acc)[TP][K::KT],
                                           double (&acc2)[K::KT]) {
  if (!z.act) return;
  int j = z.sl;
  if (TP == 1) {
    for (; j + z.S < cnt; j += 2 * z.S) {
      const double* sr = ss + j * SSTR;
      const double* s2 = sr + z.S * SSTR;
      K::acc(tx[0] - sr[0], ty[0] - sr[1], tz[0] - sr[2], sr + 3, acc[0]);
      K::acc(tx[0] - s2[0], ty[0] - s2[1], tz[0] - s2[2], s2 + 3, acc2);
    }
  }
  for (; j < cnt; j += z.S) {
    const double* sr = ss + j * SSTR;
    const double sx = sr[0], sy = sr[1], sz = sr[2];
#pragma unroll
    for (int i = 0; i < TP; ++i) K::acc(tx[i] - sx, ty[i] - sy, tz[i] - sz, sr + 3, acc[i]);
  }
}

// a9 + a10: L2T (own downward equivalent, level >= 2) and M2T (W list) ------
// Sources are generated surface points (lattice offset x radius + centre) with
// their equivalent densities; SSTR doubles per source in the chunk.
template <class K, int SSTR, int TP>
__global__ void __launch_bounds__(PT_THREADS)
    k_leaf_far(const int32_t* __restrict__ leaves, const int32_t* __restrict__ level, const int32_t* __restrict__ ijk,
               const int64_t* __restrict__ pbeg, const int64_t* __restrict__ pend, const double* __restrict__ pts,
               const int64_t* __restrict__ w_off, const int32_t* __restrict__ w_src, const double* __restrict__ ue,
               const double* __restrict__ de, int ldn, const double* __restrict__ surf, int M,
               double* __restrict__ outs, int add, const int32_t* __restrict__ row) {
  constexpr int CH = STREAM_DOUBLES / SSTR;
  __shared__ __align__(16) double ss[STREAM_DOUBLES];
  const int job = blockIdx.x, tid = threadIdx.x;
  const int b = leaves[job];
  const int64_t p0 = pbeg[b], p1 = pend[b];
  const int lb = level[b];
  const int64_t e0 = w_off[job], e1 = w_off[job + 1];
  for (int64_t t0 = p0; t0 < p1; t0 += TP * PT_THREADS) {
    Tile<TP> z((int)min((int64_t)TP * PT_THREADS, p1 - t0));
    double tx[TP], ty[TP], tz[TP], acc[TP][K::KT], acc2[K::KT];
#pragma unroll
    for (int a = 0; a < K::KT; ++a) acc2[a] = 0.0;
#pragma unroll
    for (int i = 0; i < TP; ++i) {
      const int64_t ti = t0 + min(i * z.NTT + z.tt, z.nt - 1);
      tx[i] = pts[4 * ti];
      ty[i] = pts[4 * ti + 1];
      tz[i] = pts[4 * ti + 2];
#pragma unroll
      for (int a = 0; a < K::KT; ++a) acc[i][a] = 0.0;
    }
    auto run = [&](int cnt) {
      __syncthreads();
      tile_pairs<K, SSTR, TP>(z, ss, cnt, tx, ty, tz, acc, acc2);
      __syncthreads();
    };
    int fill = 0;
    for (int64_t e = (lb >= 2 ? e0 - 1 : e0); e < e1; ++e) {
      const bool own = e < e0;
      const int sb = own ? b : w_src[e];
      const double* dens = (own ? de : ue) + (int64_t)(row ? row[sb] : sb) * ldn;
      double cx, cy, cz, h;
      box_geom(level, ijk, sb, cx, cy, cz, h);
      const double sc = (own ? ALPHA_DE : ALPHA_UE) * h;
      for (int i0 = 0; i0 < M;) {
        const int take = min(CH - fill, M - i0);
        for (int idx = tid; idx < take; idx += PT_THREADS) {
          const int i = i0 + idx;
          double* d = ss + (fill + idx) * SSTR;
          d[0] = cx + sc * surf[3 * i];
          d[1] = cy + sc * surf[3 * i + 1];
          d[2] = cz + sc * surf[3 * i + 2];
#pragma unroll
          for (int a = 0; a < K::KS; ++a) d[3 + a] = dens[i * K::KS + a];
        }
        fill += take;
        i0 += take;
        if (fill == CH) {
          run(CH);
          fill = 0;
        }
      }
    }
    if (fill) run(fill);
#pragma unroll
    for (int a = 0; a < K::KT; ++a) acc[0][a] += acc2[a];
    tile_reduce_store<TP, K::KT>(z, acc, ss, outs + t0 * K::KT, add != 0);
  }
}

// a11: P2P over the U list: merged source ranges streamed through shared memory
template <class K, int SREC, int TP>
__global__ void __launch_bounds__(PT_THREADS)
    k_p2p(const int32_t* __restrict__ leaves, const int64_t* __restrict__ pbeg, const int64_t* __restrict__ pend,
          const double* __restrict__ rec, const int64_t* __restrict__ roff, const int2* __restrict__ rng,
          double* __restrict__ outs, int add) {
  constexpr int CH = STREAM_DOUBLES / SREC;
  __shared__ __align__(16) double ss[STREAM_DOUBLES];
  const int job = blockIdx.x;
  const int b = leaves[job];
  const int64_t p0 = pbeg[b], p1 = pend[b];
  const int64_t r0 = roff[job], r1 = roff[job + 1];
  for (int64_t t0 = p0; t0 < p1; t0 += TP * PT_THREADS) {
    Tile<TP> z((int)min((int64_t)TP * PT_THREADS, p1 - t0));
    double tx[TP], ty[TP], tz[TP], acc[TP][K::KT], acc2[K::KT];
#pragma unroll
    for (int a = 0; a < K::KT; ++a) acc2[a] = 0.0;
#pragma unroll
    for (int i = 0; i < TP; ++i) {
      const int64_t ti = t0 + min(i * z.NTT + z.tt, z.nt - 1);
      tx[i] = rec[SREC * ti];
      ty[i] = rec[SREC * ti + 1];
      tz[i] = rec[SREC * ti + 2];
#pragma unroll
      for (int a = 0; a < K::KT; ++a) acc[i][a] = 0.0;
    }
    auto run = [&](int cnt) {
      __syncthreads();
      tile_pairs<K, SREC, TP>(z, ss, cnt, tx, ty, tz, acc, acc2);
      __syncthreads();
    };
    int fill = 0;
    for (int64_t r = r0; r < r1; ++r) {
      const int2 g = rng[r];
      int64_t a = g.x;
      const int64_t e = g.y;
      while (a < e) {
        const int take = (int)min((int64_t)(CH - fill), e - a);
        copy_records<SREC>(ss, fill, rec, a, take);
        fill += take;
        a += take;
        if (fill == CH) {
          run(CH);
          fill = 0;
        }
      }
    }
    if (fill) run(fill);
#pragma unroll
    for (int a = 0; a < K::KT; ++a) acc[0][a] += acc2[a];
    tile_reduce_store<TP, K::KT>(z, acc, ss, outs + t0 * K::KT, add != 0);
  }
}

// a12 -----------------------------------------------------------------------
__global__ void k_scatter(const double* __restrict__ outs, const int64_t* __restrict__ perm, int64_t n, int kt,
                          double scale, double* __restrict__ out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * kt) return;
  int64_t i = t / kt;
  int c = (int)(t - i * kt);
  out[perm[i] * kt + c] = scale * outs[t];
}

// pcol: column of the per-source parameter (b or eps, must be >= 0), or -1
__global__ void k_check_values(const double* __restrict__ v, int64_t n, int ks, int pcol, int* flag) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * ks) return;
  double x = v[t];
  if (!isfinite(x)) atomicOr(flag, 2);
  if (pcol >= 0 && (t % ks) == pcol && x < 0.0) atomicOr(flag, 2);
}

// ---------------------------------------------------------------------------
static inline unsigned nblk(int64_t n, int t = 256) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

// S2M / S2L launch: NTH threads x TQ check points per thread >= M, chosen so
// few slots idle (p = 8: 64 x 5 = 320 for 296; p = 10: 128 x 4; p = 12: 128 x 6)
template <class K, int SREC, bool ADD>
static void launch_surface(Plan& P, const int32_t* jobs, int64_t njobs, const int64_t* roff, const int2* rng,
                           double alpha) {
#define KF_SURF(TQ, NTH)                                                                                     \
  k_points_to_surface<K, SREC, TQ, ADD, NTH><<<(unsigned)njobs, NTH, 0, P.stream>>>(                       \
      jobs, roff, rng, P.d_level, P.d_ijk, P.d_pbeg, P.d_pend, P.d_rec, P.d_surf, P.M, alpha, P.d_chk, P.ldn, P.d_row)
  const int M = P.M;
  if (M <= 128) KF_SURF(1, 128);
  else if (M <= 256) KF_SURF(2, 128);
  else if (M <= 320) KF_SURF(5, 64);
  else if (M <= 384) KF_SURF(3, 128);
  else if (M <= 512) KF_SURF(4, 128);
  else if (M <= 768) KF_SURF(6, 128);
  else if (M <= 1024) KF_SURF(8, 128);
  else throw Error{KAFMM_EINVAL, "p too large for the surface kernels (M > 1024)"};
#undef KF_SURF
  KF_CHECK_LAUNCH();
  P.launches++;
}

// a11 launch: P2P over the owned leaves on stream s, storing (first writer)
// or adding to the sorted outputs
template <class KST, int SREC>
static void launch_p2p(Plan& P, cudaStream_t s, int add) {
  const Jobs& J = P.J;
  if (J.nleaf <= 0) return;
  constexpr int TPS = TPof<KST>::v;
  if (P.n >= 48 * P.nleaf)
    k_p2p<KST, SREC, TPS><<<(unsigned)J.nleaf, PT_THREADS, 0, s>>>(J.leaf_ids, P.d_pbeg, P.d_pend, P.d_rec,
                                                                   J.u_roff, J.u_rng, P.d_outs, add);
  else
    k_p2p<KST, SREC, 1><<<(unsigned)J.nleaf, PT_THREADS, 0, s>>>(J.leaf_ids, P.d_pbeg, P.d_pend, P.d_rec, J.u_roff,
                                                                 J.u_rng, P.d_outs, add);
  KF_CHECK_LAUNCH();
  P.launches++;
}

// a1-a4: gather, S2M, UC2UE, M2M (upward pass)
template <class KS, class KST, int SREC>
static void eval_up_impl(Plan& P, const double* d_src) {
  cudaStream_t st = P.stream;
  auto mark = [&](int s) {
    if (P.timing == 1 || (P.timing == 2 && (s == ST_GATHER || s == ST_TOTAL))) KF_CUDA(cudaEventRecord(P.ev[s], st));
  };
  const Jobs& J = P.J;
  P.launches = 0;
  mark(ST_GATHER);
  const int sqcol = P.kernel == KAFMM_RPY || P.kernel == KAFMM_STOKES_REG_VEL ? 3
                    : P.kernel == KAFMM_STOKES_REG_VEL_OMEGA        ? 6
                                                                    : -1;
  k_gather<<<nblk(P.nloc), 256, 0, st>>>(d_src, P.d_pts, P.d_perm, P.nloc, P.ks, SREC, sqcol, P.d_rec, P.d_flag + 1);
  KF_CHECK_LAUNCH();
  P.launches++;
  // the near field needs only the gathered records: it runs on a side stream
  // concurrently with the whole far-field chain (stage timing keeps one stream
  // so that every stage's events bracket only its own kernels)
  P.near_async = P.timing != 1 && P.side != nullptr && P.J.nleaf > 0;
  if (P.near_async) {
    KF_CUDA(cudaEventRecord(P.ev_near_in, st));
    KF_CUDA(cudaStreamWaitEvent(P.side, P.ev_near_in, 0));
    launch_p2p<KST, SREC>(P, P.side, 0);
    KF_CUDA(cudaEventRecord(P.ev_near_out, P.side));
  }
  KF_CUDA(cudaMemsetAsync(P.d_ue, 0, (size_t)P.nrow * P.ldn * 8, st));
  mark(ST_S2M);
  if (J.ns2m > 0) launch_surface<KS, SREC, false>(P, J.s2m_ids, J.ns2m, nullptr, nullptr, ALPHA_UC);
  mark(ST_UC2UE);
  launch_gemm(P, P.g_uc2ue_1, P.d_W1, P.kept_up, P.ldn, P.ldn, P.d_chk, P.ldn, P.d_t, P.ldk, GEMM_STORE);
  launch_gemm(P, P.g_uc2ue_2, P.d_W2, P.neq, P.ldk, P.ldk, P.d_t, P.ldk, P.d_ue, P.ldn, GEMM_STORE);
  mark(ST_M2M);
  for (auto& g : P.g_m2m) launch_gemm(P, g, P.d_m2m, P.neq, P.ldn, P.ldn, P.d_ue, P.ldn, P.d_ue, P.ldn, GEMM_ATOMIC);
}

// a5-a12: M2L, S2L, DC2DE + L2L, L2T + M2T, P2P, scatter (downward pass and leaves)
template <class KS, class KT_, class KST, int SREC>
static void eval_down_impl(Plan& P, double* d_out) {
  cudaStream_t st = P.stream;
  auto mark = [&](int s) {
    if (P.timing == 1 || (P.timing == 2 && (s == ST_GATHER || s == ST_TOTAL))) KF_CUDA(cudaEventRecord(P.ev[s], st));
  };
  const Jobs& J = P.J;
  const bool s2l_done = P.s2l_early;
  P.s2l_early = false;
  if (!s2l_done) KF_CUDA(cudaMemsetAsync(P.d_chk, 0, (size_t)P.nrow * P.ldn * 8, st));
  mark(ST_M2L);
  P.prod_used = 0;
  if (P.m2l_mode != M2L_DENSE) {
    run_m2l_fft(P);
  } else {
    prod_mark(P);
    launch_gemm(P, P.g_m2l, P.d_m2l, P.neq, P.ldn, P.ldn, P.d_ue, P.ldn, P.d_chk, P.ldn, GEMM_ATOMIC);
    prod_mark(P);
  }
  mark(ST_S2L);
  if (J.nx > 0 && !s2l_done) launch_surface<KS, SREC, true>(P, J.x_tgt, J.nx, J.x_roff, J.x_rng, ALPHA_DC);
  mark(ST_DC2DE);
  for (int l = 2; l <= P.depth; ++l) {
    int i = l - 2;
    launch_gemm(P, P.g_dc2de_1[i], P.d_D1, P.kept_dn, P.ldn, P.ldn, P.d_chk, P.ldn, P.d_t, P.ldk, GEMM_STORE);
    launch_gemm(P, P.g_dc2de_2[i], P.d_D2, P.neq, P.ldk, P.ldk, P.d_t, P.ldk, P.d_de, P.ldn, GEMM_STORE);
    if (l >= 3) launch_gemm(P, P.g_l2l[i], P.d_l2l, P.neq, P.ldn, P.ldn, P.d_de, P.ldn, P.d_de, P.ldn, GEMM_ADD);
  }
  mark(ST_L2L);  // L2L is interleaved with DC2DE per level; its own slot stays empty
  mark(ST_LEAF_FAR);
  // TP targets per thread pays off for leaves of >= 48 points (C5-like); small
  // leaves keep one target per thread and more source slices
  const bool big = P.nleaf > 0 && P.n >= 48 * P.nleaf;
  constexpr int TPT = TPof<KT_>::v, SST = (3 + KT_::KS + 1) / 2 * 2;
  if (P.near_async) KF_CUDA(cudaStreamWaitEvent(st, P.ev_near_out, 0));  // P2P stored first
  const int far_add = P.near_async ? 1 : 0;
  if (J.nleaf > 0) {
#define KF_FAR(TP)                                                                                             \
  k_leaf_far<KT_, SST, TP><<<(unsigned)J.nleaf, PT_THREADS, 0, st>>>(J.leaf_ids, P.d_level, P.d_ijk, P.d_pbeg,  \
                                                                    P.d_pend, P.d_pts, J.w_off, J.w_src, P.d_ue, \
                                                                    P.d_de, P.ldn, P.d_surf, P.M, P.d_outs, far_add, P.d_row)
    if (big) KF_FAR(TPT);
    else KF_FAR(1);
#undef KF_FAR
    KF_CHECK_LAUNCH();
    P.launches++;
  }
  mark(ST_P2P);
  if (!P.near_async) launch_p2p<KST, SREC>(P, st, 1);
  mark(ST_SCATTER);
  const double scale = (P.kml == 1) ? 1.0 / (4.0 * M_PI) : 1.0 / (8.0 * M_PI);
  const int64_t cnt = (J.phi - J.plo) * P.kt;
  if (cnt > 0) {
    k_scatter<<<nblk(cnt), 256, 0, st>>>(P.d_outs + J.plo * P.kt, P.d_operm + J.plo, J.phi - J.plo, P.kt, scale,
                                         d_out);
    KF_CHECK_LAUNCH();
    P.launches++;
  }
  mark(ST_TOTAL);
}

void run_eval_up(Plan& P, const double* d_src) {
  switch (P.kernel) {
    case KAFMM_LAPLACE_PGRAD: eval_up_impl<KL, KLG, 4>(P, d_src); break;
    case KAFMM_STOKESLET: eval_up_impl<KG, KG, 8>(P, d_src); break;
    case KAFMM_RPY: eval_up_impl<KRPY, KRPYL, 8>(P, d_src); break;
    case KAFMM_STOKES_REG_VEL: eval_up_impl<KGE, KGE, 8>(P, d_src); break;
    case KAFMM_STOKES_REG_VEL_OMEGA: eval_up_impl<KGET, KGETW, 12>(P, d_src); break;
    case KAFMM_LAPLACE_PGRADGRAD: eval_up_impl<KLD, KLDGG, 8>(P, d_src); break;
    case KAFMM_LAPLACE_QPGRADGRAD: eval_up_impl<KLQ, KLQGG, 12>(P, d_src); break;
    default: throw Error{KAFMM_EINVAL, "unknown kernel"};
  }
}

void run_eval_down(Plan& P, double* d_out) {
  switch (P.kernel) {
    case KAFMM_LAPLACE_PGRAD: eval_down_impl<KL, KLG, KLG, 4>(P, d_out); break;
    case KAFMM_STOKESLET: eval_down_impl<KG, KG, KG, 8>(P, d_out); break;
    case KAFMM_RPY: eval_down_impl<KRPY, KGL, KRPYL, 8>(P, d_out); break;
    case KAFMM_STOKES_REG_VEL: eval_down_impl<KGE, KG, KGE, 8>(P, d_out); break;
    case KAFMM_STOKES_REG_VEL_OMEGA: eval_down_impl<KGET, KGO, KGETW, 12>(P, d_out); break;
    case KAFMM_LAPLACE_PGRADGRAD: eval_down_impl<KLD, KLGG, KLDGG, 8>(P, d_out); break;
    case KAFMM_LAPLACE_QPGRADGRAD: eval_down_impl<KLQ, KLGG, KLQGG, 12>(P, d_out); break;
    default: throw Error{KAFMM_EINVAL, "unknown kernel"};
  }
}

// a6 ahead of a5: S2L needs only the gathered source records, so a partitioned
// evaluation issues it before the ghost-multipole exchange completes
template <class KS, int SREC>
static void eval_s2l_impl(Plan& P) {
  KF_CUDA(cudaMemsetAsync(P.d_chk, 0, (size_t)P.nrow * P.ldn * 8, P.stream));
  if (P.J.nx > 0) launch_surface<KS, SREC, true>(P, P.J.x_tgt, P.J.nx, P.J.x_roff, P.J.x_rng, ALPHA_DC);
  P.s2l_early = true;
}

void run_eval_s2l(Plan& P) {
  switch (P.kernel) {
    case KAFMM_LAPLACE_PGRAD: eval_s2l_impl<KL, 4>(P); break;
    case KAFMM_STOKESLET: eval_s2l_impl<KG, 8>(P); break;
    case KAFMM_RPY: eval_s2l_impl<KRPY, 8>(P); break;
    case KAFMM_STOKES_REG_VEL: eval_s2l_impl<KGE, 8>(P); break;
    case KAFMM_STOKES_REG_VEL_OMEGA: eval_s2l_impl<KGET, 12>(P); break;
    case KAFMM_LAPLACE_PGRADGRAD: eval_s2l_impl<KLD, 8>(P); break;
    case KAFMM_LAPLACE_QPGRADGRAD: eval_s2l_impl<KLQ, 12>(P); break;
    default: throw Error{KAFMM_EINVAL, "unknown kernel"};
  }
}

void run_eval(Plan& P, const double* d_src, double* d_out) {
  run_eval_up(P, d_src);
  run_eval_down(P, d_out);
}

// the sticky flag k_gather raises on a non-finite source value or a negative b / eps
// (d_flag[1]); read and cleared by the synchronising entry points
void take_nonfinite(Plan& P) {
  int h = 0;
  KF_CUDA(cudaMemcpyAsync(&h, P.d_flag + 1, 4, cudaMemcpyDeviceToHost, P.stream));
  KF_CUDA(cudaMemsetAsync(P.d_flag + 1, 0, 4, P.stream));
  KF_CUDA(cudaStreamSynchronize(P.stream));
  if (h) throw Error{KAFMM_ENONFINITE, "non-finite source value or negative b/eps in an evaluation since the last sync"};
}

void check_values(Plan& P, const double* d_src) {
  KF_CUDA(cudaMemsetAsync(P.d_flag, 0, 4, P.stream));
  const int pcol = (P.kernel == KAFMM_RPY || P.kernel == KAFMM_STOKES_REG_VEL) ? 3
                   : (P.kernel == KAFMM_STOKES_REG_VEL_OMEGA ? 6 : -1);
  const int64_t rows = P.dist ? P.dist->n_caller : P.n;  // the caller's rows
  k_check_values<<<nblk(rows * P.ks), 256, 0, P.stream>>>(d_src, rows, P.ks, pcol, P.d_flag);
  KF_CHECK_LAUNCH();
  int h = 0;
  KF_CUDA(cudaMemcpyAsync(&h, P.d_flag, 4, cudaMemcpyDeviceToHost, P.stream));
  KF_CUDA(cudaStreamSynchronize(P.stream));
  if (h) throw Error{KAFMM_ENONFINITE, "non-finite source value or negative b/eps"};
}

}  // namespace kafmm
