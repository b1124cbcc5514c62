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
constexpr int SURF_TQ = 6;       // check points per thread per pass (768 >= M at p = 12)

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
                         const int64_t* __restrict__ perm, int64_t n, int ks, int srec, double* __restrict__ rec) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t u = perm[i];
  double r[8];
  r[0] = pts[4 * i];
  r[1] = pts[4 * i + 1];
  r[2] = pts[4 * i + 2];
#pragma unroll
  for (int c = 3; c < 8; ++c) r[c] = 0.0;
  for (int c = 0; c < ks; ++c) r[3 + c] = vals[u * ks + c];
  if (srec == 4) {
    reinterpret_cast<double2*>(rec + 4 * i)[0] = make_double2(r[0], r[1]);
    reinterpret_cast<double2*>(rec + 4 * i)[1] = make_double2(r[2], r[3]);
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) reinterpret_cast<double2*>(rec + 8 * i)[c] = make_double2(r[2 * c], r[2 * c + 1]);
  }
}

// a2 / a6: points -> check surface of a box ------------------------------------
// jobs[j] = target box; sources = the box's own points (src_off == nullptr, S2M)
// or the leaves src_leaf[src_off[j] .. src_off[j+1]) (S2L over the X list).
template <class K, int SREC, bool ADD>
__global__ void __launch_bounds__(PT_THREADS)
    k_points_to_surface(const int32_t* __restrict__ jobs, const int64_t* __restrict__ src_off,
                        const int32_t* __restrict__ src_leaf, const int32_t* __restrict__ level,
                        const int32_t* __restrict__ ijk, const int64_t* __restrict__ pbeg,
                        const int64_t* __restrict__ pend, const double* __restrict__ rec,
                        const double* __restrict__ surf, int M, double alpha, double* __restrict__ out, int ldn) {
  __shared__ __align__(16) double ss[PT_THREADS * SREC];
  const int job = blockIdx.x, tid = threadIdx.x;
  const int b = jobs[job];
  double cx, cy, cz, h;
  box_geom(level, ijk, b, cx, cy, cz, h);
  const double sc = alpha * h;
  const int64_t e0 = src_off ? src_off[job] : 0, e1 = src_off ? src_off[job + 1] : 1;
  for (int tb = 0; tb < M; tb += PT_THREADS * SURF_TQ) {
    double tx[SURF_TQ], ty[SURF_TQ], tz[SURF_TQ], acc[SURF_TQ][K::KT];
#pragma unroll
    for (int q = 0; q < SURF_TQ; ++q) {
      int i = min(tb + tid + PT_THREADS * q, M - 1);
      tx[q] = cx + sc * surf[3 * i];
      ty[q] = cy + sc * surf[3 * i + 1];
      tz[q] = cz + sc * surf[3 * i + 2];
#pragma unroll
      for (int a = 0; a < K::KT; ++a) acc[q][a] = 0.0;
    }
    for (int64_t e = e0; e < e1; ++e) {
      const int leaf = src_off ? src_leaf[e] : b;
      const int64_t p0 = pbeg[leaf], p1 = pend[leaf];
      for (int64_t s0 = p0; s0 < p1; s0 += PT_THREADS) {
        const int cnt = (int)((p1 - s0) < PT_THREADS ? (p1 - s0) : PT_THREADS);
        __syncthreads();
        for (int idx = tid; idx < cnt * SREC; idx += PT_THREADS) ss[idx] = rec[s0 * SREC + idx];
        __syncthreads();
        for (int j = 0; j < cnt; ++j) {
          const double* sr = ss + j * SREC;
          const double sx = sr[0], sy = sr[1], sz = sr[2];
#pragma unroll
          for (int q = 0; q < SURF_TQ; ++q) K::acc(tx[q] - sx, ty[q] - sy, tz[q] - sz, sr + 3, acc[q]);
        }
      }
    }
    double* o = out + (int64_t)b * ldn;
#pragma unroll
    for (int q = 0; q < SURF_TQ; ++q) {
      int i = tb + tid + PT_THREADS * q;
      if (i < M) {
#pragma unroll
        for (int a = 0; a < K::KT; ++a) {
          if (ADD) o[i * K::KT + a] += acc[q][a];
          else o[i * K::KT + a] = acc[q][a];
        }
      }
    }
  }
}

// sliced target/source mapping shared by the leaf kernels: T targets, S slices
struct Slice {
  int T, S, tt, sl;
  __device__ Slice(int nt) {
    T = min(nt, PT_THREADS);
    S = PT_THREADS / max(T, 1);
    tt = threadIdx.x % max(T, 1);
    sl = threadIdx.x / max(T, 1);
  }
};

template <int KT>
__device__ __forceinline__ void slice_reduce_store(const Slice& z, double (&acc)[KT], double* red, double* dst,
                                                   bool add) {
  __syncthreads();
#pragma unroll
  for (int a = 0; a < KT; ++a) red[threadIdx.x * KT + a] = acc[a];
  __syncthreads();
  if (z.sl == 0) {
    for (int s = 1; s < z.S; ++s)
#pragma unroll
      for (int a = 0; a < KT; ++a) acc[a] += red[(s * z.T + z.tt) * KT + a];
#pragma unroll
    for (int a = 0; a < KT; ++a) {
      if (add) dst[z.tt * KT + a] += acc[a];
      else dst[z.tt * KT + a] = acc[a];
    }
  }
}

// a9 + a10: L2T (own downward equivalent, level >= 2) and M2T (W list) ------
template <class K, int SSTR>
__global__ void __launch_bounds__(PT_THREADS)
    k_leaf_far(const int32_t* __restrict__ leaves, const int32_t* __restrict__ level, const int32_t* __restrict__ ijk,
               const int64_t* __restrict__ pbeg, const int64_t* __restrict__ pend, const double* __restrict__ pts,
               const int64_t* __restrict__ w_off, const int32_t* __restrict__ w_src, const double* __restrict__ ue,
               const double* __restrict__ de, int ldn, const double* __restrict__ surf, int M,
               double* __restrict__ outs) {
  __shared__ __align__(16) double ss[PT_THREADS * SSTR];
  __shared__ double red[PT_THREADS * K::KT];
  const int job = blockIdx.x, tid = threadIdx.x;
  const int b = leaves[job];
  const int64_t p0 = pbeg[b], p1 = pend[b];
  const int lb = level[b];
  const int64_t e0 = w_off[job], e1 = w_off[job + 1];
  for (int64_t t0 = p0; t0 < p1; t0 += PT_THREADS) {
    Slice z((int)((p1 - t0) < PT_THREADS ? (p1 - t0) : PT_THREADS));
    const bool act = z.sl < z.S;
    const int64_t ti = t0 + z.tt;
    const double tx = pts[4 * ti], ty = pts[4 * ti + 1], tz = pts[4 * ti + 2];
    double acc[K::KT];
#pragma unroll
    for (int a = 0; a < K::KT; ++a) acc[a] = 0.0;
    for (int64_t e = (lb >= 2 ? e0 - 1 : e0); e < e1; ++e) {
      const bool own = e < e0;
      const int sb = own ? b : w_src[e];
      const double* dens = (own ? de : ue) + (int64_t)sb * ldn;
      double cx, cy, cz, h;
      box_geom(level, ijk, sb, cx, cy, cz, h);
      const double sc = (own ? 2.95 : 1.05) * h;  // ALPHA_DE / ALPHA_UE
      for (int s0 = 0; s0 < M; s0 += PT_THREADS) {
        const int cnt = min(PT_THREADS, M - s0);
        __syncthreads();
        if (tid < cnt) {
          const int i = s0 + tid;
          double* d = ss + tid * SSTR;
          d[0] = cx + sc * surf[3 * i];
          d[1] = cy + sc * surf[3 * i + 1];
          d[2] = cz + sc * surf[3 * i + 2];
#pragma unroll
          for (int a = 0; a < K::KS; ++a) d[3 + a] = dens[i * K::KS + a];
        }
        __syncthreads();
        if (act)
          for (int j = z.sl; j < cnt; j += z.S) {
            const double* sr = ss + j * SSTR;
            K::acc(tx - sr[0], ty - sr[1], tz - sr[2], sr + 3, acc);
          }
      }
    }
    slice_reduce_store<K::KT>(z, acc, red, outs + t0 * K::KT, false);
  }
}

// a11: P2P over the U list ----------------------------------------------------
template <class K, int SREC>
__global__ void __launch_bounds__(PT_THREADS)
    k_p2p(const int32_t* __restrict__ leaves, const int64_t* __restrict__ pbeg, const int64_t* __restrict__ pend,
          const double* __restrict__ rec, const int64_t* __restrict__ u_off, const int32_t* __restrict__ u_src,
          double* __restrict__ outs) {
  __shared__ __align__(16) double ss[PT_THREADS * SREC];
  __shared__ double red[PT_THREADS * K::KT];
  const int job = blockIdx.x, tid = threadIdx.x;
  const int b = leaves[job];
  const int64_t p0 = pbeg[b], p1 = pend[b];
  const int64_t e0 = u_off[job], e1 = u_off[job + 1];
  for (int64_t t0 = p0; t0 < p1; t0 += PT_THREADS) {
    Slice z((int)((p1 - t0) < PT_THREADS ? (p1 - t0) : PT_THREADS));
    const bool act = z.sl < z.S;
    const int64_t ti = t0 + z.tt;
    const double tx = rec[SREC * ti], ty = rec[SREC * ti + 1], tz = rec[SREC * ti + 2];
    double acc[K::KT];
#pragma unroll
    for (int a = 0; a < K::KT; ++a) acc[a] = 0.0;
    for (int64_t e = e0; e < e1; ++e) {
      const int sb = u_src[e];
      const int64_t q0 = pbeg[sb], q1 = pend[sb];
      for (int64_t s0 = q0; s0 < q1; s0 += PT_THREADS) {
        const int cnt = (int)((q1 - s0) < PT_THREADS ? (q1 - s0) : PT_THREADS);
        __syncthreads();
        for (int idx = tid; idx < cnt * SREC; idx += PT_THREADS) ss[idx] = rec[s0 * SREC + idx];
        __syncthreads();
        if (act)
          for (int j = z.sl; j < cnt; j += z.S) {
            const double* sr = ss + j * SREC;
            K::acc(tx - sr[0], ty - sr[1], tz - sr[2], sr + 3, acc);
          }
      }
    }
    slice_reduce_store<K::KT>(z, acc, red, outs + t0 * K::KT, true);
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

__global__ void k_check_values(const double* __restrict__ v, int64_t n, int ks, int* flag) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * ks) return;
  double x = v[t];
  if (!isfinite(x)) atomicOr(flag, 2);
  if (ks == 4 && (t % 4) == 3 && x < 0.0) atomicOr(flag, 2);
}

// ---------------------------------------------------------------------------
static inline unsigned nblk(int64_t n, int t = 256) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

template <class KS, class KT_, class KST, int SREC>
static void eval_impl(Plan& P, const double* d_src, double* d_out) {
  cudaStream_t st = P.stream;
  auto mark = [&](int s) {
    if (P.timing) KF_CUDA(cudaEventRecord(P.ev[s], st));
  };
  P.launches = 0;
  mark(ST_GATHER);
  k_gather<<<nblk(P.n), 256, 0, st>>>(d_src, P.d_pts, P.d_perm, P.n, P.ks, SREC, P.d_rec);
  KF_CHECK_LAUNCH();
  P.launches++;
  KF_CUDA(cudaMemsetAsync(P.d_ue, 0, (size_t)P.nbox * P.ldn * 8, st));
  mark(ST_S2M);
  if (P.n_s2m > 0) {
    k_points_to_surface<KS, SREC, false><<<(unsigned)P.n_s2m, PT_THREADS, 0, st>>>(
        P.d_s2m_ids, nullptr, nullptr, P.d_level, P.d_ijk, P.d_pbeg, P.d_pend, P.d_rec, P.d_surf, P.M, ALPHA_UC,
        P.d_chk, P.ldn);
    KF_CHECK_LAUNCH();
    P.launches++;
  }
  mark(ST_UC2UE);
  launch_gemm(P, P.g_uc2ue_1, P.d_W1, P.kept_up, P.ldn, P.ldn, P.d_chk, P.ldn, P.d_t, P.ldk, GEMM_STORE);
  launch_gemm(P, P.g_uc2ue_2, P.d_W2, P.neq, P.ldk, P.ldk, P.d_t, P.ldk, P.d_ue, P.ldn, GEMM_STORE);
  mark(ST_M2M);
  for (auto& g : P.g_m2m) launch_gemm(P, g, P.d_m2m, P.neq, P.ldn, P.ldn, P.d_ue, P.ldn, P.d_ue, P.ldn, GEMM_ATOMIC);
  KF_CUDA(cudaMemsetAsync(P.d_chk, 0, (size_t)P.nbox * P.ldn * 8, st));
  mark(ST_M2L);
  if (P.m2l_mode == M2L_FFT)
    run_m2l_fft(P);
  else
    launch_gemm(P, P.g_m2l, P.d_m2l, P.neq, P.ldn, P.ldn, P.d_ue, P.ldn, P.d_chk, P.ldn, GEMM_ATOMIC);
  mark(ST_S2L);
  if (P.n_xbox > 0) {
    k_points_to_surface<KS, SREC, true><<<(unsigned)P.n_xbox, PT_THREADS, 0, st>>>(
        P.d_x_tgt, P.d_x_off, P.d_x_src, P.d_level, P.d_ijk, P.d_pbeg, P.d_pend, P.d_rec, P.d_surf, P.M, ALPHA_DC,
        P.d_chk, P.ldn);
    KF_CHECK_LAUNCH();
    P.launches++;
  }
  mark(ST_DC2DE);
  float l2l_ms = 0.0f;
  for (int l = 2; l <= P.depth; ++l) {
    int i = l - 2;
    launch_gemm(P, P.g_dc2de_1[i], P.d_D1, P.kept_dn, P.ldn, P.ldn, P.d_chk, P.ldn, P.d_t, P.ldk, GEMM_STORE);
    launch_gemm(P, P.g_dc2de_2[i], P.d_D2, P.neq, P.ldk, P.ldk, P.d_t, P.ldk, P.d_de, P.ldn, GEMM_STORE);
    if (l >= 3) launch_gemm(P, P.g_l2l[i], P.d_l2l, P.neq, P.ldn, P.ldn, P.d_de, P.ldn, P.d_de, P.ldn, GEMM_ADD);
  }
  (void)l2l_ms;
  mark(ST_L2L);  // L2L is interleaved with DC2DE per level; its own slot stays empty
  mark(ST_LEAF_FAR);
  k_leaf_far<KT_, 8><<<(unsigned)P.nleaf, PT_THREADS, 0, st>>>(P.d_leaf_ids, P.d_level, P.d_ijk, P.d_pbeg,
                                                                P.d_pend, P.d_pts, P.d_w_off, P.d_w_src, P.d_ue,
                                                                P.d_de, P.ldn, P.d_surf, P.M, P.d_outs);
  KF_CHECK_LAUNCH();
  P.launches++;
  mark(ST_P2P);
  k_p2p<KST, SREC><<<(unsigned)P.nleaf, PT_THREADS, 0, st>>>(P.d_leaf_ids, P.d_pbeg, P.d_pend, P.d_rec, P.d_u_off,
                                                             P.d_u_src, P.d_outs);
  KF_CHECK_LAUNCH();
  P.launches++;
  mark(ST_SCATTER);
  const double scale = (P.kernel == KAFMM_LAPLACE_PGRAD) ? 1.0 / (4.0 * M_PI) : 1.0 / (8.0 * M_PI);
  k_scatter<<<nblk(P.n * P.kt), 256, 0, st>>>(P.d_outs, P.d_perm, P.n, P.kt, scale, d_out);
  KF_CHECK_LAUNCH();
  P.launches++;
  mark(ST_TOTAL);
}

void run_eval(Plan& P, const double* d_src, double* d_out) {
  switch (P.kernel) {
    case KAFMM_LAPLACE_PGRAD: eval_impl<KL, KLG, KLG, 4>(P, d_src, d_out); break;
    case KAFMM_STOKESLET: eval_impl<KG, KG, KG, 8>(P, d_src, d_out); break;
    case KAFMM_RPY: eval_impl<KRPY, KGL, KRPYL, 8>(P, d_src, d_out); break;
    case KAFMM_STOKES_REG_VEL: eval_impl<KGE, KG, KGE, 8>(P, d_src, d_out); break;
    default: throw Error{KAFMM_EINVAL, "unknown kernel"};
  }
}

void check_values(Plan& P, const double* d_src) {
  KF_CUDA(cudaMemsetAsync(P.d_flag, 0, 4, P.stream));
  k_check_values<<<nblk(P.n * P.ks), 256, 0, P.stream>>>(d_src, P.n, P.ks, P.d_flag);
  KF_CHECK_LAUNCH();
  int h = 0;
  KF_CUDA(cudaMemcpyAsync(&h, P.d_flag, 4, cudaMemcpyDeviceToHost, P.stream));
  KF_CUDA(cudaStreamSynchronize(P.stream));
  if (h) throw Error{KAFMM_ENONFINITE, "non-finite source value or negative b/eps"};
}

}  // namespace kafmm
