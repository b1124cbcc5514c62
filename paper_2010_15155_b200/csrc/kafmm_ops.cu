// Setup: equivalent/check surfaces and the translation operators of the ML-tree
// kernel (L or G), built once at the reference level 0 and kept resident in HBM.
//
//   surfaces        PAPER.md:632 (M = 6(m-1)^2+2 lattice-surface points);
//                   radii 1.05 h (up-equivalent, down-check) / 2.95 h (up-check,
//                   down-equivalent), reading R1
//   check->equiv    PAPER.md:140-142 "backward stable SVD": K = U S V^T of
//                   K(uc <- ue), sigma_i > 1e-12 sigma_max kept (reading R2),
//                   applied as two factors S^-1 U^T then V (never an explicit
//                   pseudo-inverse).  K(dc <- de) = K(uc <- ue)^T exactly (both
//                   surface pairs use the same lattice and G(-r) = G(r),
//                   G_ij = G_ji), so its factors are S^-1 V^T and U.
//   M2M[oct]        UC2UE_parent o K(uc_P <- ue_C)
//   L2L[oct]        DC2DE_child  o K(dc_C <- de_P)
//   M2L[o]          raw K(dc_B <- ue_C), C = B + 2h o    (M->L slot)
// Level l: kernel matrices scale by 2^l, check->equivalent factors by 2^-l
// (L and G homogeneous of degree -1); applied as GEMM alpha.
// Kernel constants 1/(4 pi), 1/(8 pi) are left out of every operator and of
// every pointwise kernel and applied once in scatter_out: the equivalent
// densities are invariant under that common scaling.
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "kafmm_internal.h"

namespace kafmm {

#define KF_CUBLAS(call)                                                                     \
  do {                                                                                      \
    cublasStatus_t s_ = (call);                                                             \
    if (s_ != CUBLAS_STATUS_SUCCESS)                                                        \
      throw Error{KAFMM_ECUDA, std::string(#call) + ": cublas status " + std::to_string(s_)}; \
  } while (0)
#define KF_CUSOLVER(call)                                                                     \
  do {                                                                                        \
    cusolverStatus_t s_ = (call);                                                             \
    if (s_ != CUSOLVER_STATUS_SUCCESS)                                                        \
      throw Error{KAFMM_ECUDA, std::string(#call) + ": cusolver status " + std::to_string(s_)}; \
  } while (0)

// K[(i,a),(j,b)] = K_ML(x_i - y_j) without constant; x_i = ct + st u_i, y_j = cs + ss u_j
__global__ void k_fill_matrix(double* K, int ld, int kml, int M, const double* __restrict__ surf, double ctx,
                              double cty, double ctz, double st, double csx, double csy, double csz, double ss) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;  // source point
  int i = blockIdx.y;                             // target point
  if (j >= M) return;
  double rx = (ctx + st * surf[3 * i]) - (csx + ss * surf[3 * j]);
  double ry = (cty + st * surf[3 * i + 1]) - (csy + ss * surf[3 * j + 1]);
  double rz = (ctz + st * surf[3 * i + 2]) - (csz + ss * surf[3 * j + 2]);
  double r2 = rx * rx + ry * ry + rz * rz;
  double ri = rsqrt(r2);
  if (kml == 1) {
    K[(size_t)i * ld + j] = ri;
  } else {
    double ri3 = ri * ri * ri;
    double r[3] = {rx, ry, rz};
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        K[(size_t)(3 * i + a) * ld + 3 * j + b] = (a == b ? ri : 0.0) + r[a] * r[b] * ri3;
  }
}

// factors from gesvd of A = K^T (column-major view of row-major K): K = V_A S U_A^T
// W1 = S^-1 U_K^T = S^-1 V_A^T (rows of VT_A), W2 = V_K = U_A (kept columns)
// D1 = S^-1 U_dc^T = S^-1 U_A^T,   D2 = V_dc = V_A
__global__ void k_factors(int n, int kept, int ldn, int ldk, const double* __restrict__ UA,
                          const double* __restrict__ VTA, const double* __restrict__ S, double* W1, double* W2,
                          double* D1, double* D2) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  int r = blockIdx.y;
  if (c >= n) return;
  if (r < kept) {
    double si = 1.0 / S[r];
    W1[(size_t)r * ldn + c] = VTA[r + (size_t)c * n] * si;
    D1[(size_t)r * ldn + c] = UA[c + (size_t)r * n] * si;
  }
  if (c < kept) {
    // row r of W2 / D2 (r < n)
    W2[(size_t)r * ldk + c] = UA[r + (size_t)c * n];
    D2[(size_t)r * ldk + c] = VTA[c + (size_t)r * n];
  }
}

static std::vector<double> lattice_unit(int p) {
  std::vector<double> u;
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j)
      for (int k = 0; k < p; ++k)
        if (std::min(i, std::min(j, k)) == 0 || std::max(i, std::max(j, k)) == p - 1) {
          u.push_back(-1.0 + 2.0 * i / (p - 1));
          u.push_back(-1.0 + 2.0 * j / (p - 1));
          u.push_back(-1.0 + 2.0 * k / (p - 1));
        }
  return u;
}

static void fill(Plan& P, double* K, int ld, const double ct[3], double st, const double cs[3], double ss) {
  dim3 grid((P.M + 127) / 128, P.M);
  k_fill_matrix<<<grid, 128, 0, P.stream>>>(K, ld, P.kml, P.M, P.d_surf, ct[0], ct[1], ct[2], st, cs[0], cs[1], cs[2],
                                            ss);
  KF_CHECK_LAUNCH();
}

// row-major C (m x n, ldc) = alpha A (m x k, lda) B (k x n, ldb)
static void gemm_rm(cublasHandle_t h, int m, int n, int k, double alpha, const double* A, int lda, const double* B,
                    int ldb, double* C, int ldc) {
  const double beta = 0.0;
  KF_CUBLAS(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, m, k, &alpha, B, ldb, A, lda, &beta, C, ldc));
}

void build_operators(Plan& P) {
  cudaStream_t st = P.stream;
  const int p = P.p, M = P.M, n = P.neq;
  std::vector<double> u = lattice_unit(p);
  if ((int)u.size() != 3 * M) throw Error{KAFMM_EINVAL, "surface size mismatch"};
  P.d_surf = dalloc<double>(P, 3 * M);
  KF_CUDA(cudaMemcpyAsync(P.d_surf, u.data(), u.size() * 8, cudaMemcpyHostToDevice, st));

  const double h0 = 0.5, c0[3] = {0.5, 0.5, 0.5};
  // K(uc <- ue) at level 0, dense n x n (no padding) for the SVD.  The factors depend
  // only on (ML kernel, p), so the process keeps one host copy per pair and later
  // plans upload it instead of re-running gesvd (setup only; the SVD is hundreds of
  // small solver launches)
  double *UA, *VTA, *S;
  KF_CUDA(cudaMallocAsync(&UA, (size_t)n * n * 8, st));
  KF_CUDA(cudaMallocAsync(&VTA, (size_t)n * n * 8, st));
  KF_CUDA(cudaMallocAsync(&S, (size_t)n * 8, st));
  struct SvdHost {
    std::vector<double> ua, vta, s;
  };
  static std::mutex svd_mu;
  static std::map<std::pair<int, int>, SvdHost> svd_cache;
  const std::pair<int, int> svd_key(P.kml, p);
  bool cached = false;
  {
    std::lock_guard<std::mutex> lk(svd_mu);
    auto it = svd_cache.find(svd_key);
    if (it != svd_cache.end()) {
      KF_CUDA(cudaMemcpyAsync(UA, it->second.ua.data(), (size_t)n * n * 8, cudaMemcpyHostToDevice, st));
      KF_CUDA(cudaMemcpyAsync(VTA, it->second.vta.data(), (size_t)n * n * 8, cudaMemcpyHostToDevice, st));
      KF_CUDA(cudaMemcpyAsync(S, it->second.s.data(), (size_t)n * 8, cudaMemcpyHostToDevice, st));
      P.h_sigma = it->second.s;
      KF_CUDA(cudaStreamSynchronize(st));
      cached = true;
    }
  }
  if (!cached) {
    double *K, *work;
    int* info;
    KF_CUDA(cudaMallocAsync(&K, (size_t)n * n * 8, st));
    KF_CUDA(cudaMallocAsync(&info, 8, st));
    fill(P, K, n, c0, ALPHA_UC * h0, c0, ALPHA_UE * h0);
    cusolverDnHandle_t sh;
    KF_CUSOLVER(cusolverDnCreate(&sh));
    KF_CUSOLVER(cusolverDnSetStream(sh, st));
    int lwork = 0;
    KF_CUSOLVER(cusolverDnDgesvd_bufferSize(sh, n, n, &lwork));
    KF_CUDA(cudaMallocAsync(&work, (size_t)lwork * 8 + 8, st));
    KF_CUSOLVER(cusolverDnDgesvd(sh, 'A', 'A', n, n, K, n, S, UA, n, VTA, n, work, lwork, nullptr, info));
    int hinfo = 0;
    P.h_sigma.resize(n);
    KF_CUDA(cudaMemcpyAsync(&hinfo, info, 4, cudaMemcpyDeviceToHost, st));
    KF_CUDA(cudaMemcpyAsync(P.h_sigma.data(), S, n * 8, cudaMemcpyDeviceToHost, st));
    KF_CUDA(cudaStreamSynchronize(st));
    cusolverDnDestroy(sh);
    KF_CUDA(cudaFreeAsync(K, st));
    KF_CUDA(cudaFreeAsync(work, st));
    KF_CUDA(cudaFreeAsync(info, st));
    if (hinfo != 0) throw Error{KAFMM_ECUDA, "gesvd did not converge: info " + std::to_string(hinfo)};
    SvdHost h;
    h.ua.resize((size_t)n * n);
    h.vta.resize((size_t)n * n);
    h.s = P.h_sigma;
    KF_CUDA(cudaMemcpy(h.ua.data(), UA, (size_t)n * n * 8, cudaMemcpyDeviceToHost));
    KF_CUDA(cudaMemcpy(h.vta.data(), VTA, (size_t)n * n * 8, cudaMemcpyDeviceToHost));
    std::lock_guard<std::mutex> lk(svd_mu);
    svd_cache.emplace(svd_key, std::move(h));
  }
  int kept = 0;
  for (int i = 0; i < n; ++i)
    if (P.h_sigma[i] > TAU * P.h_sigma[0]) ++kept;
  P.kept_up = P.kept_dn = kept;
  P.ldk = round_up(kept, GEMM_BK);
  P.rows_pad = round_up(std::max(n, kept), GEMM_BM);
  P.op_stride = (int64_t)P.rows_pad * P.ldn;

  P.d_W1 = dalloc<double>(P, (size_t)P.rows_pad * P.ldn);
  P.d_D1 = dalloc<double>(P, (size_t)P.rows_pad * P.ldn);
  P.d_W2 = dalloc<double>(P, (size_t)P.rows_pad * P.ldk);
  P.d_D2 = dalloc<double>(P, (size_t)P.rows_pad * P.ldk);
  {
    dim3 grid((n + 127) / 128, n);
    k_factors<<<grid, 128, 0, st>>>(n, kept, P.ldn, P.ldk, UA, VTA, S, P.d_W1, P.d_W2, P.d_D1, P.d_D2);
    KF_CHECK_LAUNCH();
  }

  // composed M2M and L2L
  cublasHandle_t bh;
  KF_CUBLAS(cublasCreate(&bh));
  KF_CUBLAS(cublasSetStream(bh, st));
  KF_CUBLAS(cublasSetMathMode(bh, CUBLAS_PEDANTIC_MATH));
  double* tmp;
  KF_CUDA(cudaMallocAsync(&tmp, (size_t)kept * P.ldn * 8, st));
  double* Kp;  // padded n x ldn kernel matrix
  KF_CUDA(cudaMallocAsync(&Kp, (size_t)n * P.ldn * 8, st));
  KF_CUDA(cudaMemsetAsync(Kp, 0, (size_t)n * P.ldn * 8, st));
  P.d_m2m = dalloc<double>(P, 8 * P.op_stride);
  P.d_l2l = dalloc<double>(P, 8 * P.op_stride);
  for (int o = 0; o < 8; ++o) {
    double cc[3] = {c0[0] + 0.5 * h0 * (2.0 * ((o >> 2) & 1) - 1.0), c0[1] + 0.5 * h0 * (2.0 * ((o >> 1) & 1) - 1.0),
                    c0[2] + 0.5 * h0 * (2.0 * (o & 1) - 1.0)};
    // M2M: W2 (n x kept) . (W1 (kept x n) . K(uc_P <- ue_C) (n x n))
    fill(P, Kp, P.ldn, c0, ALPHA_UC * h0, cc, ALPHA_UE * 0.5 * h0);
    gemm_rm(bh, kept, n, n, 1.0, P.d_W1, P.ldn, Kp, P.ldn, tmp, P.ldn);
    gemm_rm(bh, n, n, kept, 1.0, P.d_W2, P.ldk, tmp, P.ldn, P.d_m2m + o * P.op_stride, P.ldn);
    // L2L: 2^-1 D2 . (D1 . K(dc_C <- de_P))
    fill(P, Kp, P.ldn, cc, ALPHA_DC * 0.5 * h0, c0, ALPHA_DE * h0);
    gemm_rm(bh, kept, n, n, 1.0, P.d_D1, P.ldn, Kp, P.ldn, tmp, P.ldn);
    gemm_rm(bh, n, n, kept, 0.5, P.d_D2, P.ldk, tmp, P.ldn, P.d_l2l + o * P.op_stride, P.ldn);
  }
  KF_CUDA(cudaStreamSynchronize(st));
  cublasDestroy(bh);
  KF_CUDA(cudaFreeAsync(UA, st));
  KF_CUDA(cudaFreeAsync(VTA, st));
  KF_CUDA(cudaFreeAsync(S, st));
  KF_CUDA(cudaFreeAsync(tmp, st));
  KF_CUDA(cudaFreeAsync(Kp, st));
  KF_CUDA(cudaStreamSynchronize(st));
}

// raw M2L matrices for the 316 offsets (same enumeration as the list builder),
// only for the dense M2L variant: built on first use (C4: 12.5 GB)
void build_dense_m2l(Plan& P) {
  if (P.d_m2l) return;
  const double h0 = 0.5, c0[3] = {0.5, 0.5, 0.5};
  P.d_m2l = dalloc<double>(P, (size_t)N_OFFSETS * P.op_stride);
  int id = 0;
  for (int a = 0; a < 343; ++a) {
    int ox = a / 49 - 3, oy = (a / 7) % 7 - 3, oz = a % 7 - 3;
    if (std::max(std::abs(ox), std::max(std::abs(oy), std::abs(oz))) < 2) continue;
    double cs[3] = {c0[0] + 2.0 * h0 * ox, c0[1] + 2.0 * h0 * oy, c0[2] + 2.0 * h0 * oz};
    fill(P, P.d_m2l + (size_t)id * P.op_stride, P.ldn, c0, ALPHA_DC * h0, cs, ALPHA_UE * h0);
    ++id;
  }
  KF_CUDA(cudaStreamSynchronize(P.stream));
}

}  // namespace kafmm
