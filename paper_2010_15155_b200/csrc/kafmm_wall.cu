// RPY spheres above a no-slip wall by images (
// PAPER.md:729-779, Table X): four free-space KAFMM summations over the
// particles and their mirror images, assembled per target.
//
// Unit-cube embedding: the wall is the plane z = 1/2, particles lie in
// z in (1/2, 1), images at z' = 1 - z (exact in fp64).  Heights above the
// wall are x_3 = z - 1/2.  The point set of every summation is the 2n points
// [particles; images]; targets are the particles (rows 0..n-1).
//   RPY            [f1, f2, 0, b] at y,  [-f1, -f2, 0, b] at y^I         -> u^S, lap u^S
//   LapPGradGrad   [f3, 0, 0, 0] at y,   [-f3, y3 (-f1, -f2, f3)] at y^I  -> phi^SD, grad, hess
//   LapPGradGrad   [y3 f3/2, 0, 0, b^2 f3/6] at y, [-y3 f3/2, 0, 0, b^2 f3/6] at y^I -> phi^SDZ, grad
//   LapQPGradGrad  0 at y,  Q = b^2/3 [[f3,0,0],[0,f3,0],[f1,f2,0]] at y^I (reading R18) -> phi^Q, grad, hess
//   u     = u^S + grad phi^SDZ + x3 (grad phi^SD + grad phi^Q) - [0, 0, phi^SD + phi^Q]
//   lap u = lap u^S + 2 d/dx3 grad (phi^SD + phi^Q)
#include <algorithm>

#include "kafmm_internal.h"

namespace kafmm {

static inline unsigned nblk(int64_t n, int t = 256) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

__global__ void k_wall_points(const double* __restrict__ pts, int64_t n, double* __restrict__ p2, int* flag) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = pts[3 * i], y = pts[3 * i + 1], z = pts[3 * i + 2];
  if (!(z > 0.5 && z < 1.0)) atomicOr(flag, 1);
  p2[3 * i] = x;
  p2[3 * i + 1] = y;
  p2[3 * i + 2] = z;
  p2[3 * (n + i)] = x;
  p2[3 * (n + i) + 1] = y;
  p2[3 * (n + i) + 2] = 1.0 - z;
}

__global__ void k_wall_sources(const double* __restrict__ pts, const double* __restrict__ src, int64_t n,
                               double* __restrict__ v_rpy, double* __restrict__ v_sd, double* __restrict__ v_sdz,
                               double* __restrict__ v_q) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double f1 = src[4 * i], f2 = src[4 * i + 1], f3 = src[4 * i + 2], b = src[4 * i + 3];
  const double y3 = pts[3 * i + 2] - 0.5;
  const int64_t j = n + i;  // image row
  double* r = v_rpy + 4 * i;
  r[0] = f1, r[1] = f2, r[2] = 0.0, r[3] = b;
  r = v_rpy + 4 * j;
  r[0] = -f1, r[1] = -f2, r[2] = 0.0, r[3] = b;
  r = v_sd + 4 * i;
  r[0] = f3, r[1] = 0.0, r[2] = 0.0, r[3] = 0.0;
  r = v_sd + 4 * j;
  r[0] = -f3, r[1] = -y3 * f1, r[2] = -y3 * f2, r[3] = y3 * f3;
  const double b6 = b * b / 6.0, b3 = b * b / 3.0;
  r = v_sdz + 4 * i;
  r[0] = 0.5 * y3 * f3, r[1] = 0.0, r[2] = 0.0, r[3] = b6 * f3;
  r = v_sdz + 4 * j;
  r[0] = -0.5 * y3 * f3, r[1] = 0.0, r[2] = 0.0, r[3] = b6 * f3;
  r = v_q + 9 * i;
  for (int c = 0; c < 9; ++c) r[c] = 0.0;
  r = v_q + 9 * j;
  r[0] = b3 * f3, r[1] = 0.0, r[2] = 0.0;
  r[3] = 0.0, r[4] = b3 * f3, r[5] = 0.0;
  r[6] = b3 * f1, r[7] = b3 * f2, r[8] = 0.0;
}

__global__ void k_wall_assemble(const double* __restrict__ pts, int64_t n, const double* __restrict__ uS,
                                const double* __restrict__ pSD, const double* __restrict__ pSDZ,
                                const double* __restrict__ pQ, double* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x3 = pts[3 * i + 2] - 0.5;
  const double* s = uS + 6 * i;
  const double* d = pSD + 10 * i;
  const double* z = pSDZ + 10 * i;
  const double* q = pQ + 10 * i;
  double* o = out + 6 * i;
  for (int a = 0; a < 3; ++a) o[a] = s[a] + z[1 + a] + x3 * (d[1 + a] + q[1 + a]);
  o[2] -= d[0] + q[0];
  o[3] = s[3] + 2.0 * (d[6] + q[6]);  // d/dx3 grad = (xz, yz, zz)
  o[4] = s[4] + 2.0 * (d[8] + q[8]);
  o[5] = s[5] + 2.0 * (d[9] + q[9]);
}

}  // namespace kafmm

using namespace kafmm;

struct kafmm_wall_s {
  kafmm_plan rpy = nullptr, lap = nullptr, lapq = nullptr;
  int64_t n = 0;
  cudaStream_t stream = 0;
  double *pts = nullptr, *p2 = nullptr, *v_rpy = nullptr, *v_sd = nullptr, *v_sdz = nullptr, *v_q = nullptr;
  double *o_rpy = nullptr, *o_sd = nullptr, *o_sdz = nullptr, *o_q = nullptr;
  int* flag = nullptr;
};

static void wall_free(kafmm_wall_s* W) {
  if (!W) return;
  kafmm_destroy(W->rpy);
  kafmm_destroy(W->lap);
  kafmm_destroy(W->lapq);
  for (void* p : {(void*)W->pts, (void*)W->p2, (void*)W->v_rpy, (void*)W->v_sd, (void*)W->v_sdz, (void*)W->v_q,
                  (void*)W->o_rpy, (void*)W->o_sd, (void*)W->o_sdz, (void*)W->o_q, (void*)W->flag})
    if (p) cudaFree(p);
  delete W;
}

extern "C" {

kafmm_status kafmm_wall_setup(const double* points, int64_t n, int p, int max_pts_per_leaf, kafmm_wall* out) {
  if (out) *out = nullptr;
  if (!points || !out || n < 1 || 2 * n > INT32_MAX || p < 2 || max_pts_per_leaf < 1) {
    set_error("kafmm_wall_setup: invalid argument");
    return KAFMM_EINVAL;
  }
  kafmm_wall_s* W = new kafmm_wall_s();
  W->n = n;
  try {
    KF_CUDA(cudaMalloc(&W->p2, (size_t)2 * n * 3 * 8));
    KF_CUDA(cudaMalloc(&W->pts, (size_t)n * 3 * 8));
    KF_CUDA(cudaMalloc(&W->flag, 4));
    KF_CUDA(cudaMemset(W->flag, 0, 4));
    KF_CUDA(cudaMemcpy(W->pts, points, (size_t)n * 3 * 8, cudaMemcpyDeviceToDevice));
    k_wall_points<<<nblk(n), 256>>>(W->pts, n, W->p2, W->flag);
    KF_CHECK_LAUNCH();
    int h = 0;
    KF_CUDA(cudaMemcpy(&h, W->flag, 4, cudaMemcpyDeviceToHost));
    if (h) throw Error{KAFMM_EDOMAIN, "kafmm_wall_setup: a particle is not strictly above the wall (1/2 < z < 1)"};
    const int64_t n2 = 2 * n;
    KF_CUDA(cudaMalloc(&W->v_rpy, (size_t)n2 * 4 * 8));
    KF_CUDA(cudaMalloc(&W->v_sd, (size_t)n2 * 4 * 8));
    KF_CUDA(cudaMalloc(&W->v_sdz, (size_t)n2 * 4 * 8));
    KF_CUDA(cudaMalloc(&W->v_q, (size_t)n2 * 9 * 8));
    KF_CUDA(cudaMalloc(&W->o_rpy, (size_t)n2 * 6 * 8));
    KF_CUDA(cudaMalloc(&W->o_sd, (size_t)n2 * 10 * 8));
    KF_CUDA(cudaMalloc(&W->o_sdz, (size_t)n2 * 10 * 8));
    KF_CUDA(cudaMalloc(&W->o_q, (size_t)n2 * 10 * 8));
    kafmm_status st;
    if ((st = kafmm_setup(W->p2, n2, KAFMM_RPY, p, max_pts_per_leaf, &W->rpy)) != KAFMM_OK) throw Error{st, kafmm_last_error()};
    if ((st = kafmm_setup(W->p2, n2, KAFMM_LAPLACE_PGRADGRAD, p, max_pts_per_leaf, &W->lap)) != KAFMM_OK)
      throw Error{st, kafmm_last_error()};
    if ((st = kafmm_setup(W->p2, n2, KAFMM_LAPLACE_QPGRADGRAD, p, max_pts_per_leaf, &W->lapq)) != KAFMM_OK)
      throw Error{st, kafmm_last_error()};
  } catch (const Error& e) {
    set_error(e.msg);
    wall_free(W);
    cudaGetLastError();
    return e.st;
  }
  *out = W;
  return KAFMM_OK;
}

kafmm_status kafmm_wall_set_stream(kafmm_wall w, void* stream) {
  if (!w) return KAFMM_EINVAL;
  w->stream = (cudaStream_t)stream;
  kafmm_set_stream(w->rpy, stream);
  kafmm_set_stream(w->lap, stream);
  kafmm_set_stream(w->lapq, stream);
  return KAFMM_OK;
}

kafmm_status kafmm_wall_eval(kafmm_wall w, const double* src_values, double* trg_out) {
  if (!w || !src_values || !trg_out) {
    set_error("kafmm_wall_eval: null argument");
    return KAFMM_EINVAL;
  }
  try {
    const int64_t n = w->n;
    k_wall_sources<<<nblk(n), 256, 0, w->stream>>>(w->pts, src_values, n, w->v_rpy, w->v_sd, w->v_sdz, w->v_q);
    KF_CHECK_LAUNCH();
    kafmm_status st;
    if ((st = kafmm_eval(w->rpy, w->v_rpy, w->o_rpy)) != KAFMM_OK) return st;
    if ((st = kafmm_eval(w->lap, w->v_sd, w->o_sd)) != KAFMM_OK) return st;
    if ((st = kafmm_eval(w->lap, w->v_sdz, w->o_sdz)) != KAFMM_OK) return st;
    if ((st = kafmm_eval(w->lapq, w->v_q, w->o_q)) != KAFMM_OK) return st;
    k_wall_assemble<<<nblk(n), 256, 0, w->stream>>>(w->pts, n, w->o_rpy, w->o_sd, w->o_sdz, w->o_q, trg_out);
    KF_CHECK_LAUNCH();
  } catch (const Error& e) {
    set_error(e.msg);
    return e.st;
  }
  return KAFMM_OK;
}

void kafmm_wall_destroy(kafmm_wall w) { wall_free(w); }

}  // extern "C"
