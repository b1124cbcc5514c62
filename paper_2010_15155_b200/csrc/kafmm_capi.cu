// extern "C" boundary of libkafmm.so (include/kafmm.h).  Every entry point
// catches internal errors and turns them into a kafmm_status; the detail
// string is kept per thread for kafmm_last_error().
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include "kafmm_internal.h"

namespace kafmm {
static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

static int dims(int kernel, int* ks, int* kt) {
  switch (kernel) {
    case KAFMM_LAPLACE_PGRAD: *ks = 1; *kt = 4; return 0;
    case KAFMM_STOKESLET: *ks = 3; *kt = 3; return 0;
    case KAFMM_RPY: *ks = 4; *kt = 6; return 0;
    case KAFMM_STOKES_REG_VEL: *ks = 4; *kt = 3; return 0;
    case KAFMM_STOKES_REG_VEL_OMEGA: *ks = 7; *kt = 6; return 0;
    case KAFMM_LAPLACE_PGRADGRAD: *ks = 4; *kt = 10; return 0;
    case KAFMM_LAPLACE_QPGRADGRAD: *ks = 9; *kt = 10; return 0;
    default: return -1;
  }
}

static void free_plan(kafmm_plan_s* P) {
  if (!P) return;
  cudaStreamSynchronize(P->stream);
  if (P->side) cudaStreamSynchronize(P->side);
  if (P->gstream) cudaStreamSynchronize(P->gstream);
  if (P->gexec) cudaGraphExecDestroy(P->gexec);
  for (void* p : P->allocs) cudaFree(p);
  for (auto& e : P->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : P->prod_ev)
    if (e) cudaEventDestroy(e);
  if (P->side) cudaStreamDestroy(P->side);
  if (P->gstream) cudaStreamDestroy(P->gstream);
  if (P->ev_gin) cudaEventDestroy(P->ev_gin);
  if (P->ev_gout) cudaEventDestroy(P->ev_gout);
  if (P->ev_near_in) cudaEventDestroy(P->ev_near_in);
  if (P->ev_near_out) cudaEventDestroy(P->ev_near_out);
  if (P->cstream) {
    cudaStreamSynchronize(P->cstream);
    cudaStreamDestroy(P->cstream);
  }
  if (P->ev_up) cudaEventDestroy(P->ev_up);
  if (P->ev_ghost) cudaEventDestroy(P->ev_ghost);
  delete P->dist;
  delete P;
}
}  // namespace kafmm

using namespace kafmm;

static void collect_stage_times(Plan& P) {
  if (!P.timing) return;
  KF_CUDA(cudaEventSynchronize(P.ev[ST_TOTAL]));
  if (P.timing == 1)
    for (int s = 0; s < ST_TOTAL; ++s) KF_CUDA(cudaEventElapsedTime(&P.stage_ms[s], P.ev[s], P.ev[s + 1]));
  else
    for (int s = 0; s < ST_TOTAL; ++s) P.stage_ms[s] = 0.0f;
  KF_CUDA(cudaEventElapsedTime(&P.stage_ms[ST_TOTAL], P.ev[0], P.ev[ST_TOTAL]));
  float prod = 0.0f;
  for (int i = 0; i + 1 < P.prod_used; i += 2) {
    float t = 0.0f;
    KF_CUDA(cudaEventElapsedTime(&t, P.prod_ev[i], P.prod_ev[i + 1]));
    prod += t;
  }
  P.stage_ms[ST_M2L_PRODUCT] = prod;
}

#define KF_API_BEGIN try {
#define KF_API_END                                 \
  }                                                \
  catch (const Error& e) {                         \
    set_error(e.msg);                              \
    return e.st;                                   \
  }                                                \
  catch (const std::bad_alloc&) {                  \
    set_error("host allocation failed");           \
    return KAFMM_ENOMEM;                           \
  }                                                \
  catch (...) {                                    \
    set_error("unknown internal error");           \
    return KAFMM_ECUDA;                            \
  }

namespace kafmm {
// problem constants of a plan (no device work)
static void init_plan(Plan& P, int kernel, int p, int cap, int64_t n, int ks, int kt) {
  P.kernel = kernel;
  P.p = p;
  P.cap = cap;
  P.n = n;
  P.ks = ks;
  P.kt = kt;
  const bool laplace =
      kernel == KAFMM_LAPLACE_PGRAD || kernel == KAFMM_LAPLACE_PGRADGRAD || kernel == KAFMM_LAPLACE_QPGRADGRAD;
  P.kml = laplace ? 1 : 3;
  P.srec = (3 + ks + 3) / 4 * 4;  // x, y, z + source values, padded to 32 bytes
  P.M = 6 * (p - 1) * (p - 1) + 2;
  P.neq = P.kml * P.M;
  P.ldn = round_up(P.neq, GEMM_BK);
  P.stream = 0;
}

// tree, lists, operators, GEMM batches, FFT M2L tables and chunks
void build_plan_core(Plan& P, const double* points) {
  build_tree_and_lists(P, points);
  build_operators(P);
  build_gemm_batches(P);
  size_t fr = 0, tot = 0;
  KF_CUDA(cudaMemGetInfo(&fr, &tot));
  // spectra budget of the FFT M2L chunks: larger chunks transform fewer halo boxes twice
  int64_t budget = std::min<int64_t>((int64_t)40 << 30, (int64_t)(fr / 3));
  const char* env = getenv("KAFMM_FFT_BUDGET_MB");
  if (env) budget = (int64_t)atoll(env) << 20;
  build_fft_m2l(P, budget);
  const char* m = getenv("KAFMM_M2L");
  if (m && std::string(m) == "dense") P.m2l_mode = M2L_DENSE;
  if (P.m2l_mode == M2L_DENSE) build_dense_m2l(P);
  P.nrow = P.nbox;
  P.d_crow = P.d_child;
  P.nloc = P.n;
  P.d_operm = P.d_perm;
}

// per-evaluation workspaces (sized by rows and local points), streams, events
void alloc_workspaces(Plan& P) {
  P.d_rec = dalloc<double>(P, (size_t)P.nloc * P.srec);
  P.d_outs = dalloc<double>(P, (size_t)P.nloc * P.kt);
  P.d_ue = dalloc<double>(P, (size_t)P.nrow * P.ldn);
  P.d_chk = dalloc<double>(P, (size_t)P.nrow * P.ldn);
  P.d_de = dalloc<double>(P, (size_t)P.nrow * P.ldn);
  P.d_t = dalloc<double>(P, (size_t)P.nrow * P.ldk);
  for (auto& e : P.ev) KF_CUDA(cudaEventCreate(&e));
  KF_CUDA(cudaStreamCreateWithFlags(&P.side, cudaStreamNonBlocking));
  KF_CUDA(cudaStreamCreateWithFlags(&P.gstream, cudaStreamNonBlocking));
  KF_CUDA(cudaEventCreateWithFlags(&P.ev_gin, cudaEventDisableTiming));
  KF_CUDA(cudaEventCreateWithFlags(&P.ev_gout, cudaEventDisableTiming));
  KF_CUDA(cudaEventCreateWithFlags(&P.ev_near_in, cudaEventDisableTiming));
  KF_CUDA(cudaEventCreateWithFlags(&P.ev_near_out, cudaEventDisableTiming));
  KF_CUDA(cudaStreamCreateWithFlags(&P.cstream, cudaStreamNonBlocking));
  KF_CUDA(cudaEventCreateWithFlags(&P.ev_up, cudaEventDisableTiming));
  KF_CUDA(cudaEventCreateWithFlags(&P.ev_ghost, cudaEventDisableTiming));
  KF_CUDA(cudaStreamSynchronize(P.stream));
}
}  // namespace kafmm

extern "C" {

kafmm_status kafmm_kernel_dims(int kernel, int* k_s, int* k_t) {
  int a, b;
  if (dims(kernel, &a, &b) != 0) {
    set_error("unknown kernel");
    return KAFMM_EINVAL;
  }
  if (k_s) *k_s = a;
  if (k_t) *k_t = b;
  return KAFMM_OK;
}


static kafmm_status check_setup_args(int64_t n, int kernel, int p, int max_pts, int* ks, int* kt, const char* who) {
  if (n < 1 || n > INT32_MAX || p < 2 || max_pts < 1 || dims(kernel, ks, kt) != 0) {
    set_error(std::string(who) + ": invalid argument");
    return KAFMM_EINVAL;
  }
  if (6 * (p - 1) * (p - 1) + 2 > KAFMM_MAX_SURFACE) {  // the leaf kernels stage one surface per CTA
    set_error(std::string(who) + ": p too large (surface of 6(p-1)^2+2 points exceeds 1024; p <= 14)");
    return KAFMM_EINVAL;
  }
  return KAFMM_OK;
}

kafmm_status kafmm_setup(const double* points, int64_t n, int kernel, int p, int max_pts_per_leaf,
                         kafmm_plan* out) {
  if (out) *out = nullptr;
  int ks, kt;
  if (!points || !out) {
    set_error("kafmm_setup: invalid argument");
    return KAFMM_EINVAL;
  }
  if (kafmm_status st = check_setup_args(n, kernel, p, max_pts_per_leaf, &ks, &kt, "kafmm_setup")) return st;
  kafmm_plan_s* P = nullptr;
  KF_API_BEGIN
  int dev = 0;
  KF_CUDA(cudaGetDevice(&dev));
  P = new kafmm_plan_s();
  init_plan(*P, kernel, p, max_pts_per_leaf, n, ks, kt);
  build_plan_core(*P, points);
  alloc_workspaces(*P);
  *out = P;
  return KAFMM_OK;
  }
  catch (const Error& e) {
    set_error(e.msg);
    free_plan(P);
    cudaGetLastError();
    return e.st;
  }
  catch (const std::bad_alloc&) {
    set_error("host allocation failed");
    free_plan(P);
    return KAFMM_ENOMEM;
  }
}

// multi-GPU: the plan of this rank's part of a point set spread over the ranks
static kafmm_status setup_dist_common(const double* local_points, int64_t n_local, int kernel, int p, int max_pts,
                                      Comm* comm, bool owns, kafmm_plan* out) {
  if (out) *out = nullptr;
  int ks, kt;
  if (!out || n_local < 0 || (n_local > 0 && !local_points) || !comm) {
    if (owns) delete comm;
    set_error("kafmm_setup_dist: invalid argument");
    return KAFMM_EINVAL;
  }
  if (kafmm_status st = check_setup_args(1, kernel, p, max_pts, &ks, &kt, "kafmm_setup_dist")) {
    if (owns) delete comm;
    return st;
  }
  kafmm_plan_s* P = nullptr;
  KF_API_BEGIN
  P = new kafmm_plan_s();
  P->dist = new DistState();
  P->dist->comm = comm;
  P->dist->owns_comm = owns;
  init_plan(*P, kernel, p, max_pts, 0, ks, kt);
  setup_dist(*P, local_points, n_local);
  *out = P;
  return KAFMM_OK;
  }
  catch (const Error& e) {
    set_error(e.msg);
    if (P) free_plan(P);
    else if (owns) delete comm;
    cudaGetLastError();
    return e.st;
  }
  catch (const std::bad_alloc&) {
    set_error("host allocation failed");
    if (P) free_plan(P);
    else if (owns) delete comm;
    return KAFMM_ENOMEM;
  }
}

kafmm_status kafmm_get_unique_id(unsigned char id[128]) {
  if (!id) return KAFMM_EINVAL;
  KF_API_BEGIN
  nccl_unique_id(id);
  return KAFMM_OK;
  KF_API_END
}

kafmm_status kafmm_setup_dist(const double* local_points, int64_t n_local, int kernel, int p, int max_pts_per_leaf,
                              int rank, int world, const unsigned char id[128], kafmm_plan* out) {
  if (out) *out = nullptr;
  if (!id || world < 1 || rank < 0 || rank >= world) {
    set_error("kafmm_setup_dist: invalid rank / world / id");
    return KAFMM_EINVAL;
  }
  Comm* c = nullptr;
  KF_API_BEGIN
  c = make_nccl_comm(id, rank, world);
  KF_API_END
  return setup_dist_common(local_points, n_local, kernel, p, max_pts_per_leaf, c, true, out);
}

kafmm_status kafmm_comm_local_create(int world, kafmm_comm* comms) {
  if (world < 1 || !comms) return KAFMM_EINVAL;
  KF_API_BEGIN
  std::vector<Comm*> c(world);
  make_local_comms(world, c.data());
  for (int r = 0; r < world; ++r) comms[r] = reinterpret_cast<kafmm_comm>(c[r]);
  return KAFMM_OK;
  KF_API_END
}

void kafmm_comm_destroy(kafmm_comm comm) { delete reinterpret_cast<Comm*>(comm); }

kafmm_status kafmm_setup_dist_comm(const double* local_points, int64_t n_local, int kernel, int p,
                                   int max_pts_per_leaf, kafmm_comm comm, kafmm_plan* out) {
  return setup_dist_common(local_points, n_local, kernel, p, max_pts_per_leaf, reinterpret_cast<Comm*>(comm), false,
                           out);
}

kafmm_status kafmm_dist_query(kafmm_plan plan, int what, int64_t* out) {
  if (!plan || !out) return KAFMM_EINVAL;
  const Plan& P = *plan;
  if (!P.dist) {
    set_error("kafmm_dist_query: not a partitioned plan");
    return KAFMM_ESTATE;
  }
  const DistState& D = *P.dist;
  if (what == 0) {
    const int64_t v[14] = {D.rank, D.world, D.n_global, D.n_caller, D.n_owned, P.nloc, D.n_ghost_points,
                           P.nrow, D.n_ghost_boxes, D.nshared, P.bytes,
                           8 * (D.e1.stotal + D.e3.stotal + D.e4.stotal + D.nshared * P.neq), D.n_v_local,
                           D.n_p2p_local};
    for (int i = 0; i < 14; ++i) out[i] = v[i];
  } else if (what == 1) {
    for (int i = 0; i <= D.world; ++i) out[i] = D.cuts[i];
  } else if (what == 2) {
    for (size_t i = 0; i < D.counts.size(); ++i) out[i] = D.counts[i];
  } else {
    return KAFMM_EINVAL;
  }
  return KAFMM_OK;
}

kafmm_status kafmm_set_stream(kafmm_plan plan, void* stream) {
  if (!plan) return KAFMM_EINVAL;
  plan->stream = (cudaStream_t)stream;
  return KAFMM_OK;
}

kafmm_status kafmm_eval(kafmm_plan plan, const double* src_values, double* trg_out) {
  if (!plan || !src_values || !trg_out) {
    set_error("kafmm_eval: null argument");
    return KAFMM_EINVAL;
  }
  KF_API_BEGIN
  Plan& P = *plan;
  if (P.dist) {  // partitioned plan: this caller's rows in and out, exchanges inside
    run_eval_dist(P, src_values, trg_out);
    collect_stage_times(P);
    return KAFMM_OK;
  }
  if (P.use_graph && P.timing == 0 && P.graph_warm) {
    if (!P.gexec || P.g_src != src_values || P.g_out != trg_out || P.g_mode != P.m2l_mode) {
      if (P.gexec) KF_CUDA(cudaGraphExecDestroy(P.gexec));
      P.gexec = nullptr;
      cudaStream_t user = P.stream;
      P.stream = P.gstream;
      cudaGraph_t g = nullptr;
      KF_CUDA(cudaStreamBeginCapture(P.gstream, cudaStreamCaptureModeThreadLocal));
      try {
        run_eval(P, src_values, trg_out);
      } catch (...) {
        cudaStreamEndCapture(P.gstream, &g);
        if (g) cudaGraphDestroy(g);
        P.stream = user;
        throw;
      }
      KF_CUDA(cudaStreamEndCapture(P.gstream, &g));
      P.stream = user;
      KF_CUDA(cudaGraphInstantiate(&P.gexec, g, 0));
      KF_CUDA(cudaGraphDestroy(g));
      P.g_src = src_values;
      P.g_out = trg_out;
      P.g_mode = P.m2l_mode;
    }
    KF_CUDA(cudaEventRecord(P.ev_gin, P.stream));
    KF_CUDA(cudaStreamWaitEvent(P.gstream, P.ev_gin, 0));
    KF_CUDA(cudaGraphLaunch(P.gexec, P.gstream));
    KF_CUDA(cudaEventRecord(P.ev_gout, P.gstream));
    KF_CUDA(cudaStreamWaitEvent(P.stream, P.ev_gout, 0));
    return KAFMM_OK;
  }
  run_eval(P, src_values, trg_out);  // (also the first, uncaptured, evaluation of graph mode:
  P.graph_warm = true;                // one-time kernel attribute setup happens outside capture)
  collect_stage_times(P);
  return KAFMM_OK;
  KF_API_END
}

// Target rows of the union carry zero strength; for the regularised Stokes
// kernels their blob size is set to 1 so that a target coinciding with another
// point gives 0 * finite instead of 0 * (1/0) (reading R19).
__global__ void k_fill_col(double* v, int64_t lo, int64_t hi, int ks, int col, double x) {
  int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < hi) v[i * ks + col] = x;
}

kafmm_status kafmm_setup2(const double* src_points, int64_t n_src, const double* trg_points, int64_t n_trg,
                          int kernel, int p, int max_pts_per_leaf, kafmm_plan* out) {
  if (out) *out = nullptr;
  if (!src_points || !trg_points || !out || n_src < 1 || n_trg < 1 || n_src + n_trg > INT32_MAX) {
    set_error("kafmm_setup2: invalid argument");
    return KAFMM_EINVAL;
  }
  double* u = nullptr;
  if (cudaMalloc(&u, (size_t)(n_src + n_trg) * 3 * 8) != cudaSuccess) {
    set_error("kafmm_setup2: out of memory");
    return KAFMM_ENOMEM;
  }
  if (cudaMemcpy(u, src_points, (size_t)n_src * 24, cudaMemcpyDeviceToDevice) != cudaSuccess ||
      cudaMemcpy(u + 3 * n_src, trg_points, (size_t)n_trg * 24, cudaMemcpyDeviceToDevice) != cudaSuccess) {
    const cudaError_t e = cudaGetLastError();
    cudaFree(u);
    set_error(std::string("kafmm_setup2: copying the point sets failed (device pointers of n x 3 doubles "
                          "expected): ") + cudaGetErrorString(e));
    return KAFMM_EINVAL;
  }
  kafmm_status st = kafmm_setup(u, n_src + n_trg, kernel, p, max_pts_per_leaf, out);
  cudaFree(u);
  if (st != KAFMM_OK) return st;
  Plan& P = **out;
  try {
    P.n_src = n_src;
    P.d_uvals = dalloc<double>(P, (size_t)P.n * P.ks);  // zero (dalloc clears): target rows stay 0
    P.d_uout = dalloc<double>(P, (size_t)P.n * P.kt);
    const int pcol = kernel == KAFMM_STOKES_REG_VEL ? 3 : kernel == KAFMM_STOKES_REG_VEL_OMEGA ? 6 : -1;
    if (pcol >= 0) {
      k_fill_col<<<(unsigned)((n_trg + 255) / 256), 256, 0, P.stream>>>(P.d_uvals, n_src, P.n, P.ks, pcol, 1.0);
      KF_CHECK_LAUNCH();
    }
    KF_CUDA(cudaStreamSynchronize(P.stream));
  } catch (const Error& e) {
    set_error(e.msg);
    kafmm_destroy(*out);
    *out = nullptr;
    return e.st;
  }
  return KAFMM_OK;
}

kafmm_status kafmm_eval2(kafmm_plan plan, const double* src_values, double* trg_out) {
  if (!plan || !src_values || !trg_out) {
    set_error("kafmm_eval2: null argument");
    return KAFMM_EINVAL;
  }
  if (plan->n_src < 0) {
    set_error("kafmm_eval2: plan not made by kafmm_setup2");
    return KAFMM_ESTATE;
  }
  KF_API_BEGIN
  Plan& P = *plan;
  KF_CUDA(cudaMemcpyAsync(P.d_uvals, src_values, (size_t)P.n_src * P.ks * 8, cudaMemcpyDeviceToDevice, P.stream));
  run_eval(P, P.d_uvals, P.d_uout);
  collect_stage_times(P);
  KF_CUDA(cudaMemcpyAsync(trg_out, P.d_uout + (size_t)P.n_src * P.kt, (size_t)(P.n - P.n_src) * P.kt * 8,
                          cudaMemcpyDeviceToDevice, P.stream));
  return KAFMM_OK;
  KF_API_END
}

kafmm_status kafmm_set_graph(kafmm_plan plan, int on) {
  if (!plan) return KAFMM_EINVAL;
  plan->use_graph = on != 0;
  return KAFMM_OK;
}

kafmm_status kafmm_eval_host(kafmm_plan plan, const double* src_values, double* trg_out) {
  if (!plan || !src_values || !trg_out) {
    set_error("kafmm_eval_host: null argument");
    return KAFMM_EINVAL;
  }
  KF_API_BEGIN
  Plan& P = *plan;
  const int64_t rows = P.dist ? P.dist->n_caller : P.n;  // the caller's rows
  if (!P.d_stage_in) {
    P.d_stage_in = dalloc<double>(P, (size_t)std::max<int64_t>(1, rows) * P.ks);
    P.d_stage_out = dalloc<double>(P, (size_t)std::max<int64_t>(1, rows) * P.kt);
  }
  KF_CUDA(cudaMemcpyAsync(P.d_stage_in, src_values, (size_t)rows * P.ks * 8, cudaMemcpyHostToDevice, P.stream));
  if (P.dist) run_eval_dist(P, P.d_stage_in, P.d_stage_out);
  else run_eval(P, P.d_stage_in, P.d_stage_out);
  KF_CUDA(cudaMemcpyAsync(trg_out, P.d_stage_out, (size_t)rows * P.kt * 8, cudaMemcpyDeviceToHost, P.stream));
  KF_CUDA(cudaStreamSynchronize(P.stream));
  take_nonfinite(P);
  return KAFMM_OK;
  KF_API_END
}

kafmm_status kafmm_check_values(kafmm_plan plan, const double* src_values) {
  if (!plan || !src_values) return KAFMM_EINVAL;
  KF_API_BEGIN
  check_values(*plan, src_values);
  return KAFMM_OK;
  KF_API_END
}

kafmm_status kafmm_sync(kafmm_plan plan) {
  if (!plan) return KAFMM_EINVAL;
  KF_API_BEGIN
  KF_CUDA(cudaStreamSynchronize(plan->stream));
  KF_CUDA(cudaGetLastError());
  take_nonfinite(*plan);
  return KAFMM_OK;
  KF_API_END
}

void kafmm_destroy(kafmm_plan plan) { free_plan(plan); }

const char* kafmm_status_string(int s) {
  switch (s) {
    case KAFMM_OK: return "ok";
    case KAFMM_EINVAL: return "invalid argument";
    case KAFMM_EDOMAIN: return "point outside [0,1)^3";
    case KAFMM_ENONFINITE: return "non-finite input";
    case KAFMM_ENOMEM: return "out of memory";
    case KAFMM_ECUDA: return "CUDA error";
    case KAFMM_ENCCL: return "NCCL error";
    case KAFMM_ESTATE: return "invalid state";
    default: return "unknown status";
  }
}

const char* kafmm_last_error(void) { return g_last_error.c_str(); }

kafmm_status kafmm_get_info(kafmm_plan plan, kafmm_info* info) {
  if (!plan || !info) return KAFMM_EINVAL;
  Plan& P = *plan;
  std::memset(info, 0, sizeof(*info));
  info->n_points = P.n;
  info->kernel = P.kernel;
  info->p = P.p;
  info->max_pts = P.cap;
  info->depth = P.depth;
  info->k_s = P.ks;
  info->k_t = P.kt;
  info->n_surf = P.M;
  info->n_equiv = P.neq;
  info->kept_up = P.kept_up;
  info->kept_dn = P.kept_dn;
  info->n_boxes = P.nbox;
  info->n_leaves = P.nleaf;
  info->n_u_pairs = P.n_u;
  info->n_v_pairs = P.n_v;
  info->n_w_pairs = P.n_w;
  info->n_p2p = P.n_p2p;
  info->workspace_bytes = P.bytes;
  return KAFMM_OK;
}

kafmm_status kafmm_get_tree(kafmm_plan plan, int32_t* level, int32_t* ijk, int32_t* parent, int32_t* is_leaf,
                            int64_t* pt_begin, int64_t* pt_end) {
  if (!plan) return KAFMM_EINVAL;
  KF_API_BEGIN
  Plan& P = *plan;
  const int64_t nb = P.nbox;
  if (level) KF_CUDA(cudaMemcpy(level, P.d_level, nb * 4, cudaMemcpyDeviceToHost));
  if (ijk) KF_CUDA(cudaMemcpy(ijk, P.d_ijk, nb * 12, cudaMemcpyDeviceToHost));
  if (parent) KF_CUDA(cudaMemcpy(parent, P.d_parent, nb * 4, cudaMemcpyDeviceToHost));
  if (is_leaf) {
    std::string tmp(nb, '\0');
    KF_CUDA(cudaMemcpy(&tmp[0], P.d_leaf, nb, cudaMemcpyDeviceToHost));
    for (int64_t b = 0; b < nb; ++b) is_leaf[b] = tmp[b] ? 1 : 0;
  }
  if (pt_begin) KF_CUDA(cudaMemcpy(pt_begin, P.d_pbeg, nb * 8, cudaMemcpyDeviceToHost));
  if (pt_end) KF_CUDA(cudaMemcpy(pt_end, P.d_pend, nb * 8, cudaMemcpyDeviceToHost));
  return KAFMM_OK;
  KF_API_END
}

kafmm_status kafmm_get_permutation(kafmm_plan plan, int64_t* perm) {
  if (!plan || !perm) return KAFMM_EINVAL;
  if (plan->dist) {
    set_error("kafmm_get_permutation: a partitioned plan holds only its local points");
    return KAFMM_ESTATE;
  }
  KF_API_BEGIN
  KF_CUDA(cudaMemcpy(perm, plan->d_perm, plan->n * 8, cudaMemcpyDeviceToHost));
  return KAFMM_OK;
  KF_API_END
}

kafmm_status kafmm_get_list(kafmm_plan plan, int which, int32_t* tgt, int32_t* src) {
  if (!plan || !tgt || !src) return KAFMM_EINVAL;
  KF_API_BEGIN
  Plan& P = *plan;
  std::vector<int32_t> leaves(P.nleaf);
  KF_CUDA(cudaMemcpy(leaves.data(), P.d_leaf_ids, P.nleaf * 4, cudaMemcpyDeviceToHost));
  if (which == 'U' || which == 'W') {
    int64_t cnt = which == 'U' ? P.n_u : P.n_w;
    std::vector<int64_t> off(P.nleaf + 1);
    KF_CUDA(cudaMemcpy(off.data(), which == 'U' ? P.d_u_off : P.d_w_off, (P.nleaf + 1) * 8, cudaMemcpyDeviceToHost));
    if (cnt) KF_CUDA(cudaMemcpy(src, which == 'U' ? P.d_u_src : P.d_w_src, cnt * 4, cudaMemcpyDeviceToHost));
    for (int64_t s = 0; s < P.nleaf; ++s)
      for (int64_t e = off[s]; e < off[s + 1]; ++e) tgt[e] = leaves[s];
  } else if (which == 'V') {
    std::vector<int2> pr(P.n_v);
    if (P.n_v) KF_CUDA(cudaMemcpy(pr.data(), P.d_v_pairs, P.n_v * 8, cudaMemcpyDeviceToHost));
    for (int64_t e = 0; e < P.n_v; ++e) {
      tgt[e] = pr[e].y;
      src[e] = pr[e].x;
    }
  } else if (which == 'X') {
    std::vector<int32_t> tg(P.n_xbox);
    std::vector<int64_t> off(P.n_xbox + 1);
    if (P.n_xbox) {
      KF_CUDA(cudaMemcpy(tg.data(), P.d_x_tgt, P.n_xbox * 4, cudaMemcpyDeviceToHost));
      KF_CUDA(cudaMemcpy(off.data(), P.d_x_off, (P.n_xbox + 1) * 8, cudaMemcpyDeviceToHost));
      KF_CUDA(cudaMemcpy(src, P.d_x_src, P.n_w * 4, cudaMemcpyDeviceToHost));
    }
    for (int64_t s = 0; s < P.n_xbox; ++s)
      for (int64_t e = off[s]; e < off[s + 1]; ++e) tgt[e] = tg[s];
  } else {
    throw Error{KAFMM_EINVAL, "kafmm_get_list: which must be U, V, W or X"};
  }
  return KAFMM_OK;
  KF_API_END
}

kafmm_status kafmm_set_timing(kafmm_plan plan, int on) {
  if (!plan) return KAFMM_EINVAL;
  if (on < 0 || on > 2) return KAFMM_EINVAL;
  plan->timing = on;
  return KAFMM_OK;
}

kafmm_status kafmm_stage_times(kafmm_plan plan, float* ms) {
  if (!plan || !ms) return KAFMM_EINVAL;
  for (int s = 0; s < KAFMM_N_STAGES; ++s) ms[s] = plan->stage_ms[s];
  return KAFMM_OK;
}

const char* kafmm_stage_name(int s) {
  static const char* names[KAFMM_N_STAGES] = {"gather_src", "s2m",      "uc2ue", "m2m",     "m2l",        "s2l",
                                              "dc2de+l2l",  "l2l(in dc2de)", "l2t+m2t", "p2p", "scatter_out", "total",
                                              "m2l_product"};
  return (s >= 0 && s < KAFMM_N_STAGES) ? names[s] : "?";
}

kafmm_status kafmm_set_m2l_mode(kafmm_plan plan, int mode) {
  if (!plan || mode < 0 || mode > 3) return KAFMM_EINVAL;
  if (mode != 0 && plan->NF == 0 && plan->depth >= 2) {
    set_error("FFT M2L not available for this p");
    return KAFMM_EINVAL;
  }
  KF_API_BEGIN
  if (mode == M2L_DENSE) build_dense_m2l(*plan);
  plan->m2l_mode = mode;
  return KAFMM_OK;
  KF_API_END
}

kafmm_status kafmm_get_m2l_mode(kafmm_plan plan, int* mode) {
  if (!plan || !mode) return KAFMM_EINVAL;
  *mode = plan->m2l_mode;
  return KAFMM_OK;
}

kafmm_status kafmm_fft_stats(kafmm_plan plan, int64_t* st) {
  if (!plan || !st) return KAFMM_EINVAL;
  for (int i = 0; i < 10; ++i) st[i] = 0;
  for (const FftChunk& ch : plan->fft_chunks) {
    st[0] += 1;
    st[8] += ch.nsrc_children;
    st[9] += ch.nitems;
    st[1] += ch.nq;
    st[2] += ch.npar;
    st[3] += ch.nt;
    st[4] += ch.npairs;
    st[5] += (plan->m2l_mode == M2L_FFT_PAIRS || (plan->m2l_mode == M2L_FFT && ch.block_fill < pair_fill_threshold())) ? 1 : 0;
  }
  st[6] = plan->NF;
  st[7] = plan->fft_budget;
  return KAFMM_OK;
}

kafmm_status kafmm_launch_count(kafmm_plan plan, int* n) {
  if (!plan || !n) return KAFMM_EINVAL;
  *n = plan->launches;
  return KAFMM_OK;
}

}  // extern "C"
