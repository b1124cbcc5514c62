/*
 * kafmm.h -- C ABI of the B200-native Kernel Aggregated FMM evaluation pass.
 *
 * Method: Yan & Blackwell, "Kernel Aggregated Fast Multipole Method",
 * arXiv 2010.15155.  The library approximates the kernel sum
 *     g_i(x^a) = sum_b K_ij(x^a, y^b, s^b)                 Eq. (1)/(2)
 * with a kernel-independent FMM whose eight traversal stages use the kernels
 * of the paper's kernel tables (Table I; Tables IV/V,
 * PAPER.md:292-349): the ML-tree stages (M2M, M2L, L2L) use the linear
 * Laplace kernel L or Stokeslet G, the S-row the (possibly nonlinear)
 * source kernel, the T-column the target kernel.
 *
 * Sources and targets are the same point set.
 *
 * Memory: every pointer argument named "device" is a CUDA device pointer on
 * the current device with 8-byte alignment (e.g. torch.Tensor.data_ptr());
 * arrays are row-major, C-contiguous float64.  The caller owns its arrays; the
 * plan owns every tree, list, operator and workspace buffer until
 * kafmm_destroy().  kafmm_setup copies the points, so they may be freed on
 * return.  No exception ever crosses this ABI: every entry point returns a
 * status; the detail string of the last failure on the calling thread is
 * kafmm_last_error().
 *
 * There is no CPU fallback: without a CUDA device every entry point that
 * computes returns KAFMM_ECUDA.
 */
#ifndef KAFMM_H
#define KAFMM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct kafmm_plan_s* kafmm_plan; /* opaque; owned by the library */

typedef enum {
  KAFMM_OK = 0,
  KAFMM_EINVAL = 1,     /* null pointer, n < 1, n > 2^31-1, p < 2 or p > 14, max_pts < 1, unknown kernel */
  KAFMM_EDOMAIN = 2,    /* a point outside [0,1)^3 */
  KAFMM_ENONFINITE = 3, /* NaN/Inf in points or values, or negative b / eps */
  KAFMM_ENOMEM = 4,     /* device allocation failed */
  KAFMM_ECUDA = 5,      /* CUDA / cuBLAS / cuSOLVER error (detail in kafmm_last_error) */
  KAFMM_ENCCL = 6,      /* NCCL error, or libnccl.so.2 missing (multi-GPU plans) */
  KAFMM_ESTATE = 7      /* invalid plan state */
} kafmm_status;

/* Kernel summation problems (Table XI).
 *   LAPLACE_PGRAD   k_s=1 [q]        k_t=4 [phi, dphi/dx, dphi/dy, dphi/dz]
 *                   phi = sum q/(4 pi r), grad w.r.t. the target
 *   STOKESLET       k_s=3 [f]        k_t=3 [u], u = sum G f
 *   RPY             k_s=4 [f, b]     k_t=6 [u, lap u], u = sum G^RPY(b) f, lap u = sum lap G f
 *                   (Eqs. RPYflow/RPYkernel, Table IV); the target
 *                   radius assembly u + a^2/6 lap u (Eq. RPYtrgvel) is the caller's
 *   STOKES_REG_VEL  k_s=4 [f, eps]   k_t=3 [u], u = sum G^eps f
 *   STOKES_REG_VEL_OMEGA  k_s=7 [f, t, eps]  k_t=6 [u, omega]:
 *                   u = sum G^eps f + T^eps t, omega = sum Omega^eps f + W^eps t
 *                   (Table VI; ML tree G, T column G (+) Omega)
 *   LAPLACE_PGRADGRAD  k_s=4 [q, d]  k_t=10 [phi, grad phi, grad grad phi (xx,xy,xz,yy,yz,zz)]
 *                   charges and dipoles at every point, phi = sum (q + d . grad_y)/(4 pi r)
 *                   (Table III; ML tree L)
 *   LAPLACE_QPGRADGRAD k_s=9 [Q (3x3 row-major)]  k_t=10 as LAPLACE_PGRADGRAD,
 *                   phi = sum Q_jk d2/dx_j dx_k 1/(4 pi r) (Table XI)
 * Self pairs (r^2 == 0) are skipped by the singular kernels and kept by the
 * regularized ones, where G^eps(0) = 1/(4 pi eps) is finite. */
typedef enum {
  KAFMM_LAPLACE_PGRAD = 1,
  KAFMM_STOKESLET = 2,
  KAFMM_RPY = 3,
  KAFMM_STOKES_REG_VEL = 4,
  KAFMM_STOKES_REG_VEL_OMEGA = 5,
  KAFMM_LAPLACE_PGRADGRAD = 6,
  KAFMM_LAPLACE_QPGRADGRAD = 7
} kafmm_kernel;

/* Source and target dimensions of a kernel.  EINVAL for an unknown kernel. */
kafmm_status kafmm_kernel_dims(int kernel, int* k_s, int* k_t);

/* Build the plan: Morton-sort the points, build the adaptive octree (a box
 * splits iff it holds more than max_pts_per_leaf points and its level < 20),
 * the U/V/W/X lists and the translation operators at
 * multipole order p (M = 6(p-1)^2+2 surface points).
 *   points            device, n x 3 (x, y, z), every coordinate in [0, 1)
 *   n                 number of points (>= 1)
 *   kernel            a kafmm_kernel value
 *   p                 multipole order m of the paper, 2 <= p <= 14 (M = 6(p-1)^2+2 <= 1024 surface
 *                     points, the leaf kernels' limit); the FFT M2L covers p = 3..8, 10, 12, other
 *                     orders use the dense M2L
 *   max_pts_per_leaf  leaf capacity, >= 1
 *   out               receives the plan (NULL on failure)
 * Synchronous: returns after the plan is complete. */
kafmm_status kafmm_setup(const double* points, int64_t n, int kernel, int p,
                         int max_pts_per_leaf, kafmm_plan* out);

/* Stream for subsequent kafmm_eval calls (default: the legacy default stream).
 * `stream` is a cudaStream_t passed as void*. */
kafmm_status kafmm_set_stream(kafmm_plan plan, void* stream);

/* One evaluation pass (the hot path): S2M, UC2UE, M2M, M2L, S2L, DC2DE, L2L,
 * L2T, M2T and P2P, then un-permute to user order.
 *   src_values  device, n x k_s, user (setup) order
 *   trg_out     device, n x k_t, user order, overwritten
 * Asynchronous on the plan's stream; trg_out is valid after stream sync.
 * A plan serves one evaluation at a time (single workspace).
 * Input errors found on the device (a NaN/Inf source value, a negative b or eps)
 * raise a sticky flag while the values are gathered; the next kafmm_sync (or
 * kafmm_eval_host, which synchronises) returns KAFMM_ENONFINITE and clears it,
 * so the hot path itself never waits on the host. */
kafmm_status kafmm_eval(kafmm_plan plan, const double* src_values, double* trg_out);

/* End-to-end variant with HOST buffers: copies src_values host->device, runs
 * kafmm_eval and copies trg_out device->host, then synchronises the stream.
 *   src_values  host, n x k_s (pinned memory gives full copy bandwidth)
 *   trg_out     host, n x k_t */
kafmm_status kafmm_eval_host(kafmm_plan plan, const double* src_values, double* trg_out);

/* Separate source and target point sets (STKFMM takes SL
 * and target points as different sets).  The octree is built on the union
 * [sources; targets]; targets carry zero source strength and only the target
 * rows are returned, so the result is sum over sources of K(x_t, y_s) s_s,
 * with pairs at r^2 == 0 skipped by the singular kernels as usual.
 *   src_points  device, n_src x 3;  trg_points  device, n_trg x 3 (both in [0,1)^3)
 *   kafmm_eval2: src_values device n_src x k_s, trg_out device n_trg x k_t.
 * kafmm_eval on such a plan is EINVAL-free but works on the union rows; use
 * kafmm_eval2.  ESTATE if kafmm_eval2 is called on a plan from kafmm_setup. */
kafmm_status kafmm_setup2(const double* src_points, int64_t n_src, const double* trg_points, int64_t n_trg,
                          int kernel, int p, int max_pts_per_leaf, kafmm_plan* out);
kafmm_status kafmm_eval2(kafmm_plan plan, const double* src_values, double* trg_out);

/* Validate source values (finite; b / eps >= 0) on the device.  Synchronous.
 * kafmm_eval itself does not check, to keep the hot path free of host syncs. */
kafmm_status kafmm_check_values(kafmm_plan plan, const double* src_values);

/* Waits for the plan's stream; surfaces asynchronous CUDA errors, and
 * KAFMM_ENONFINITE if an evaluation since the last sync saw a non-finite source
 * value or a negative b / eps (the outputs of that evaluation are then undefined). */
kafmm_status kafmm_sync(kafmm_plan plan);

void kafmm_destroy(kafmm_plan plan);

const char* kafmm_status_string(int status);
const char* kafmm_last_error(void);

/* ---- introspection (tests, bench) ------------------------------------- */
typedef struct {
  int64_t n_points;
  int kernel, p, max_pts, depth;
  int k_s, k_t;
  int n_surf;           /* M = 6(p-1)^2 + 2 */
  int n_equiv;          /* n = k * M, length of one equivalent/check vector */
  int kept_up, kept_dn; /* singular values kept by UC2UE / DC2DE (tau = 1e-12) */
  int64_t n_boxes, n_leaves;
  int64_t n_u_pairs;    /* (target leaf, source leaf) U-list entries */
  int64_t n_v_pairs;    /* M2L (target box, source box) pairs */
  int64_t n_w_pairs;    /* M2T pairs == S2L (X-list) pairs */
  int64_t n_p2p;        /* point-point interactions in P2P */
  int64_t workspace_bytes;
} kafmm_info;

kafmm_status kafmm_get_info(kafmm_plan plan, kafmm_info* info);

/* Copy the octree to HOST arrays of length info.n_boxes (any may be NULL):
 * level, ijk (n_boxes x 3, integer coords at the box's level), parent (-1 for
 * root), is_leaf (0/1), pt_begin/pt_end (range in Morton order). Boxes are
 * ordered by level, then Morton key. */
kafmm_status kafmm_get_tree(kafmm_plan plan, int32_t* level, int32_t* ijk, int32_t* parent,
                            int32_t* is_leaf, int64_t* pt_begin, int64_t* pt_end);

/* HOST array of length n: perm[i] = user index of the i-th point in Morton order. */
kafmm_status kafmm_get_permutation(kafmm_plan plan, int64_t* perm);

/* Interaction lists as HOST pair arrays (target box, source box), lengths from
 * kafmm_get_info: which = 'U' (n_u_pairs), 'V' (n_v_pairs), 'W' (n_w_pairs:
 * target leaf, source box), 'X' (n_w_pairs: target box, source leaf). */
kafmm_status kafmm_get_list(kafmm_plan plan, int which, int32_t* tgt, int32_t* src);

/* Per-stage device times (ms) of the most recent kafmm_eval when stage
 * timing is on (kafmm_set_timing(plan, 1)); names via kafmm_stage_name.
 * Mode 1 runs every stage on the plan's stream so that its events bracket
 * only that stage (the near field then does not overlap the far field);
 * mode 2 records only the total and the M2L product (slots 11, 12) and keeps
 * the overlap; 0 turns timing off.
 * Slot 12 ("m2l_product") is the device time of the M2L product kernels
 * alone (the frequency-space DMMA products of the FFT variant, or the dense
 * DMMA GEMMs), a part of slot 4 ("m2l"). */
#define KAFMM_N_STAGES 13
kafmm_status kafmm_set_timing(kafmm_plan plan, int on);
kafmm_status kafmm_stage_times(kafmm_plan plan, float* ms /* KAFMM_N_STAGES */);
const char* kafmm_stage_name(int stage);
/* M2L variant used by kafmm_eval:
 *   0 = dense: raw kernel matrices grouped by V offset on the FP64 tensor cores
 *   1 = FFT (default when p is in {3..8, 10, 12}): convolution on the (2p-1)^3
 *       lattice grid; the frequency-space product runs per chunk of target
 *       parents as DMMA parent blocks (8x8 child blocks x 26 directions), or
 *       per V pair where fewer than 35% of those block entries are V pairs
 *   2 = FFT, parent blocks everywhere;  3 = FFT, per V pair everywhere.
 * All compute the same matrices; results agree to rounding.  EINVAL for an
 * unknown mode or FFT with an unsupported p.  (Environment KAFMM_M2L=dense at
 * setup selects dense.) */
kafmm_status kafmm_set_m2l_mode(kafmm_plan plan, int mode);
kafmm_status kafmm_get_m2l_mode(kafmm_plan plan, int* mode);

/* FFT M2L work summary, st[10]: chunks, source parent blocks (incl. halos
 * transformed once per chunk), target parents, target boxes, V pairs, chunks
 * whose product runs per pair under the current mode, frequency bins NF,
 * spectra budget in bytes, existing source children (transforms per component),
 * items of the sparse-chunk product stream. */
kafmm_status kafmm_fft_stats(kafmm_plan plan, int64_t* st);

/* CUDA graph replay of kafmm_eval (on = 1): the first evaluation with a given
 * (src_values, trg_out, M2L mode) is captured into a graph on an internal
 * stream, later ones with the same pointers replay it; the plan's stream is
 * joined by events, so ordering is unchanged for the caller.  Ignored while
 * stage timing is on.  Default off. */
kafmm_status kafmm_set_graph(kafmm_plan plan, int on);

/* Kernel launches issued by one kafmm_eval. */
kafmm_status kafmm_launch_count(kafmm_plan plan, int* n);

/* FP64 throughput of the current device (roofline denominator; no FP64 figure
 * is in MEASURED_PEAKS.json): which = 0 DMMA.8x8x4 tensor-core loop,
 * 1 DFMA loop, over 4 CTAs of 256 threads per SM.  Result in TFLOP/s. */
kafmm_status kafmm_fp64_peak(int which, double* tflops);

/* ---- multi-GPU (the paper's MPI domain decomposition,
 * PAPER.md:600-603 and App. D :918-933) ---------------------------------------
 * One process per GPU.  Each rank passes its own rows of the point set; the
 * global point set is the concatenation of the ranks' rows in rank order.
 * Setup all-gathers the points, builds the global octree and lists on every
 * rank (the same deterministic build), cuts the Morton-sorted points into
 * contiguous ranges of whole leaves balancing an estimate of the work, and
 * keeps on each rank only what its range needs: per-box equivalent / check
 * rows for the boxes whose subtree holds its points, the boxes straddling
 * ranks and the remote boxes its V / W lists name (ghosts); source records for
 * its points and the points of remote U / X leaves.
 * kafmm_eval (and kafmm_eval_host) on such a plan take this caller's n_local
 * rows of source values and return its n_local rows of outputs; inside, the
 * plan exchanges source values, straddling-box partial multipoles (all-reduce),
 * ghost multipoles and outputs over NCCL on the plan's stream, with the near
 * field (P2P) overlapping the multipole exchanges.  Every rank must call
 * kafmm_eval the same number of times (collective).  Results equal the
 * single-GPU plan's to rounding.
 *
 * kafmm_get_unique_id: a new NCCL unique id (rank 0; the caller broadcasts the
 *   128 bytes, e.g. with torch.distributed).  ENCCL if libnccl.so.2 cannot be
 *   opened (it is loaded at run time; a process that imported torch uses
 *   torch's copy).
 * kafmm_setup_dist: collective over `world` ranks; local_points device n_local x 3
 *   in [0,1)^3 (n_local may be 0; the total must be >= 1).  The plan owns its
 *   NCCL communicator.  ENCCL on a communicator failure. */
kafmm_status kafmm_get_unique_id(unsigned char id[128]);
kafmm_status kafmm_setup_dist(const double* local_points, int64_t n_local, int kernel, int p, int max_pts_per_leaf,
                              int rank, int world, const unsigned char id[128], kafmm_plan* out);

/* In-process test transport: `world` communicators whose ranks are host
 * threads of this process sharing one GPU (a host barrier plus device copies;
 * the ranks' kernels never wait on each other).  comms[world] receives the
 * handles; each is borrowed by one kafmm_setup_dist_comm call from its own
 * thread and must outlive that plan; free with kafmm_comm_destroy. */
typedef struct kafmm_comm_s* kafmm_comm;
kafmm_status kafmm_comm_local_create(int world, kafmm_comm* comms);
void kafmm_comm_destroy(kafmm_comm comm);
kafmm_status kafmm_setup_dist_comm(const double* local_points, int64_t n_local, int kernel, int p,
                                   int max_pts_per_leaf, kafmm_comm comm, kafmm_plan* out);

/* Partition facts of a kafmm_setup_dist plan (ESTATE for a single-GPU plan):
 *   what = 0: out[14] = rank, world, global points, caller rows, owned points,
 *             local points (owned + ghost), ghost points, heavy rows, ghost
 *             boxes, straddling boxes, plan device bytes, bytes this rank sends
 *             per eval (values, ghost UE, outputs, all-reduce), V pairs with a
 *             target on this rank, P2P pairs of its leaves
 *   what = 1: out[world + 1] = Morton cuts (rank r owns sorted points [c_r, c_r+1))
 *   what = 2: out[6 world] = rows per peer: values sent, values received, ghost
 *             UE sent, ghost UE received, outputs sent, outputs received */
kafmm_status kafmm_dist_query(kafmm_plan plan, int what, int64_t* out);

/* ---- RPY above a no-slip wall (Table X) ----
 * Particles in [0,1) x [0,1) x (1/2, 1) above the wall plane z = 1/2 (device,
 * n x 3); the library adds their mirror images (z -> 1 - z) and runs four
 * KAFMM summations over the 2n points (RPY, LapPGradGrad twice,
 * LapQPGradGrad), then assembles per particle
 *   u = u^S + grad phi^SDZ + x3 (grad phi^SD + grad phi^Q) - [0, 0, phi^SD + phi^Q],
 *   lap u = lap u^S + 2 d/dx3 grad (phi^SD + phi^Q),   x3 = z - 1/2.
 * src_values: device n x 4 [f, b]; trg_out: device n x 6 [u, lap u], user order.
 * EDOMAIN if a particle is not strictly above the wall.  The quadrupole sum
 * sits at the image points (reading R18). */
typedef struct kafmm_wall_s* kafmm_wall;
kafmm_status kafmm_wall_setup(const double* points, int64_t n, int p, int max_pts_per_leaf, kafmm_wall* out);
kafmm_status kafmm_wall_set_stream(kafmm_wall w, void* stream);
kafmm_status kafmm_wall_eval(kafmm_wall w, const double* src_values, double* trg_out);
void kafmm_wall_destroy(kafmm_wall w);

#ifdef __cplusplus
}
#endif
#endif /* KAFMM_H */
