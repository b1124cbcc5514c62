// Internal plan structure shared by the translation units of libkafmm.so.
// Not part of the ABI (include/kafmm.h is).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdlib>

#include <atomic>
#include <string>
#include <vector>

#include "../../include/kafmm.h"

namespace kafmm {

// Morton keys: 21 bits per axis, x in the highest bit of each 3-bit group, so
// the 3-bit group of a level is the child octant 4*cx + 2*cy + cz.
constexpr int QBITS = 21;
constexpr int MAX_LEVEL = 20;
constexpr int N_OFFSETS = 316;  // {-3..3}^3 minus {-1..1}^3 (V-list offsets)
// Function attributes (large dynamic shared memory) are per device: true the first
// time this is called for the current device with this flag word (thread-safe).
inline bool first_on_device(std::atomic<uint64_t>& done) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  return !(done.fetch_or(bit) & bit);
}
constexpr int KAFMM_MAX_SURFACE = 1024;  // surface points per box the leaf kernels support (p <= 14)

// Surface radii in units of the box half-width (reading R1).
constexpr double ALPHA_UE = 1.05, ALPHA_UC = 2.95, ALPHA_DC = 1.05, ALPHA_DE = 2.95;
constexpr double TAU = 1e-12;  // SVD truncation (reading R2)

// Tiling of the grouped FP64 GEMM (gemm_dmma.cuh).
constexpr int GEMM_BM = 128, GEMM_BN = 64, GEMM_BK = 16;

struct GemmTile {  // one CTA column-tile: up to GEMM_BN items sharing operator `op`
  int op;
  int item0;
  int nitem;
  int pad_;
  double alpha;
};

enum GemmMode { GEMM_STORE = 0, GEMM_ADD = 1, GEMM_ATOMIC = 2 };

struct GemmBatch {  // one launch of the grouped GEMM
  std::vector<GemmTile> h_tiles;
  GemmTile* d_tiles = nullptr;
  int2* d_items = nullptr;  // x = input column (box / leaf slot), y = output column
  bool owns_items = true;   // false when d_items aliases another array (the V-pair list)
  int64_t n_items = 0;
  int ntiles() const { return (int)h_tiles.size(); }
};

struct LevelRange {
  int64_t begin, end;  // box ids [begin, end) of one level
};

// FFT M2L work unit (kafmm_fft.cu): a Morton-contiguous run of target parents
// at level-1 (non-leaf), their children (the M2L targets) and the source
// parents Q (non-leaf colleagues of the target parents, whose children are
// the sources), sized to a memory budget.
struct FftChunk {
  int level = 0;
  int64_t npar = 0, nq = 0, nt = 0;
  int32_t* d_qbox = nullptr;  // nq source parent box ids
  int32_t* d_nbr = nullptr;   // npar x 26: local q of the colleague in direction d, or -1
  int32_t* d_tbox = nullptr;  // nt target box ids
  int2* d_tpb = nullptr;      // nt: (local parent index, child octant)
  int32_t* d_toff = nullptr;  // npar + 1: targets of local parent P are [toff[P], toff[P+1])
  // child occupancy for the sparse-chunk product (k_m2l_items): bit c of tpat[P] =
  // target parent P's child c exists (and is active on this rank)
  int64_t npairs = 0;           // V pairs of the chunk
  uint8_t* d_tpat = nullptr;    // npar
  // item stream of the sparse product (k_m2l_items): per unit (target parent, or half of
  // one) the (colleague direction d, source child c) items with a non-empty target mask,
  // CSR over the units in processing order
  int32_t* d_ioff = nullptr;    // units + 1
  int2* d_items = nullptr;      // {spectra block offset, item word: d*64+c | vmask << 11 | r << 19 | S << 29}
  int64_t nitems = 0;           // items, or groups (unit, d, cx) when groups
  bool groups = false;          // stream built for k_m2l_groups
  int64_t nsrc_children = 0;    // existing children of the chunk's source parents
  int32_t* d_ord = nullptr;     // units: processing order (parent id, or 2 parent + half)
  int32_t* d_wrange = nullptr;  // nrange + 1: each warp's positions in that order
  int64_t nrange = 0;
  int64_t nper = 0;             // ranges per CTA (k_m2l_groups takes them dynamically)
  double block_fill = 1.0;      // V pairs / (8x8 child blocks the DMMA product runs)
};

// M2L variants: dense per-offset GEMMs, or the FFT lattice convolution whose
// frequency-space product runs per chunk as DMMA parent blocks or, where the
// blocks are mostly empty (sparse adaptive trees), per V pair.
enum M2LMode { M2L_DENSE = 0, M2L_FFT = 1, M2L_FFT_BLOCKS = 2, M2L_FFT_PAIRS = 3 };
constexpr double FFT_PAIR_FILL = 0.35;  // block fill below which a chunk runs per pair (M2L_FFT)
// the threshold in use: FFT_PAIR_FILL, or KAFMM_PAIR_FILL from the environment (tuning knob)
inline double pair_fill_threshold() {
  static const double v = getenv("KAFMM_PAIR_FILL") ? atof(getenv("KAFMM_PAIR_FILL")) : FFT_PAIR_FILL;
  return v;
}

// The work lists the evaluation kernels run over.  For a plan built by
// kafmm_setup they alias the full lists; kafmm_restrict (multi-GPU, one rank
// per GPU) replaces them with the part of the tree this rank owns.
struct Jobs {
  int64_t plo = 0, phi = 0;          // owned points, Morton (sorted) order
  int32_t* leaf_ids = nullptr;       // owned leaves (L2T, M2T, P2P jobs)
  int64_t nleaf = 0;
  int64_t* w_off = nullptr;          // W list per job (CSR)
  int32_t* w_src = nullptr;
  int64_t* u_roff = nullptr;         // P2P merged source ranges per job (CSR)
  int2* u_rng = nullptr;
  int32_t* s2m_ids = nullptr;        // owned leaves at level >= 2
  int64_t ns2m = 0;
  int32_t* x_tgt = nullptr;          // active boxes with a non-empty X list
  int64_t nx = 0;
  int64_t* x_roff = nullptr;
  int2* x_rng = nullptr;
};

// Collectives of the multi-GPU evaluation (kafmm_comm.cu): NCCL, or an
// in-process group of host threads (test transport).  Counts and
// displacements are in doubles; every call is ordered on stream s.
struct Comm {
  int rank = 0, world = 1;
  virtual ~Comm() {}
  virtual void alltoallv(const double* sbuf, const int64_t* sdispl, const int64_t* scount, double* rbuf,
                         const int64_t* rdispl, const int64_t* rcount, cudaStream_t s) = 0;
  virtual void allreduce(double* buf, int64_t count, cudaStream_t s) = 0;
  virtual const char* kind() const = 0;
  std::vector<int64_t> allgather_count(int64_t mine, cudaStream_t s);
};
Comm* make_nccl_comm(const unsigned char id[128], int rank, int world);
void make_local_comms(int world, Comm** out);
void nccl_unique_id(unsigned char id[128]);

// One rank's side of the partitioned evaluation (kafmm_dist.cu).  The plan of a
// rank holds the global tree and lists but heavy per-box rows (UE, CHK, DE, T)
// only for its active, shared and ghost boxes, and source records only for its
// owned points and the remote points its U / X lists name.
struct Exchange {  // one all-to-all-v: counts and displacements in doubles, per peer
  std::vector<int64_t> scount, sdispl, rcount, rdispl;
  int64_t stotal = 0, rtotal = 0;
  double* d_sbuf = nullptr;
  double* d_rbuf = nullptr;
};
struct DistState {
  Comm* comm = nullptr;
  bool owns_comm = false;
  int rank = 0, world = 1;
  int64_t n_global = 0, n_caller = 0;   // all points; this caller's rows
  std::vector<int64_t> caller_off;      // world + 1: first global user row of each caller
  std::vector<int64_t> cuts;            // world + 1: Morton ranges of the ranks
  Exchange e1, e3, e4;                  // values, ghost UE, outputs
  int64_t* d_val_idx = nullptr;         // E1 send: caller-local value rows, per destination
  int64_t* d_out_idx = nullptr;         // E4 receive: caller-local output rows, per source
  int32_t* d_ue_send_rows = nullptr;    // E3: UE rows packed for the peers
  int32_t* d_ue_recv_rows = nullptr;    // E3: ghost UE rows unpacked
  int32_t* d_shared_rows = nullptr;     // E2: rows of the boxes straddling ranks
  int64_t nshared = 0;
  double* d_shared_buf = nullptr;
  int64_t n_ghost_boxes = 0, n_ghost_points = 0, n_owned = 0;
  int64_t n_v_local = 0, n_p2p_local = 0;  // M2L pairs with an active target, P2P pairs of owned leaves
  std::vector<int64_t> counts;          // 6 x world: val send/recv, ue send/recv, out send/recv (rows)
  ~DistState() {
    if (owns_comm) delete comm;
  }
};

enum Stage {
  ST_GATHER = 0, ST_S2M, ST_UC2UE, ST_M2M, ST_M2L, ST_S2L, ST_DC2DE, ST_L2L,
  ST_LEAF_FAR, ST_P2P, ST_SCATTER, ST_TOTAL,
  ST_M2L_PRODUCT  // reported only: device time of the M2L product kernels (part of ST_M2L)
};

struct Plan {
  // problem
  int kernel = 0, p = 0, cap = 0;
  int64_t n = 0;
  int ks = 0, kt = 0;   // user source / target dims
  int kml = 0;          // ML-tree kernel dimension: 1 (L) or 3 (G)
  int srec = 0;         // doubles per sorted source record (4 Laplace, 8 Stokes family)
  int M = 0, neq = 0, ldn = 0;   // surface points, equivalent vector length, padded
  int kept_up = 0, kept_dn = 0, ldk = 0;
  cudaStream_t stream = 0;
  cudaStream_t side = nullptr;         // near field (P2P) overlapped with the far-field chain
  cudaEvent_t ev_near_in = nullptr, ev_near_out = nullptr;
  // multi-GPU: the E2 / E3 exchanges run on cstream while the plan's stream runs S2L
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_up = nullptr, ev_ghost = nullptr;
  bool s2l_early = false;              // S2L already issued for this evaluation (before M2L)
  bool near_async = false;             // P2P of the current eval runs on `side`
  // CUDA graph of one evaluation (kafmm_set_graph): captured on `cap` for a
  // given (src, out, M2L mode) and replayed; the caller's stream is joined by events
  bool use_graph = false, graph_warm = false;
  cudaStream_t gstream = nullptr;
  cudaGraphExec_t gexec = nullptr;
  const double* g_src = nullptr;
  double* g_out = nullptr;
  int g_mode = -1;
  cudaEvent_t ev_gin = nullptr, ev_gout = nullptr;
  int timing = 0;                      // 0 off, 1 per-stage events (one stream), 2 total + M2L product only
  cudaEvent_t ev[ST_TOTAL + 1] = {};
  float stage_ms[ST_M2L_PRODUCT + 1] = {};
  std::vector<cudaEvent_t> prod_ev;  // start/stop pairs around the M2L product launches (timing on)
  int prod_used = 0;
  int launches = 0;

  // tree (device unless noted)
  int depth = 0;
  int64_t nbox = 0, nleaf = 0;
  std::vector<LevelRange> levels;  // host
  std::vector<uint8_t> box_active; // host; empty = every box (single plan), else the
                                   // boxes whose subtree holds points of this rank
  int32_t* d_level = nullptr;
  int32_t* d_ijk = nullptr;        // 3 per box
  int32_t* d_parent = nullptr;
  int32_t* d_child = nullptr;      // 8 per box, -1 if empty
  uint8_t* d_leaf = nullptr;
  int64_t* d_pbeg = nullptr;
  int64_t* d_pend = nullptr;
  uint64_t* d_key = nullptr;       // Morton prefix of the box at its level
  int64_t* d_perm = nullptr;       // Morton position -> user index
  double* d_pts = nullptr;         // sorted points, 4 doubles each (x, y, z, 0)

  // lists (CSR, device)
  int32_t* d_leaf_ids = nullptr;   // all leaves, level-major
  int64_t* d_u_off = nullptr;      // per leaf slot
  int32_t* d_u_src = nullptr;
  int64_t* d_w_off = nullptr;      // per leaf slot
  int32_t* d_w_src = nullptr;
  int64_t n_u = 0, n_w = 0, n_v = 0, n_p2p = 0;
  int32_t* d_s2m_ids = nullptr;    // leaves at level >= 2 (S2M jobs)
  int64_t n_s2m = 0;
  int2* d_u_rng = nullptr;         // P2P: merged source point ranges [x, y) per leaf slot
  int64_t* d_u_roff = nullptr;     // (CSR offsets, nleaf + 1)
  int2* d_x_rng = nullptr;         // S2L: merged source point ranges per X target
  int64_t* d_x_roff = nullptr;     // (CSR offsets, n_xbox + 1)
  int32_t* d_x_tgt = nullptr;      // boxes with a non-empty X list
  int64_t* d_x_off = nullptr;
  int32_t* d_x_src = nullptr;
  int64_t n_xbox = 0;
  int2* d_v_pairs = nullptr;       // (src, tgt) sorted by (level, offset) -- also the M2L items

  // operators (device, padded row-major)
  double* d_surf = nullptr;        // M x 3 unit lattice offsets (-1 + 2 i/(p-1))
  double* d_W1 = nullptr;          // UC2UE first factor  S^-1 U^T   (kept_up x ldn)
  double* d_W2 = nullptr;          // UC2UE second factor V          (neq x ldk)
  double* d_D1 = nullptr;          // DC2DE first factor             (kept_dn x ldn)
  double* d_D2 = nullptr;          // DC2DE second factor            (neq x ldk)
  double* d_m2m = nullptr;         // 8 x (neq_pad x ldn)
  double* d_l2l = nullptr;         // 8 x (neq_pad x ldn)
  double* d_m2l = nullptr;         // 316 x (neq_pad x ldn)
  int64_t op_stride = 0;           // elements between consecutive n x n operators
  int rows_pad = 0;                // neq rounded up to GEMM_BM
  std::vector<double> h_sigma;

  // FFT M2L (convolution on the NG^3 lattice grid, NG = 2p - 1)
  int m2l_mode = M2L_FFT;
  int NG = 0, NZ = 0, NF = 0;      // grid, half-spectrum NG/2+1, bins NG*NG*NZ
  // frequency groups of the sparse-chunk product: NFG groups of 32 slots, each a union
  // of whole orbits {(+-fx, +-fy, fz)}; spectra rows are stored in group-slot order
  // (position fpos[f] = 32 g + slot), NFP = 32 NFG >= NF positions per row
  int NFG = 0, NFP = 0;
  int16_t* d_fpos = nullptr;       // [NF] position of frequency f
  int* d_rslot = nullptr;          // [NFG][32] slots of R f, R in {id, x, y, xy reflections}, 4 x 5 bits
  double2* d_tbase = nullptr;      // [NFG][56][ncomp][32] spectra of the 56 offsets with o >= 0
  int ncomp = 0;                   // stored components per operator spectrum: 1 (L) or 6 (sym. G)
  double2* d_that = nullptr;       // [NF][316][ncomp] operator spectra at level 0
  int16_t* d_lat = nullptr;        // M x 3 integer lattice coordinates of the surface points
  int16_t* d_lmap = nullptr;       // p^3 lattice -> surface index or -1 (FFT forward z pass)
  int16_t* d_aidx = nullptr;       // DMMA A-fragment gather table [26][8kml/4][kml][32]
  double *d_wz = nullptr, *d_wf = nullptr, *d_wi = nullptr;  // DFT-pass twiddle fragments
  std::vector<FftChunk> fft_chunks;
  double2* d_ub = nullptr;         // source spectra: dense chunks [NF][nq][8 kml], sparse chunks [NFG][nq][8 kml][32]
  double2* d_cb = nullptr;         // [npar][8 kml][NFP] target check spectra, target-major, group-slot order
  int64_t fft_max_nq = 0, fft_max_npar = 0, fft_budget = 0;

  Jobs J;
  bool restricted = false;
  // heavy per-box rows: UE / CHK / DE / T row of box b is d_row[b] (identity for a
  // single-GPU plan; compacted to active + shared + ghost boxes on a rank)
  int64_t nrow = 0;
  int32_t* d_row = nullptr;
  int32_t* d_crow = nullptr;       // 8 per box: row of the child, or -1 (FFT forward)
  std::vector<int32_t> h_row;      // host copy (empty: identity)
  int64_t nloc = 0;                // points with source records (n, or owned + ghost on a rank)
  int64_t* d_operm = nullptr;      // scatter_out: Morton position -> output row (d_perm unless partitioned)
  DistState* dist = nullptr;
  // kafmm_setup2: rows [0, n_src) of the union are sources, the rest targets
  int64_t n_src = -1;
  double* d_uvals = nullptr;   // union source values (target rows stay zero)
  double* d_uout = nullptr;    // union outputs

  // GEMM batches
  GemmBatch g_uc2ue_1, g_uc2ue_2;              // S2M leaves (level >= 2)
  std::vector<GemmBatch> g_m2m;                // per parent level, bottom-up order
  GemmBatch g_m2l;
  std::vector<GemmBatch> g_dc2de_1, g_dc2de_2, g_l2l;  // per level (2..depth)

  // workspaces (device)
  double* d_rec = nullptr;         // n x srec sorted source records
  double* d_outs = nullptr;        // n x kt sorted outputs
  double* d_ue = nullptr;          // nbox x ldn
  double* d_chk = nullptr;         // nbox x ldn (upward check at leaves, then downward check)
  double* d_de = nullptr;          // nbox x ldn
  double* d_t = nullptr;           // nbox x ldk (first-factor temporaries)
  double* d_stage_in = nullptr;    // n x ks (eval_host staging)
  double* d_stage_out = nullptr;   // n x kt
  int* d_flag = nullptr;
  int64_t bytes = 0;

  std::vector<void*> allocs;
  std::vector<int64_t> alloc_bytes;  // size of allocs[i] (plan byte count after dfree)
};

// error handling -----------------------------------------------------------
void set_error(const std::string& msg);
struct Error {
  kafmm_status st;
  std::string msg;
};
#define KF_CUDA(call)                                                                        \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      throw ::kafmm::Error{e_ == cudaErrorMemoryAllocation ? KAFMM_ENOMEM : KAFMM_ECUDA,     \
                           std::string(#call) + ": " + cudaGetErrorString(e_)};              \
  } while (0)
#define KF_CHECK_LAUNCH() KF_CUDA(cudaGetLastError())

template <class T>
T* dalloc(Plan& P, size_t count) {
  void* p = nullptr;
  size_t b = count * sizeof(T);
  if (b == 0) b = 8;
  KF_CUDA(cudaMalloc(&p, b));
  KF_CUDA(cudaMemsetAsync(p, 0, b, P.stream));
  P.allocs.push_back(p);
  P.alloc_bytes.push_back((int64_t)b);
  P.bytes += (int64_t)b;
  return (T*)p;
}

// release a dalloc'ed buffer early (re-planning after kafmm_restrict)
inline void dfree(Plan& P, void* p) {
  if (!p) return;
  for (size_t i = 0; i < P.allocs.size(); ++i)
    if (P.allocs[i] == p) {
      cudaFree(p);
      P.allocs[i] = nullptr;
      P.bytes -= P.alloc_bytes[i];
      P.alloc_bytes[i] = 0;
    }
}

inline void free_batch(Plan& P, GemmBatch& g) {
  dfree(P, g.d_tiles);
  if (g.owns_items) dfree(P, g.d_items);
  g = GemmBatch();
}

// event around an M2L product launch (stage timing only)
inline void prod_mark(Plan& P) {
  if (!P.timing) return;
  if ((int)P.prod_ev.size() <= P.prod_used) {
    cudaEvent_t e;
    KF_CUDA(cudaEventCreate(&e));
    P.prod_ev.push_back(e);
  }
  KF_CUDA(cudaEventRecord(P.prod_ev[P.prod_used++], P.stream));
}

inline int round_up(int a, int b) { return (a + b - 1) / b * b; }

// translation units
void build_tree_and_lists(Plan& P, const double* d_points);   // kafmm_tree.cu
void build_operators(Plan& P);                               // kafmm_ops.cu
void build_dense_m2l(Plan& P);                               // kafmm_ops.cu (lazy)
void build_gemm_batches(Plan& P);                            // kafmm_tree.cu
void upload_batch(Plan& P, GemmBatch& g, const std::vector<int2>& h_items);
void run_eval(Plan& P, const double* d_src, double* d_out);  // kafmm_eval.cu
void run_eval_up(Plan& P, const double* d_src);               // a1-a4
void run_eval_down(Plan& P, double* d_out);
void run_eval_s2l(Plan& P);  // CHK reset + S2L ahead of M2L (multi-GPU overlap); run_eval_down then skips them                   // a5-a12
void build_m2l_batch(Plan& P);                                // kafmm_dist.cu
void setup_dist(Plan& P, const double* d_local_points, int64_t n_local);  // kafmm_dist.cu (P.dist->comm set)
void run_eval_dist(Plan& P, const double* d_local_src, double* d_local_out);
void alloc_workspaces(Plan& P);                               // kafmm_capi.cu
void build_plan_core(Plan& P, const double* d_points);        // kafmm_capi.cu: tree, lists, operators, batches
void check_values(Plan& P, const double* d_src);
void take_nonfinite(Plan& P);             // kafmm_eval.cu
void launch_gemm(Plan& P, const GemmBatch& g, const double* A, int M, int K, int lda,
                 const double* B, int ldb, double* C, int ldc, int mode);  // kafmm_gemm.cu
void build_fft_m2l(Plan& P, int64_t budget_bytes);           // kafmm_fft.cu
void build_fft_chunks(Plan& P, int64_t budget_bytes);        // kafmm_fft.cu
void run_m2l_fft(Plan& P);                                   // kafmm_fft.cu

}  // namespace kafmm

// the opaque ABI handle is the plan itself
struct kafmm_plan_s : public kafmm::Plan {};
