// Grouped gather-GEMM on the FP64 tensor cores (DMMA.8x8x4, sm_100a).
//
// Every per-box translation of the evaluation pass is a small dense product
// y_out = alpha * A_op * x_in between an n x n (or kept x n) operator and
// box vectors:
//   UC2UE / DC2DE   A = S^-1 U^T then V                 (two launches)
//   M2M             A = M2M[octant(child)], atomic into the parent
//   M2L             A = M2L[offset], alpha = 2^level, atomic into the target
//   L2L             A = L2L[octant(child)], added into the child
// Items (input column, output column) that share one operator are grouped
// into tiles of 64 on the host at setup; a CTA computes a 128-row x 64-item
// block of one tile, so the operator tile is reused across 64 box vectors and
// the 64 gathered box vectors across 128 operator rows.
//
// FP64 tensor cores on sm_100a are warp-level `mma.sync ... f64` (tcgen05
// has no f64 kind), so this is a classic cp.async multistage pipeline:
// 3 stages of A (128 x 16) and B (64 x 16) in shared memory, 8 warps each
// owning a 32 x 32 accumulator block (16 DMMA per k4 step).
#include "kafmm_internal.h"

namespace kafmm {

constexpr int BM = GEMM_BM, BN = GEMM_BN, BK = GEMM_BK;
constexpr int STAGES = 3;
constexpr int SA = BK + 4;  // padded row stride (doubles): conflict-free 64-bit fragment loads
constexpr int THREADS = 256;
constexpr size_t GEMM_SMEM = (size_t)STAGES * (BM + BN) * SA * sizeof(double);

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int MODE>
__global__ void __launch_bounds__(THREADS, 2)
    k_gemm_dmma(const double* __restrict__ A, int64_t a_stride, int lda, int M, int K, const double* __restrict__ B,
                int ldb, double* __restrict__ C, int ldc, const GemmTile* __restrict__ tiles,
                const int2* __restrict__ items) {
  extern __shared__ __align__(16) double smem[];
  double* As = smem;                      // [STAGES][BM][SA]
  double* Bs = smem + STAGES * BM * SA;   // [STAGES][BN][SA]
  __shared__ int s_in[BN], s_out[BN];
  // flattened grid: row blocks fastest, so the CTAs sharing one tile's 64
  // gathered vectors run together and hit them in L2
  const int nrb = (M + BM - 1) / BM;
  const GemmTile t = tiles[blockIdx.x / nrb];
  const int m0 = (blockIdx.x % nrb) * BM;
  const int tid = threadIdx.x;
  if (tid < BN) {
    if (tid < t.nitem) {
      int2 it = items[t.item0 + tid];
      s_in[tid] = it.x;
      s_out[tid] = it.y;
    } else {
      s_in[tid] = -1;
      s_out[tid] = -1;
    }
  }
  __syncthreads();
  const double* Ab = A + (int64_t)t.op * a_stride + (int64_t)m0 * lda;
  const int KT = K / BK;

  auto load_stage = [&](int s, int kt) {
    const int k0 = kt * BK;
#pragma unroll
    for (int q = 0; q < (BM * BK / 2) / THREADS; ++q) {
      int c = tid + THREADS * q;
      int row = c >> 3, kk = (c & 7) * 2;
      cp_async16(&As[(s * BM + row) * SA + kk], Ab + (int64_t)row * lda + k0 + kk, 16);
    }
#pragma unroll
    for (int q = 0; q < (BN * BK / 2) / THREADS; ++q) {
      int c = tid + THREADS * q;
      int it = c >> 3, kk = (c & 7) * 2;
      int col = s_in[it];
      const double* src = col >= 0 ? B + (int64_t)col * ldb + k0 + kk : B;
      cp_async16(&Bs[(s * BN + it) * SA + kk], src, col >= 0 ? 16 : 0);
    }
  };

  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp & 3, wn = warp >> 2;
  const int g = lane >> 2, tq = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_stage(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      int nk = kt + STAGES - 1;
      if (nk < KT) load_stage(nk % STAGES, nk);
      cp_async_commit();
    }
    const int s = kt % STAGES;
    const double* as = As + (s * BM + wm * 32 + g) * SA + tq;
    const double* bs = Bs + (s * BN + wn * 32 + g) * SA + tq;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = as[i * 8 * SA + ks * 4];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = bs[j * 8 * SA + ks * 4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_async_wait<0>();

  const double alpha = t.alpha;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + wm * 32 + i * 8 + g;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int oc = s_out[wn * 32 + j * 8 + 2 * tq + e];
        if (oc < 0) continue;
        double* dst = C + (int64_t)oc * ldc + row;
        const double v = alpha * acc[i][j][e];
        if (MODE == GEMM_STORE) *dst = v;
        else if (MODE == GEMM_ADD) *dst += v;
        else atomicAdd(dst, v);
      }
    }
  }
}

void launch_gemm(Plan& P, const GemmBatch& g, const double* A, int M, int K, int lda, const double* B, int ldb,
                 double* C, int ldc, int mode) {
  if (g.ntiles() == 0) return;
  static std::atomic<uint64_t> init{0};
  if (first_on_device(init)) {
    KF_CUDA(cudaFuncSetAttribute(k_gemm_dmma<GEMM_STORE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GEMM_SMEM));
    KF_CUDA(cudaFuncSetAttribute(k_gemm_dmma<GEMM_ADD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GEMM_SMEM));
    KF_CUDA(cudaFuncSetAttribute(k_gemm_dmma<GEMM_ATOMIC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GEMM_SMEM));
  }
  if (K % BK != 0 || lda % 2 != 0 || ldb % 2 != 0) throw Error{KAFMM_EINVAL, "gemm: bad padding"};
  dim3 grid((unsigned)(((M + BM - 1) / BM) * (int64_t)g.ntiles()));
  if (mode == GEMM_STORE)
    k_gemm_dmma<GEMM_STORE><<<grid, THREADS, GEMM_SMEM, P.stream>>>(A, P.op_stride, lda, M, K, B, ldb, C, ldc,
                                                                    g.d_tiles, g.d_items);
  else if (mode == GEMM_ADD)
    k_gemm_dmma<GEMM_ADD><<<grid, THREADS, GEMM_SMEM, P.stream>>>(A, P.op_stride, lda, M, K, B, ldb, C, ldc,
                                                                  g.d_tiles, g.d_items);
  else
    k_gemm_dmma<GEMM_ATOMIC><<<grid, THREADS, GEMM_SMEM, P.stream>>>(A, P.op_stride, lda, M, K, B, ldb, C, ldc,
                                                                     g.d_tiles, g.d_items);
  KF_CHECK_LAUNCH();
  P.launches++;
}

}  // namespace kafmm
