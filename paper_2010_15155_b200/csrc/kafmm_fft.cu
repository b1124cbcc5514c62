// M2L as a convolution on the regular lattice grid (SURVEY.md §8(a) a5,
// option b; the paper's M2L cost remark P:633 refers to PVFMM's FFT M2L).
//
// The upward-equivalent surface of a source box C and the downward-check
// surface of a target box B (both radius 1.05 h) are boundary points of p^3
// lattices with the same spacing delta = 2*1.05 h/(p-1).  For C = B + 2h o,
//     check_B(I) = sum_J K(delta (I - J) - 2 h o) ue_C(J),   I, J in [0,p)^3,
// a 3D linear convolution with the kernel grid t_o(D) = K(delta D - 2 h o),
// D in [-(p-1), p-1]^3.  Zero-padded to NG = 2p - 1 (the smallest size at
// which D -> D mod NG is one-to-one) it is a circular convolution:
//     check_B = IDFT( sum_{C in V(B)} That_o . DFT(ue_C) )  on the lattice.
// This is exactly the dense M2L (up to rounding): same matrices, factored.
//
// Hot path per level and chunk (all on the plan's stream):
//   k_fft_fwd   one CTA per (source parent, child octant): real DFT of ue (p^3
//               cube, surface only non-zero), staged z, y, x in shared memory,
//               -> ub[f][parent][8 kml] (frequency-major, zero for a missing child)
//   k_m2l_dmma  per frequency a complex GEMM over target parents: the 26
//               colleague directions x 8x8 (target child, source child) blocks,
//               o = 2d + oct(c) - oct(b), adjacent pairs zero (PVFMM-style
//               blocking), on the FP64 tensor cores (DMMA.8x8x4)
//   k_fft_inv   one CTA per target box: inverse DFT, evaluated only at the
//               downward-check surface points, times 2^l / NG^3, added to CHK
// Operator spectra That_o (316 offsets, level 0) are computed once at setup
// with cuFFT (setup only; not on the hot path).
#include <cufft.h>

#include <algorithm>
#include <numeric>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "kafmm_internal.h"
#include "kafmm_spos.h"

namespace kafmm {

static inline unsigned nblk(int64_t n, int t = 256) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

// ---------------------------------------------------------------------------
// setup: kernel grids t_o and their spectra
// ---------------------------------------------------------------------------
// grid index -> lattice difference D in [-(p-1), p-1] (NG >= 2p - 1), or INT_MIN for padding
__device__ __forceinline__ int dmap(int g, int p, int NG) {
  return g < p ? g : (g >= NG - (p - 1) ? g - NG : INT_MIN);
}

__global__ void k_kernel_grid(int p, int NG, int kml, double delta, const int8_t* __restrict__ offs, double* grid) {
  const int NG3 = NG * NG * NG;
  int g = blockIdx.x * blockDim.x + threadIdx.x;
  int o = blockIdx.y;
  if (g >= NG3) return;
  int gx = g / (NG * NG), gy = (g / NG) % NG, gz = g % NG;
  int Dx = dmap(gx, p, NG), Dy = dmap(gy, p, NG), Dz = dmap(gz, p, NG);
  int nc = kml == 1 ? 1 : 6;
  double* out = grid + (int64_t)o * nc * NG3 + g;
  if (Dx == INT_MIN || Dy == INT_MIN || Dz == INT_MIN) {
    for (int c = 0; c < nc; ++c) out[(int64_t)c * NG3] = 0.0;
    return;
  }
  // level 0: h = 1/2, so 2 h o = o
  double rx = delta * Dx - offs[3 * o], ry = delta * Dy - offs[3 * o + 1], rz = delta * Dz - offs[3 * o + 2];
  double ri = rsqrt(rx * rx + ry * ry + rz * rz);
  if (kml == 1) {
    out[0] = ri;
  } else {
    double ri3 = ri * ri * ri;
    out[0 * (int64_t)NG3] = ri + rx * rx * ri3;
    out[1 * (int64_t)NG3] = rx * ry * ri3;
    out[2 * (int64_t)NG3] = rx * rz * ri3;
    out[3 * (int64_t)NG3] = ri + ry * ry * ri3;
    out[4 * (int64_t)NG3] = ry * rz * ri3;
    out[5 * (int64_t)NG3] = ri + rz * rz * ri3;
  }
}

__global__ void k_spectra_transpose(int NF, int nc, const double2* __restrict__ in, double2* __restrict__ that) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // over [316][nc][NF]
  if (t >= (int64_t)N_OFFSETS * nc * NF) return;
  int f = (int)(t % NF);
  int64_t oc = t / NF;
  int c = (int)(oc % nc), o = (int)(oc / nc);
  that[((int64_t)f * N_OFFSETS + o) * nc + c] = in[t];
}

// ---------------------------------------------------------------------------
// hot path kernels
// ---------------------------------------------------------------------------
// Padded row lengths (complex entries) of the shared-memory arrays of the DFT passes:
// forward z output [x y][fz] (ZS), forward y output [x][fy][fz] (YS), extra doubles between
// the transforms of one CTA (FPAD), inverse x output [x][fy][fz] (DS) and y output
// [x][y][fz] (ES).  Chosen by scripts/fft_banks.py, which replays every fragment load and
// store of the passes and counts shared-memory wavefronts; unpadded rows of NZ = p
// entries (p = 8: 128 B) put a warp's lines or outputs in one bank group (ncu, C5: 62-67%
// of the DFT passes' wavefronts were bank conflicts, profiles/r02_C5_dft_ncu.txt).
template <int P>
struct FftPad {  // {ZS, YS, FPAD, DS, ES}; NZ = P
  static constexpr int T[8][5] = {{5, 6, 8, 9, 3},     {4, 6, 8, 6, 6},     {12, 6, 4, 6, 6},  {12, 6, 0, 6, 6},
                                  {12, 10, 4, 10, 10}, {12, 10, 8, 10, 10}, {12, 10, 0, 10, 10},
                                  {12, 14, 8, 14, 14}};
  static constexpr int I = P <= 8 ? P - 3 : (P == 10 ? 6 : 7);
  static constexpr int ZS = T[I][0], YS = T[I][1], FPAD = T[I][2], DS = T[I][3], ES = T[I][4];
};

template <int P>
struct FftDims {
  static constexpr int NG = 2 * P - 1, NZ = NG / 2 + 1, NF = NG * NG * NZ;
  static_assert(FftPad<P>::ZS >= NZ && FftPad<P>::YS >= NZ && FftPad<P>::DS >= NZ && FftPad<P>::ES >= NZ, "pad");
  // inverse: x-pass output [x][fy][fz] + y-pass output [x][y][fz] (complex, padded rows) + twiddles
  static constexpr size_t INV_SMEM =
      (size_t)2 * (P * NG * FftPad<P>::DS + P * P * FftPad<P>::ES + NG) * sizeof(double);
};

__device__ __forceinline__ void cmac(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// The DFT passes run as small real GEMMs on the FP64 tensor cores: a pass maps
// the NIN inputs of every line to NOUT complex outputs,
//     out[line][o] = sum_i in[line][i] w^(s o i),  w = exp(2 pi i / NG),
// written as C[line][(o, re|im)] = sum_(i, re|im) A[line][(i, re|im)] B[(i, .)][(o, .)]
// with B the 2x2 real blocks of the twiddles (1x2 for a real input).  Lines
// are the M dimension (8 per DMMA), the twiddle matrix B sits in registers for
// the whole pass (one table per pass shape, built at setup), and a lane's C
// fragment holds the (re, im) pair of one output, stored as one 16-B word.
template <int P>
struct DftShape {
  static constexpr int NG = 2 * P - 1, NZ = NG / 2 + 1;
  // forward z (real in: P -> NZ), forward y / x (complex: P -> NG), inverse x / y (complex: NG -> P)
  static constexpr int KZ = (P + 3) / 4, NZT = (2 * NZ + 7) / 8;
  static constexpr int KF = (2 * P + 3) / 4, NFT = (2 * NG + 7) / 8;
  static constexpr int KI = (2 * NG + 3) / 4, NIT = (2 * P + 7) / 8;
};

// fragment tables: [ks][nt][lane] twiddle block entries (host-built, see
// build_fft_m2l) in global memory; a lane reads its own entry right before
// each DMMA (coalesced, L1-resident: every CTA of the launch reads the same
// few KB), which keeps the register count low and costs no shared memory

#ifndef KF_DFT_MT
#define KF_DFT_MT 2
#endif
// MT m-tiles of 8 lines at once (independent DMMA accumulator chains: the
// passes are short, NKS <= 12, so one tile's chains alone leave the tensor
// pipe waiting on DMMA latency)
template <int MT, int NKS, int NNT, class LoadA, class StoreC>
__device__ __forceinline__ void dft_tiles(int mt0, int mstep, int nlines, int nout, const double* __restrict__ wtab,
                                          LoadA& loadA, StoreC& storeC) {
  const int lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  int line[MT];
  bool ok[MT];
  double acc[MT][NNT][2];
#pragma unroll
  for (int u = 0; u < MT; ++u) {
    line[u] = (mt0 + u * mstep) * 8 + g;
    ok[u] = line[u] < nlines;
#pragma unroll
    for (int n = 0; n < NNT; ++n) acc[u][n][0] = acc[u][n][1] = 0.0;
  }
#pragma unroll
  for (int k = 0; k < NKS; ++k) {
    double a[MT];
#pragma unroll
    for (int u = 0; u < MT; ++u) a[u] = ok[u] ? loadA(line[u], 4 * k + tq) : 0.0;
#pragma unroll
    for (int n = 0; n < NNT; ++n) {
      const double w = __ldg(wtab + (k * NNT + n) * 32 + lane);
#pragma unroll
      for (int u = 0; u < MT; ++u) dmma(acc[u][n][0], acc[u][n][1], a[u], w);
    }
  }
#pragma unroll
  for (int u = 0; u < MT; ++u)
    if (ok[u]) {
#pragma unroll
      for (int n = 0; n < NNT; ++n) {
        const int o = 4 * n + tq;
        if (o < nout) storeC(line[u], o, make_double2(acc[u][n][0], acc[u][n][1]));
      }
    }
}

// one pass over nlines lines by the CTA's warps; loadA(line, k) -> double,
// storeC(line, o, double2) for o < nout
template <int NKS, int NNT, class LoadA, class StoreC>
__device__ __forceinline__ void dft_pass(int nlines, int nout, const double* __restrict__ wtab, LoadA loadA,
                                         StoreC storeC) {
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int ntile = (nlines + 7) / 8;
  int mt = warp;
#if KF_DFT_MT > 1
  for (; mt + (KF_DFT_MT - 1) * nw < ntile; mt += KF_DFT_MT * nw)
    dft_tiles<KF_DFT_MT, NKS, NNT>(mt, nw, nlines, nout, wtab, loadA, storeC);
#endif
  for (; mt < ntile; mt += nw) dft_tiles<1, NKS, NNT>(mt, nw, nlines, nout, wtab, loadA, storeC);
}

// forward: one CTA per (source parent block q, group of NB transform slots);
// slot s = c kml + e is (child octant c, component e), the order of ub's last
// index.  Each transform: the child's upward equivalent density on the p^3
// lattice (non-zero on the surface only) -> its real DFT on the NG^3 grid,
// z (real -> half spectrum), y, x passes on the tensor cores over the lines of
// all the group's transforms at once.  The z pass reads the density straight
// from UE through the lattice -> surface-index map (no dense p^3 cube in
// shared memory); the x pass has the transform index fastest, so one
// frequency's stores are consecutive 16-B words.  A missing child's slots are
// zero-filled when the chunk's product reads parent blocks, else skipped.
template <int P>
struct FwdCfg {
  using D = FftDims<P>;
  // doubles per transform (z, y outputs, padded rows)
  static constexpr int PER = 2 * (P * P * FftPad<P>::ZS + P * D::NG * FftPad<P>::YS) + FftPad<P>::FPAD;
  template <int NB>
  static constexpr size_t smem() { return (size_t)NB * PER * sizeof(double); }
};

template <int N, class T>
__device__ __forceinline__ T pick(const T (&a)[N], int t, int n) {  // a[t] without local memory
  T r = a[0];
#pragma unroll
  for (int j = 1; j < N; ++j)
    if (j < n && t == j) r = a[j];
  return r;
}

template <int P, int NB, int NBC>
__device__ __forceinline__ void fwd_body(double* __restrict__ sm, const double* (&src)[NB], const int (&slot)[NB],
                                         const int16_t* __restrict__ lmap, int kml, double2* __restrict__ ub,
                                         int64_t nq, int64_t q, int R, const double* __restrict__ wz,
                                         const double* __restrict__ wf, const int16_t* __restrict__ fpos) {
  using D = FftDims<P>;
  using S = DftShape<P>;
  constexpr int NG = D::NG, NZ = D::NZ, NGNZ = NG * NZ, PER = FwdCfg<P>::PER, PP = P * P;
  constexpr int ZS = FftPad<P>::ZS, YS = FftPad<P>::YS, YO = 2 * PP * ZS;
  dft_pass<S::KZ, S::NZT>(  // z: lines (t; x, y), real input from UE
      PP * NBC, NZ, wz,
      [&](int L, int k) {
        const int t = L / PP, xy = L - t * PP;
        if (k >= P) return 0.0;
        const int m = __ldg(lmap + xy * P + k);
        return m >= 0 ? __ldg(pick<NB>(src, t, NBC) + m * kml) : 0.0;
      },
      [&](int L, int o, double2 v) {
        const int t = L / PP, xy = L - t * PP;
        reinterpret_cast<double2*>(sm + t * PER)[xy * ZS + o] = v;
      });
  __syncthreads();
  dft_pass<S::KF, S::NFT>(  // y: lines (t; x, fz)
      P * NZ * NBC, NG, wf,
      [&](int L, int k) {
        const int t = L / (P * NZ), r = L - t * (P * NZ), x = r / NZ, fz = r - x * NZ, y = k >> 1;
        return y < P ? sm[t * PER + 2 * ((x * P + y) * ZS + fz) + (k & 1)] : 0.0;
      },
      [&](int L, int o, double2 v) {
        const int t = L / (P * NZ), r = L - t * (P * NZ), x = r / NZ, fz = r - x * NZ;
        reinterpret_cast<double2*>(sm + t * PER + YO)[(x * NG + o) * YS + fz] = v;
      });
  __syncthreads();
  dft_pass<S::KF, S::NFT>(  // x: lines (fy, fz; t) -> global, frequency major
      NGNZ * NBC, NG, wf,
      [&](int L, int k) {
        const int r = L / NBC, t = L - r * NBC, x = k >> 1, fy = r / NZ, fz = r - fy * NZ;
        return x < P ? sm[t * PER + YO + 2 * ((x * NG + fy) * YS + fz) + (k & 1)] : 0.0;
      },
      [&](int L, int o, double2 v) {
        const int r = L / NBC, t = L - r * NBC, f = o * NGNZ + r, sl = pick<NB>(slot, t, NBC);
        if (fpos) {  // sparse chunks: [group][q][R][slot] (k_m2l_items)
          const int fp = __ldg(fpos + f);
          ub[(((int64_t)(fp >> 5) * nq + q) * R + sl) * 32 + (fp & 31)] = v;
        } else
          ub[((int64_t)f * nq + q) * R + sl] = v;
      });
}

template <int P, int NB, int NBC>
__device__ __forceinline__ void fwd_dispatch(int nb, double* sm, const double* (&src)[NB], const int (&slot)[NB],
                                             const int16_t* lmap, int kml, double2* ub, int64_t nq, int64_t q, int R,
                                             const double* wz, const double* wf, const int16_t* fpos) {
  if (nb == NBC) fwd_body<P, NB, NBC>(sm, src, slot, lmap, kml, ub, nq, q, R, wz, wf, fpos);
  else if constexpr (NBC > 1)
    fwd_dispatch<P, NB, NBC - 1>(nb, sm, src, slot, lmap, kml, ub, nq, q, R, wz, wf, fpos);
}

template <int P, int NB>
__global__ void __launch_bounds__(256)
    k_fft_fwd(const int32_t* __restrict__ qbox, const int32_t* __restrict__ child, int64_t nq,
              const double* __restrict__ ue, int ldn, int kml, const int16_t* __restrict__ lmap,
              double2* __restrict__ ub, int zero_missing, const double* __restrict__ wz,
              const double* __restrict__ wf, const int16_t* __restrict__ fpos) {
  using D = FftDims<P>;
  constexpr int NF = D::NF;
  extern __shared__ __align__(16) double sm[];
  const int R = 8 * kml;
  const int ng = (R + NB - 1) / NB;
  const int64_t q = blockIdx.x / ng;
  const int s0 = (blockIdx.x % ng) * NB;
  const int64_t qb = qbox[q];
  // this CTA's transforms, compacted: slots with an existing child
  const double* src[NB];
  int slot[NB];
  int nb = 0;
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    src[j] = ue;
    slot[j] = 0;
  }
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const int sl = s0 + j;
    if (sl >= R) break;
    const int64_t b = child[8 * qb + sl / kml];
    if (b >= 0) {
#pragma unroll
      for (int i = 0; i < NB; ++i)
        if (i == nb) {
          src[i] = ue + b * ldn + sl % kml;
          slot[i] = sl;
        }
      ++nb;
    } else if (zero_missing) {
      for (int f = threadIdx.x; f < NF; f += blockDim.x) ub[((int64_t)f * nq + q) * R + sl] = make_double2(0.0, 0.0);
    }
  }
  if (nb == 0) return;
  fwd_dispatch<P, NB, NB>(nb, sm, src, slot, lmap, kml, ub, nq, q, R, wz, wf, zero_missing ? nullptr : fpos);
}

// inverse: one CTA per target box; its check spectrum cb[parent][b kml + a][f] (one contiguous row,
// read by the x pass straight from global memory) -> x and y passes on the tensor cores (outputs
// only for x, y < p), the z pass evaluated only at the downward-check surface points, times
// 2^l / NG^3, added to CHK.  NG is odd, so there is no Nyquist bin.
template <int P>
__global__ void __launch_bounds__(256)
    k_fft_inv(const int32_t* __restrict__ tbox, const int2* __restrict__ tpb, int64_t npar,
              int lev, const double2* __restrict__ cb, int kml,
              const int16_t* __restrict__ lat, int M, double* __restrict__ chk, int ldn,
              const double* __restrict__ wi, const int16_t* __restrict__ fpos, int NFP) {
  using D = FftDims<P>;
  using S = DftShape<P>;
  constexpr int NG = D::NG, NZ = D::NZ, NGNZ = NG * NZ;
  extern __shared__ __align__(16) double sm[];
  constexpr int DS = FftPad<P>::DS, ES = FftPad<P>::ES;
  double2* Dx = reinterpret_cast<double2*>(sm);  // [x][fy][fz], rows of DS
  double2* E = Dx + P * NG * DS;                 // [x][y][fz], rows of ES
  double2* tw = E + P * P * ES;                  // exp(+2 pi i j / NG)
  const double* Dd = reinterpret_cast<const double*>(Dx);
  const int t = blockIdx.x, tid = threadIdx.x, bd = blockDim.x;
  const int64_t box = tbox[t];
  const int2 pb = tpb[t];
  const int R = 8 * kml;
  const double scale = ldexp(1.0, lev) / (double)(NG * NG * NG);
  for (int j = tid; j < NG; j += bd) {
    double sn, cs;
    sincospi(2.0 * j / NG, &sn, &cs);
    tw[j] = make_double2(cs, sn);
  }
  __syncthreads();
  for (int a = 0; a < kml; ++a) {
    // target-major: one contiguous row, frequency f at position fpos[f]
    const double* col = reinterpret_cast<const double*>(cb + ((int64_t)pb.x * R + pb.y * kml + a) * NFP);
    dft_pass<S::KI, S::NIT>(  // x: lines (fy, fz), outputs x < P
        NGNZ, P, wi,
        [&](int line, int k) {
          const int fx = k >> 1;
          return fx < NG ? __ldg(col + 2 * __ldg(fpos + fx * NGNZ + line) + (k & 1)) : 0.0;
        },
        [&](int line, int o, double2 v) {
          const int fy = line / NZ, fz = line - fy * NZ;
          Dx[(o * NG + fy) * DS + fz] = v;
        });
    __syncthreads();
    dft_pass<S::KI, S::NIT>(  // y: lines (x, fz), outputs y < P
        P * NZ, P, wi,
        [&](int line, int k) {
          const int x = line / NZ, fz = line - x * NZ, fy = k >> 1;
          return fy < NG ? Dd[2 * ((x * NG + fy) * DS + fz) + (k & 1)] : 0.0;
        },
        [&](int line, int o, double2 v) {
          const int x = line / NZ, fz = line - x * NZ;
          E[(x * P + o) * ES + fz] = v;
        });
    __syncthreads();
    double* o = chk + box * ldn;
    for (int m = tid; m < M; m += bd) {  // z: half spectrum -> real, only at surface points
      int x = lat[3 * m], y = lat[3 * m + 1], z = lat[3 * m + 2];
      const double2* e = E + (x * P + y) * ES;
      double v = 0.0;
      int k = z;
      for (int fz = 1; fz < NZ; ++fz) {
        v = fma(e[fz].x, tw[k].x, fma(-e[fz].y, tw[k].y, v));
        k += z;
        if (k >= NG) k -= NG;
      }
      o[m * kml + a] += scale * fma(2.0, v, e[0].x);
    }
    __syncthreads();
  }
}

// Hadamard stage on the FP64 tensor cores.  For one frequency f and a target
// parent P, with Q_d the colleague of P in direction d (26 of them):
//     C_P(f)[b, a] = sum_d sum_{c, e} T_{o(d,c,b)}(f)[a, e] U_{Q_d}(f)[c, e],
//     o(d, c, b) = 2 d + oct(c) - oct(b),  T = 0 for adjacent (c, b)
// i.e. per frequency a complex GEMM  C[8k x npar] = A_f[8k x 26*8k] B_f
// whose A is the same for every parent.  A warp owns all 8k rows and NT x 8
// parents; the A fragments are gathered from the frequency's operator spectra
// in shared memory through a precomputed index table, the B fragments are the
// colleagues' child blocks (one 16-B load per lane), and a complex product is
// three DMMA.8x8x4 (Gauss / Karatsuba): with A = a + ib, B = c + id,
//     P1 = sum a c,  P2 = sum b d,  P3 = sum (a + b)(c + d),
//     Re = P1 - P2,  Im = P3 - P1 - P2,
// the sums a + b and c + d formed in registers (one DADD per fragment),
// the three accumulators combined once in the epilogue.
#ifndef KF_DM_WARPS
#define KF_DM_WARPS 4
#endif
constexpr int DM_WARPS = KF_DM_WARPS;

#ifndef KF_DMMA_MINB1
#define KF_DMMA_MINB1 1
#endif
#ifndef KF_DMMA_MINB3
#define KF_DMMA_MINB3 4  // Stokes family: cap 128 registers, 4 CTAs per SM (C3 product -14%, profiles/r01_dmma_ab.txt)
#endif
__device__ const int16_t d_spos1[N_OFFSETS] = KF_SPOS1_INIT;
__device__ const int16_t d_spos3[N_OFFSETS * 6] = KF_SPOS3_INIT;

template <int KML, int NT>
__global__ void __launch_bounds__(DM_WARPS * 32, KML == 1 ? KF_DMMA_MINB1 : KF_DMMA_MINB3)
    k_m2l_dmma(int64_t npar, int64_t nq, int npb, const double2* __restrict__ that, const double2* __restrict__ ub,
               double2* __restrict__ cb, const int32_t* __restrict__ nbr, const int16_t* __restrict__ aidx,
               const int16_t* __restrict__ fpos, int NFP) {
  constexpr int NC = KML == 1 ? 1 : 6, R = 8 * KML, KS = R / 4, PPW = NT * 8;
  // the frequency's spectra at the bank-conflict-minimising positions of kafmm_spos.h
  // (the A-fragment gather below reads them through aidx, which holds those positions)
  __shared__ double2 sT[KML == 1 ? SPOS1_N : SPOS3_N];
  const int16_t* spos = KML == 1 ? d_spos1 : d_spos3;
  const int64_t f = blockIdx.x / npb;
  const int pb = blockIdx.x % npb;
  for (int i = threadIdx.x; i < N_OFFSETS * NC; i += DM_WARPS * 32) sT[spos[i]] = that[f * N_OFFSETS * NC + i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int64_t P0 = ((int64_t)pb * DM_WARPS + warp) * PPW;
  if (P0 >= npar) return;
  double acc[KML][NT][3][2];  // P1, P2, P3 (see above)
#pragma unroll
  for (int m = 0; m < KML; ++m)
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int k = 0; k < 3; ++k) acc[m][n][k][0] = acc[m][n][k][1] = 0.0;
  const double2* ubf = ub + f * nq * R;
  int qn[NT];  // colleague block of the next direction (prefetched)
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    const int64_t Pn = P0 + n * 8 + g;
    qn[n] = Pn < npar ? nbr[Pn * 26] : -1;
  }
  for (int d = 0; d < 26; ++d) {
    int64_t qb[NT];
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      qb[n] = qn[n] >= 0 ? (int64_t)qn[n] * R + tq : -1;
      const int64_t Pn = P0 + n * 8 + g;
      qn[n] = (d + 1 < 26 && Pn < npar) ? nbr[Pn * 26 + d + 1] : -1;
    }
    {  // a direction none of the warp's parents has a (non-leaf) colleague in: no work
      bool any = false;
#pragma unroll
      for (int n = 0; n < NT; ++n) any |= qb[n] >= 0;
      if (!__any_sync(0xffffffffu, any)) continue;
    }
    const int16_t* ai_tab = aidx + d * KS * KML * 32 + lane;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      double ar[KML], ai[KML], as[KML];
#pragma unroll
      for (int m = 0; m < KML; ++m) {
        const int idx = ai_tab[(ks * KML + m) * 32];
        const double2 t = idx >= 0 ? sT[idx] : make_double2(0.0, 0.0);
        ar[m] = t.x;
        ai[m] = t.y;
        as[m] = t.x + t.y;
      }
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const double2 u = qb[n] >= 0 ? ubf[qb[n] + ks * 4] : make_double2(0.0, 0.0);
        const double us = u.x + u.y;
#pragma unroll
        for (int m = 0; m < KML; ++m) {
          dmma(acc[m][n][0][0], acc[m][n][0][1], ar[m], u.x);
          dmma(acc[m][n][1][0], acc[m][n][1][1], ai[m], u.y);
          dmma(acc[m][n][2][0], acc[m][n][2][1], as[m], us);
        }
      }
    }
  }
  double2* cbf = cb + fpos[f];  // cb is target-major [parent][8 kml][NFP], group-slot order
#pragma unroll
  for (int m = 0; m < KML; ++m)
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t Pn = P0 + n * 8 + 2 * tq + e;
        if (Pn < npar) {
          const double p1 = acc[m][n][0][e], p2 = acc[m][n][1][e];
          cbf[(Pn * R + m * 8 + g) * NFP] = make_double2(p1 - p2, acc[m][n][2][e] - p1 - p2);
        }
      }
}

// The same product for chunks whose parent blocks are mostly empty (sparse
// adaptive trees: points on surfaces), without the empty child slots.
// A warp owns one target parent P for all 26 directions and 32 frequency bins
// (lane = bin), so every branch on the occupancy of P's and its colleagues'
// children is warp-uniform: absent (b, c) child pairs cost nothing.  For each
// colleague Q_d and existing source child c the lane loads U_{Q_d, c}(f) once
// (3 components, one 512-B run per warp) and applies it to every existing,
// non-adjacent target child b:  C_b += T_{2d + c - b}(f) U_c  (9 complex
// multiply-adds into registers, acc[8][kml]).
// Operator spectra: a CTA holds 32 bins in shared memory, so the 316 offsets do
// not fit (316 x 6 x 32 x 16 B = 970 KB).  The cube reflections shrink the
// table: with S = diag(sx, sy, sz) the signs of o,
//     T_o(f) = S [conj if sz < 0] T_|o|(R f) S,
// R reflecting fx iff sx != sz and fy iff sy != sz (G(Rr) = S G(r) S; a
// reflection of the lattice differences reflects the bin; T(-f) = conj T(f)
// for the z axis of the half spectrum), so 56 offsets |o| suffice if a CTA's
// bins are closed under (fx, fy) -> (+-fx, +-fy): the bins are grouped into
// such orbits (build_fft_m2l), 32 per group, orbits never straddling an
// 8-lane phase, so the reflected reads of a warp stay bank-conflict free.
// Table: 56 x 6 x 32 x 16 B = 172 KB (Stokes family), 28 KB (Laplace).
// c_pinfo[d][b][c]: base offset index (6 bits), reflection r (2 bits), conj
// (1 bit) and the sign flips of the xy, xz, yz components (3 bits), or 0xFFFF
// for an adjacent pair (not in the V list).
constexpr int N_BASE = 56;
constexpr int SP_WARPS = 12;  // 384 threads, one CTA per SM (172 KB table), <= 170 registers
__constant__ uint16_t c_pinfo[26 * 64];
// c_grow[row], row = (dd * 2 + h) * 2 + cx: what k_m2l_groups needs per group, loaded once
// in the group header (the offset 2d + c - b of a group's pairs depends only on the row
// and delta = (cy - ty, cz - tz), index DL = 3 (DY + 1) + DZ + 1).  12 words:
//   0-4  nine 16-bit fields f(DL) = base offset index << 5 | 8 x reflection r;
//   5    SX (sign-bit mask: o_x < 0);  6, 7  SY for DY >= 0 / DY < 0;  8, 9  SZ likewise;
//   10, 11  SX ^ SZ likewise.
// The sign flips of an offset are 3-input XORs of these: conj = SZ, xy = SX ^ SY,
// xy ^ conj = (SX ^ SZ) ^ SY, xz = SX ^ SZ, xz ^ conj = SX, yz = SY ^ SZ, yz ^ conj = SY.
__constant__ uint4 c_grow[26 * 2 * 2 * 3];

__device__ __forceinline__ double xsign(double v, unsigned m) {  // flip the sign bit if m = 0x80000000
  return __hiloint2double(__double2hiint(v) ^ (int)m, __double2loint(v));
}

// The sparse-chunk product over a precomputed item stream (the default for sparse
// chunks).  Same arithmetic and table as round 2's first sparse kernel; what changes is how a warp
// finds its work.  Per chunk, setup lists for every target parent P its items
// (d, c): a non-leaf colleague Q_d and an existing child c of it such that some
// existing child b of P is a V-list target of c, with
//     vmask = { b : b exists, 2d + c - b non-adjacent }   (8 bits),
// stored as int2 {q, d | c << 5 | vmask << 8}, parents in chunk order (ioff: CSR).
// A warp owns a contiguous run of parents and walks their items as one stream:
// items and parent boundaries arrive 32 at a time (one coalesced load per lane,
// broadcast by shuffles, the next batch in flight), and the source spectra of the
// next item are loaded while the current one is applied, so no global load sits
// between two items' multiply-adds (that kernel walked the 26 directions with a
// dependent nbr -> qpat -> ub load chain per direction: 2/3 of them empty on the
// C5 sphere cloud, and long-scoreboard stalls were 1/3 of its samples,
// profiles/r02_C5_product_ncu.txt).
// 16-B shared-memory load through a 32-bit shared address (the generic-pointer form
// re-derived the CTA's shared window -- S2UR SR_CgaCtaId, an XU-pipe op -- in front of
// every b block; the XU pipe then ran at 3.5x its sustained rate in ncu)
__device__ __forceinline__ double2 lds_f64x2(unsigned a) {
  double2 v;
  asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}

// Signs per item.  For an item (d, c) every target child b sees o = 2d + c - b with the
// same sign choice S = diag(sx, sy, sz): along an axis with d_k != 0 the sign of o_k is
// that of d_k for every b; along an axis with d_k = 0, o_k = c_k - b_k is in {0, 1} when
// c_k = 1 (take +) and in {-1, 0} when c_k = 0 (take -), and o_k = 0 admits either sign
// (the kernel grid of such an offset is symmetric under that axis's reflection).  So the
// reflection slot and the sign masks of S [conj] T S are uniform over the item: setup
// stores S in bits 16-18 of the item word, the masks are formed once per item, and a
// block costs the base-offset lookup, six table loads and the sign flips.  (One code
// variant per sign pattern, with the flips folded into the multiply-adds, overflowed
// the instruction cache: 2.4x slower, profiles/r02_C5_product_ncu.txt.)
struct ItemSigns {
  unsigned tslot;                            // shared address of the item's reflected bin slot
  unsigned mc, mxy, mxyc, mxz, mxzc, myz, myzc;  // sign-bit masks (bit 31)
};

template <int KML>
__device__ __forceinline__ void sparse_block(double2 (&o)[KML], const double2 (&U)[KML], unsigned t,
                                             const ItemSigns& sg) {
  if (KML == 1) {
    const double2 t0 = lds_f64x2(t);
    cmac(o[0], make_double2(t0.x, xsign(t0.y, sg.mc)), U[0]);
  } else {
    double2 T[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) T[k] = lds_f64x2(t + k * 32 * 16);
    T[0].y = xsign(T[0].y, sg.mc);
    T[3].y = xsign(T[3].y, sg.mc);
    T[5].y = xsign(T[5].y, sg.mc);
    T[1] = make_double2(xsign(T[1].x, sg.mxy), xsign(T[1].y, sg.mxyc));
    T[2] = make_double2(xsign(T[2].x, sg.mxz), xsign(T[2].y, sg.mxzc));
    T[4] = make_double2(xsign(T[4].x, sg.myz), xsign(T[4].y, sg.myzc));
    cmac(o[0], T[0], U[0]);
    cmac(o[0], T[1], U[KML > 1 ? 1 : 0]);
    cmac(o[0], T[2], U[KML > 2 ? 2 : 0]);
    cmac(o[KML > 1 ? 1 : 0], T[1], U[0]);
    cmac(o[KML > 1 ? 1 : 0], T[3], U[KML > 1 ? 1 : 0]);
    cmac(o[KML > 1 ? 1 : 0], T[4], U[KML > 2 ? 2 : 0]);
    cmac(o[KML > 2 ? 2 : 0], T[2], U[0]);
    cmac(o[KML > 2 ? 2 : 0], T[4], U[KML > 1 ? 1 : 0]);
    cmac(o[KML > 2 ? 2 : 0], T[5], U[KML > 2 ? 2 : 0]);
  }
}

#ifndef KF_BPAIR
#define KF_BPAIR 1
#endif
// all blocks of one item: target children in pairs (b, b + 1), two independent blocks
// (12 multiply-add chains) in flight when both are valid.  Item word y (setup,
// build_fft_chunks): bits 0-10 d * 64 + c (the c_pinfo row), 11-18 vmask, 19-20 the
// reflection r, 29-31 the signs sx, sy, sz; slots4 packs the lane's 4 reflected slots.
template <int KML, int NB>
__device__ __forceinline__ void sparse_apply(double2 (&acc)[NB][KML], const double2 (&U)[KML], unsigned y,
                                             unsigned sT32, unsigned slots4, int boff) {
  constexpr unsigned OB = (KML == 1 ? 1 : 6) * 32 * 16;  // bytes per base offset in the table
  const unsigned vm = (y >> 11) & 255u;
  const uint16_t* inf = c_pinfo + (y & 2047u) + boff * 8;
  ItemSigns sg;
  sg.tslot = sT32 + __byte_perm(slots4, 0u, ((y >> 19) & 3u) | 0x4440u) * 16u;
  const unsigned y1 = y << 1, y2 = y << 2;  // sy, sx at bit 31
  sg.mc = y & 0x80000000u;
  sg.mxy = (y1 ^ y2) & 0x80000000u;
  sg.mxz = (y ^ y2) & 0x80000000u;
  sg.myz = (y ^ y1) & 0x80000000u;
  sg.mxyc = sg.mxy ^ sg.mc;
  sg.mxzc = sg.mxz ^ sg.mc;
  sg.myzc = sg.myz ^ sg.mc;
#if KF_BPAIR == 0
#pragma unroll
  for (int b = 0; b < NB; ++b)
    if ((vm >> b) & 1u) sparse_block<KML>(acc[b], U, sg.tslot + (inf[b * 8] & 63u) * OB, sg);
  return;
#endif
#pragma unroll
  for (int b = 0; b < NB; b += 2) {
    const unsigned two = (vm >> b) & 3u;
    if (two == 3u) {
      const unsigned t0 = sg.tslot + (inf[b * 8] & 63u) * OB, t1 = sg.tslot + (inf[(b + 1) * 8] & 63u) * OB;
      sparse_block<KML>(acc[b], U, t0, sg);
      sparse_block<KML>(acc[b + 1], U, t1, sg);
    } else if (two == 1u) {
      sparse_block<KML>(acc[b], U, sg.tslot + (inf[b * 8] & 63u) * OB, sg);
    } else if (two == 2u) {
      sparse_block<KML>(acc[b + 1], U, sg.tslot + (inf[(b + 1) * 8] & 63u) * OB, sg);
    }
  }
}

#ifndef KF_ITEM_PF
#define KF_ITEM_PF 6
#endif
constexpr int ITEM_PF = KF_ITEM_PF;  // items ahead whose source spectra are prefetched into L2

// NB = 8: a warp's unit is a target parent (all 8 children in registers, 12 warps);
// NB = 4: a half parent (children 4h .. 4h + 3, h = the x bit of the octant; ord carries
// 2P + h), half the accumulators, 16 warps per SM -- the source spectra of an item are
// loaded once per half
#ifndef KF_ITEM_WARPS4
#define KF_ITEM_WARPS4 16
#endif
template <int NB>
struct ItemCfg {
  static constexpr int WARPS = NB == 8 ? SP_WARPS : KF_ITEM_WARPS4;
};

template <int KML, int NB>
__global__ void __launch_bounds__(ItemCfg<NB>::WARPS * 32, 1)
    k_m2l_items(int64_t npar, int64_t nq, int NFP, int nrange, const double2* __restrict__ tbase,
                const int* __restrict__ rslot, const double2* __restrict__ ub, double2* __restrict__ cb,
                const int32_t* __restrict__ ioff, const int2* __restrict__ items, const uint8_t* __restrict__ tpat,
                const int32_t* __restrict__ wrange, const int32_t* __restrict__ ord) {
  constexpr int NC = KML == 1 ? 1 : 6, R = 8 * KML;
  extern __shared__ __align__(16) double2 sTb[];  // [N_BASE][NC][32]
  const int g = blockIdx.y;
  {
    const double4* src = reinterpret_cast<const double4*>(tbase + (int64_t)g * N_BASE * NC * 32);
    double4* dst = reinterpret_cast<double4*>(sTb);
    for (int i = threadIdx.x; i < N_BASE * NC * 16; i += ItemCfg<NB>::WARPS * 32) dst[i] = src[i];
  }
  __syncthreads();
  unsigned sT32;  // produced after the barrier (volatile), so no table read moves above it
  asm volatile("mov.u32 %0, %1;" : "=r"(sT32) : "r"((unsigned)__cvta_generic_to_shared(sTb)));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned slots4;  // the lane's bin slot under the 4 reflections, one byte each
  {
    const int rs = rslot[g * 32 + lane];
    slots4 = (rs & 31) | (((rs >> 5) & 31) << 8) | (((rs >> 10) & 31) << 16) | (((rs >> 15) & 31) << 24);
  }
  const double2* ubg = ub + (int64_t)g * nq * R * 32 + lane;
  // the warp's parents: positions [wrange[r], wrange[r + 1]) of the processing order ord
  // (setup deals the chunk's parents round-robin to the nrange warps of a frequency group,
  // so at any time the running warps share a window of Morton-adjacent parents and the
  // source spectra they read stay in L2)
  const int r = blockIdx.x * ItemCfg<NB>::WARPS + warp;
  if (r >= nrange) return;
  const int pa = wrange[r], pe = wrange[r + 1];
  // parent boundaries, ids and patterns, 32 positions per batch: lane l holds
  // ioff[pb + l + 1], ord[pb + l] and its pattern
  int pb = pa;
  int pend = ioff[min(pb + lane + 1, pe)];
  // unit id (parent, or 2 parent + half) and its child pattern (NB bits)
  auto unit_pat = [&](int id) {
    return NB == 8 ? (unsigned)tpat[id] : ((unsigned)tpat[id >> 1] >> (4 * (id & 1))) & 15u;
  };
  int pid = pb + lane < pe ? ord[pb + lane] : 0;
  unsigned ppat = pb + lane < pe ? unit_pat(pid) : 0u;
  const int ibeg = ioff[pa], iend = ioff[pe];
  // item batches: lane l holds items[ib + l] (bat) and items[ib + 32 + l] (batn); an item
  // is {x = offset of its source spectra block (KML rows of 32 bins) from the group base,
  // y = item word (sparse_apply)}
  int ib = ibeg;
  int2 bat = ib + lane < iend ? items[ib + lane] : make_int2(0, 0);
  int2 batn = ib + 32 + lane < iend ? items[ib + 32 + lane] : make_int2(0, 0);
  double2 acc[NB][KML];
#pragma unroll
  for (int b = 0; b < NB; ++b)
#pragma unroll
    for (int a = 0; a < KML; ++a) acc[b][a] = make_double2(0.0, 0.0);
  int P = pa;
  int boff = 0;  // first child of the current unit
  int pcur_end = __shfl_sync(0xffffffffu, pend, 0);
  // store the finished parent P (every existing child, zero if it had no items), next parent
  auto flush = [&]() {
    const unsigned bm = __shfl_sync(0xffffffffu, ppat, P - pb);
    const int id = __shfl_sync(0xffffffffu, pid, P - pb);
    double2* o = cb + ((int64_t)(NB == 8 ? id : id >> 1) * R + boff * KML) * NFP + g * 32 + lane;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      if ((bm >> b) & 1u) {
#pragma unroll
        for (int a = 0; a < KML; ++a) o[(int64_t)(b * KML + a) * NFP] = acc[b][a];
      }
#pragma unroll
      for (int a = 0; a < KML; ++a) acc[b][a] = make_double2(0.0, 0.0);
    }
    ++P;
    if (P < pe && P - pb == 32) {
      pb = P;
      pend = ioff[min(pb + lane + 1, pe)];
      pid = pb + lane < pe ? ord[pb + lane] : 0;
      ppat = pb + lane < pe ? unit_pat(pid) : 0u;
    }
    if (P < pe) {
      pcur_end = __shfl_sync(0xffffffffu, pend, P - pb);
      if (NB == 4) boff = 4 * (__shfl_sync(0xffffffffu, pid, P - pb) & 1);
    }
  };
  if (NB == 4) boff = 4 * (__shfl_sync(0xffffffffu, pid, 0) & 1);
  // item j's field (x or y), j in [ib, ib + 64), warp-uniform
  auto field = [&](int j, bool wantx) {
    const int k = j - ib;
    const int2 src = k < 32 ? bat : batn;
    return __shfl_sync(0xffffffffu, wantx ? src.x : src.y, k & 31);
  };
  auto load_u = [&](int off, double2(&Ud)[KML]) {
#pragma unroll
    for (int e = 0; e < KML; ++e) Ud[e] = ubg[off + e * 32];
  };
  // one item: refill the batch window, pull the spectra ITEM_PF items ahead into L2, load
  // the next item's spectra into Un (in flight during this item's products), apply
  auto step = [&](int i, double2(&Uc)[KML], double2(&Un)[KML], unsigned& yc) {
    while (i == pcur_end) flush();  // parents ending here (also those without items)
    const int j = i + 1;
    if (j - ib == 32) {
      ib = j;
      bat = batn;
      batn = ib + 32 + lane < iend ? items[ib + 32 + lane] : make_int2(0, 0);
    }
    if (i + ITEM_PF < iend) {
      const int off = field(i + ITEM_PF, true);
      if (lane < KML * 4) asm volatile("prefetch.global.L2 [%0];" ::"l"(ubg - lane + off + lane * 8));
    }
    unsigned yn = 0;
    if (j < iend) {
      load_u(field(j, true), Un);
      yn = (unsigned)field(j, false);
    }
    sparse_apply<KML, NB>(acc, Uc, yc, sT32, slots4, boff);
    yc = yn;
  };
  double2 U0[KML], U1[KML];
  unsigned y = 0;
  if (ibeg < iend) {
    for (int j = ibeg + 1; j <= ibeg + ITEM_PF && j < iend; ++j) {
      const int off = field(j, true);
      if (lane < KML * 4) asm volatile("prefetch.global.L2 [%0];" ::"l"(ubg - lane + off + lane * 8));
    }
    load_u(field(ibeg, true), U0);
    y = (unsigned)field(ibeg, false);
  }
  for (int i = ibeg; i < iend; i += 2) {  // two items per trip: the spectra registers alternate
    step(i, U0, U1, y);
    if (i + 1 < iend) step(i + 1, U1, U0, y);
  }
  while (P < pe) flush();
}

// ---------------------------------------------------------------------------
// Sparse-chunk product with operator reuse (k_m2l_groups, the default for sparse chunks).
// k_m2l_items loads one operator T_o(f) (6 x 16 B per lane) per V pair: six LDS.128 for
// 36 DFMA, i.e. 24 shared-memory wavefronts per 18 FP64-pipe cycles -- the table, not the
// FP64 pipe, bounds it.  But the offset o = 2d + c - b of a child pair depends only on
// c - b within one colleague: in a half-parent unit (target children b = 4h + t, t =
// (ty, tz)) and one x half cx of colleague Q_d (source children c = 4cx + c', c' = (cy, cz)),
// the 16 pairs (t, c') share 9 offsets, indexed by delta = (cy - ty, cz - tz).  A group =
// (unit, d, cx) with its 16-bit pair mask: the lane holds the 4 source spectra and the
// 4 accumulators, and each offset's T is loaded once for all the valid pairs that use
// it (full 4 x 4 blocks: 9 loads per 16 pairs).  Group word y: bits 0-6 the c_grow row
// (dd * 2 + h) * 2 + cx, bits 7-22 the pair mask (bit 4t + c'), bits 23-26 the source mask.
//
// Everything that steers a group is warp-uniform, and the kernel tells the compiler so:
// the group word goes through a ballot (lane l contributes bit l; a ballot is uniform by
// construction), so the pair tests compile to plain branches without BSSY / BSYNC
// reconvergence pairs, and each offset's table address, reflection selector and sign
// masks (S [conj] T_|o|(R f) S) derive from the group's c_grow row, loaded once per group
// (ncu, C5 level 9, before: 42.6% of the warp instructions were DFMA, 15.4% branch
// bookkeeping, 18% LOP3).

// pairs (t, c') of one offset delta = (cy - ty, cz - tz), DY, DZ in {-1, 0, 1}
template <int DY, int DZ>
struct GDelta {
  static constexpr int cp(int t) { return 2 * (((t >> 1) & 1) + DY) + ((t & 1) + DZ); }
  static constexpr bool ok(int t) {
    return ((t >> 1) & 1) + DY >= 0 && ((t >> 1) & 1) + DY <= 1 && (t & 1) + DZ >= 0 && (t & 1) + DZ <= 1;
  }
  static constexpr unsigned mask() {
    return (ok(0) ? 1u << cp(0) : 0u) | (ok(1) ? 1u << (4 + cp(1)) : 0u) | (ok(2) ? 1u << (8 + cp(2)) : 0u) |
           (ok(3) ? 1u << (12 + cp(3)) : 0u);
  }
};

__device__ __forceinline__ double xsign2(double v, unsigned m1, unsigned m2) {  // one LOP3
  return __hiloint2double(__double2hiint(v) ^ (int)m1 ^ (int)m2, __double2loint(v));
}

// the group's row of c_grow in registers
struct GRow {
  unsigned w[5], sx, sy[2], sz[2], sxz[2];
};

// one offset of a group: load T once (Stokes family: in two halves, T0..T2 then T3..T5,
// 12 registers live instead of 24), apply it to every valid pair of the delta.  The
// table address comes from the row's field by a few fixed-latency integer operations (a
// constant load per offset put ~70 cycles ahead of every T load: ncu, C5 level 9).
template <int KML, int DY, int DZ>
__device__ __forceinline__ void group_delta(double2 (&acc)[4][KML], const double2 (&U)[4][KML], unsigned pm,
                                            const GRow& g, unsigned sT32, unsigned slots4) {
  using D = GDelta<DY, DZ>;
  if (!(pm & D::mask())) return;
  constexpr int DL = 3 * (DY + 1) + DZ + 1;
  constexpr unsigned OB32 = (KML == 1 ? 1 : 6) * 16;  // operator bytes / 32
  const unsigned f = (DL & 1) ? g.w[DL / 2] >> 16 : g.w[DL / 2];  // bits 16.. of an even field: masked below
  const unsigned slot = (slots4 >> (f & 31u)) & 0xFFu;
  const unsigned ta = (f & 0xFFE0u) * OB32 + sT32 + slot * 16u;
  const unsigned SY = g.sy[DY < 0], SZ = g.sz[DZ < 0], SXZ = g.sxz[DZ < 0];
  if (KML == 1) {
    double2 T0 = lds_f64x2(ta);
    T0.y = xsign(T0.y, SZ);
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (D::ok(t) && ((pm >> (4 * t + D::cp(t))) & 1u)) cmac(acc[t][0], T0, U[D::ok(t) ? D::cp(t) : 0][0]);
    return;
  }
  {
    double2 T0 = lds_f64x2(ta), T1 = lds_f64x2(ta + 512), T2 = lds_f64x2(ta + 1024);
    T0.y = xsign(T0.y, SZ);
    T1 = make_double2(xsign2(T1.x, g.sx, SY), xsign2(T1.y, SXZ, SY));
    T2 = make_double2(xsign(T2.x, SXZ), xsign(T2.y, g.sx));
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (D::ok(t) && ((pm >> (4 * t + D::cp(t))) & 1u)) {
        const int c = D::ok(t) ? D::cp(t) : 0;
        cmac(acc[t][0], T0, U[c][0]);
        cmac(acc[t][0], T1, U[c][KML > 1 ? 1 : 0]);
        cmac(acc[t][0], T2, U[c][KML > 2 ? 2 : 0]);
        cmac(acc[t][KML > 1 ? 1 : 0], T1, U[c][0]);
        cmac(acc[t][KML > 2 ? 2 : 0], T2, U[c][0]);
      }
  }
  {
    double2 T3 = lds_f64x2(ta + 1536), T4 = lds_f64x2(ta + 2048), T5 = lds_f64x2(ta + 2560);
    T3.y = xsign(T3.y, SZ);
    T5.y = xsign(T5.y, SZ);
    T4 = make_double2(xsign2(T4.x, SY, SZ), xsign(T4.y, SY));
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (D::ok(t) && ((pm >> (4 * t + D::cp(t))) & 1u)) {
        const int c = D::ok(t) ? D::cp(t) : 0;
        cmac(acc[t][KML > 1 ? 1 : 0], T3, U[c][KML > 1 ? 1 : 0]);
        cmac(acc[t][KML > 1 ? 1 : 0], T4, U[c][KML > 2 ? 2 : 0]);
        cmac(acc[t][KML > 2 ? 2 : 0], T4, U[c][KML > 1 ? 1 : 0]);
        cmac(acc[t][KML > 2 ? 2 : 0], T5, U[c][KML > 2 ? 2 : 0]);
      }
  }
}

// 12 warps (<= 170 registers: 4 sources + 4 accumulators + the operator, no spills); 16
// warps at 128 registers spill and measured slower (C5 product 557 vs 500 ms)
#ifndef KF_GROUP_WARPS
#define KF_GROUP_WARPS 12
#endif
#ifndef KF_GROUP_CHUNK
#define KF_GROUP_CHUNK 4
#endif

constexpr int GROUP_WARPS = KF_GROUP_WARPS;
constexpr int GROUP_CHUNK = KF_GROUP_CHUNK;  // unit positions per dynamically taken range

template <int KML>
__global__ void __launch_bounds__(GROUP_WARPS * 32, 1)
    k_m2l_groups(int64_t nq, int NFP, int nper, const double2* __restrict__ tbase, const int* __restrict__ rslot,
                 const double2* __restrict__ ub, double2* __restrict__ cb, const int32_t* __restrict__ ioff,
                 const int2* __restrict__ items, const uint8_t* __restrict__ tpat, const int32_t* __restrict__ wrange,
                 const int32_t* __restrict__ ord) {
  constexpr int NC = KML == 1 ? 1 : 6, R = 8 * KML;
  extern __shared__ __align__(16) double2 sTb[];  // [N_BASE][NC][32]
  __shared__ int s_next;  // the CTA's next untaken range
  const int g = blockIdx.y;
  {
    const double4* src = reinterpret_cast<const double4*>(tbase + (int64_t)g * N_BASE * NC * 32);
    double4* dst = reinterpret_cast<double4*>(sTb);
    for (int i = threadIdx.x; i < N_BASE * NC * 16; i += GROUP_WARPS * 32) dst[i] = src[i];
  }
  if (threadIdx.x == 0) s_next = GROUP_WARPS;  // ranges 0 .. GROUP_WARPS - 1 go to the warps directly
  __syncthreads();
  unsigned sT32;
  asm volatile("mov.u32 %0, %1;" : "=r"(sT32) : "r"((unsigned)__cvta_generic_to_shared(sTb)));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned slots4;
  {
    const int rs = rslot[g * 32 + lane];
    slots4 = (rs & 31) | (((rs >> 5) & 31) << 8) | (((rs >> 10) & 31) << 16) | (((rs >> 15) & 31) << 24);
  }
  const double2* ubg = ub + (int64_t)g * nq * R * 32;  // the frequency group's spectra rows
  for (int rc = warp; rc < nper;) {
  const int r = blockIdx.x * nper + rc;
  const int pa = wrange[r], pe = wrange[r + 1];
  int pb = pa;
  int pend = ioff[min(pb + lane + 1, pe)];
  auto unit_pat = [&](int id) { return ((unsigned)tpat[id >> 1] >> (4 * (id & 1))) & 15u; };
  int pid = pb + lane < pe ? ord[pb + lane] : 0;
  unsigned ppat = pb + lane < pe ? unit_pat(pid) : 0u;
  const int ibeg = ioff[pa], iend = ioff[pe];
  int ib = ibeg;  // lane l holds groups ib + l (bat) and ib + 32 + l (batn)
  int2 bat = ib + lane < iend ? items[ib + lane] : make_int2(0, 0);
  int2 batn = ib + 32 + lane < iend ? items[ib + 32 + lane] : make_int2(0, 0);
  double2 acc[4][KML];
#pragma unroll
  for (int b = 0; b < 4; ++b)
#pragma unroll
    for (int a = 0; a < KML; ++a) acc[b][a] = make_double2(0.0, 0.0);
  int P = pa;
  int h = 0;  // x bit of the current unit's target children
  int pcur_end = __shfl_sync(0xffffffffu, pend, 0);
  auto flush = [&]() {
    const unsigned bm = __shfl_sync(0xffffffffu, ppat, P - pb);
    const int id = __shfl_sync(0xffffffffu, pid, P - pb);
    double2* o = cb + ((int64_t)(id >> 1) * R + 4 * h * KML) * NFP + g * 32 + lane;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      if ((bm >> b) & 1u) {
#pragma unroll
        for (int a = 0; a < KML; ++a) o[(int64_t)(b * KML + a) * NFP] = acc[b][a];
      }
#pragma unroll
      for (int a = 0; a < KML; ++a) acc[b][a] = make_double2(0.0, 0.0);
    }
    ++P;
    if (P < pe && P - pb == 32) {
      pb = P;
      pend = ioff[min(pb + lane + 1, pe)];
      pid = pb + lane < pe ? ord[pb + lane] : 0;
      ppat = pb + lane < pe ? unit_pat(pid) : 0u;
    }
    if (P < pe) {
      pcur_end = __shfl_sync(0xffffffffu, pend, P - pb);
      h = __shfl_sync(0xffffffffu, pid, P - pb) & 1;
    }
  };
  h = __shfl_sync(0xffffffffu, pid, 0) & 1;
  // L2 prefetch of the groups' spectra rows (4 children x KML rows of 512 B = 4 x KML x 4
  // lines each, the present children only), lane-parallel: lane l pulls the lines of the
  // group it holds -- the first batch up front, then the next batch (batn, groups ib + 32
  // ..) once the current one is 8 groups in, i.e. 24 to 55 groups ahead of their use.
  // 48 predicated prefetches per 32 groups instead of two broadcasts, address arithmetic
  // and two prefetches per group (measured equal: C5 product 426 vs 427 ms).
  constexpr int LPC = KML * 4;  // 128-B lines per child
  auto prefetch_own = [&](int2 it) {
    const double2* pl = ubg + it.x;
    const unsigned sm = ((unsigned)it.y >> 23) & 15u;
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if ((sm >> c) & 1u) {
#pragma unroll
        for (int l = 0; l < LPC; ++l) asm volatile("prefetch.global.L2 [%0];" ::"l"(pl + (c * LPC + l) * 8));
      }
  };
  prefetch_own(bat);
  for (int i = ibeg; i < iend; ++i) {
    while (i == pcur_end) flush();
    if (i - ib == 32) {
      ib = i;
      bat = batn;
      batn = ib + 32 + lane < iend ? items[ib + 32 + lane] : make_int2(0, 0);
    }
    const int k = i - ib;
    const int off = __shfl_sync(0xffffffffu, bat.x, k);
    const unsigned y = (unsigned)__shfl_sync(0xffffffffu, bat.y, k);
    // past the end batn holds zeros: an empty source mask, nothing prefetched
    if (k == 8) prefetch_own(batn);
    double2 U[4][KML];
    const double2* pu = ubg + (off + lane);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if ((y >> (23 + c)) & 1u) {  // absent children: no pair bit reads U[c]
#pragma unroll
        for (int e = 0; e < KML; ++e) U[c][e] = pu[(c * KML + e) * 32];
      }
    }
    const unsigned yu = __ballot_sync(0xffffffffu, (y >> lane) & 1u);  // = y, known uniform
    const unsigned pm = (yu >> 7) & 0xFFFFu;
    GRow gi;
    {
      const uint4* gr = c_grow + (yu & 127u) * 3;
      const uint4 q0 = gr[0], q1 = gr[1], q2 = gr[2];
      gi.w[0] = q0.x, gi.w[1] = q0.y, gi.w[2] = q0.z, gi.w[3] = q0.w, gi.w[4] = q1.x;
      gi.sx = q1.y, gi.sy[0] = q1.z, gi.sy[1] = q1.w;
      gi.sz[0] = q2.x, gi.sz[1] = q2.y, gi.sxz[0] = q2.z, gi.sxz[1] = q2.w;
    }
    group_delta<KML, 0, 0>(acc, U, pm, gi, sT32, slots4);
    group_delta<KML, 0, 1>(acc, U, pm, gi, sT32, slots4);
    group_delta<KML, 0, -1>(acc, U, pm, gi, sT32, slots4);
    group_delta<KML, 1, 0>(acc, U, pm, gi, sT32, slots4);
    group_delta<KML, -1, 0>(acc, U, pm, gi, sT32, slots4);
    group_delta<KML, 1, 1>(acc, U, pm, gi, sT32, slots4);
    group_delta<KML, 1, -1>(acc, U, pm, gi, sT32, slots4);
    group_delta<KML, -1, 1>(acc, U, pm, gi, sT32, slots4);
    group_delta<KML, -1, -1>(acc, U, pm, gi, sT32, slots4);
  }
  while (P < pe) flush();
  {
    int nx = 0;
    if (lane == 0) nx = atomicAdd(&s_next, 1);
    rc = __shfl_sync(0xffffffffu, nx, 0);
  }
  }
}

// base table of the sparse product: tbase[g][ob][c][s] = That_{o(ob)}(f(g, s))[c] (0 on padding slots)
__global__ void k_tbase(int nfg, int nc, const int32_t* __restrict__ gfreq, const int16_t* __restrict__ boff,
                        const double2* __restrict__ that, double2* __restrict__ tbase) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // over [nfg][56][nc][32]
  if (t >= (int64_t)nfg * N_BASE * nc * 32) return;
  const int s = (int)(t % 32);
  const int64_t r = t / 32;
  const int c = (int)(r % nc), ob = (int)((r / nc) % N_BASE), g = (int)(r / nc / N_BASE);
  const int f = gfreq[g * 32 + s];
  tbase[t] = f >= 0 ? that[((int64_t)f * N_OFFSETS + boff[ob]) * nc + c] : make_double2(0.0, 0.0);
}

// ---------------------------------------------------------------------------
// host
// ---------------------------------------------------------------------------
static bool chunk_uses_pairs(const Plan& Pl, const FftChunk& ch) {
  return Pl.m2l_mode == M2L_FFT_PAIRS || (Pl.m2l_mode == M2L_FFT && ch.block_fill < pair_fill_threshold());
}

// transforms per forward CTA: 2 (measured after the z pass started reading UE directly:
// C2 M2L transforms 3.5 -> 2.8 ms with nb 1 / 4 slower, profiles/r01_fft_rework_ab.txt;
// C4 (p = 12) 206 -> 177 ms against 1); KAFMM_FWD_NB=1|2|4 overrides (tuning knob)
static int fwd_nb(int) {
  static const char* e = getenv("KAFMM_FWD_NB");
  if (e) return atoi(e) >= 4 ? 4 : (atoi(e) >= 2 ? 2 : 1);
  return 2;
}

template <int P>
static void set_smem_attrs() {
  static std::atomic<uint64_t> done{0};
  if (!first_on_device(done)) return;
  KF_CUDA(cudaFuncSetAttribute(k_fft_fwd<P, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)FwdCfg<P>::template smem<1>()));
  if (FwdCfg<P>::template smem<2>() <= 227 * 1024)
    KF_CUDA(cudaFuncSetAttribute(k_fft_fwd<P, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)FwdCfg<P>::template smem<2>()));
  if (FwdCfg<P>::template smem<4>() <= 227 * 1024)
    KF_CUDA(cudaFuncSetAttribute(k_fft_fwd<P, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)FwdCfg<P>::template smem<4>()));
  KF_CUDA(cudaFuncSetAttribute(k_fft_inv<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)FftDims<P>::INV_SMEM));
}

template <int P, int NB>
static void launch_fwd_nb(Plan& Pl, const FftChunk& ch) {
  const int ng = (8 * Pl.kml + NB - 1) / NB;
  k_fft_fwd<P, NB><<<(unsigned)(ch.nq * ng), 256, FwdCfg<P>::template smem<NB>(), Pl.stream>>>(
      ch.d_qbox, Pl.d_crow, ch.nq, Pl.d_ue, Pl.ldn, Pl.kml, Pl.d_lmap, Pl.d_ub, chunk_uses_pairs(Pl, ch) ? 0 : 1,
      Pl.d_wz, Pl.d_wf, Pl.d_fpos);
}

template <int P>
static void launch_fwd(Plan& Pl, const FftChunk& ch) {
  set_smem_attrs<P>();
  int nb = fwd_nb(P);
  while (nb > 1 && (nb == 4 ? FwdCfg<P>::template smem<4>() : FwdCfg<P>::template smem<2>()) > 227 * 1024) nb /= 2;
  if (nb == 4) launch_fwd_nb<P, 4>(Pl, ch);
  else if (nb == 2) launch_fwd_nb<P, 2>(Pl, ch);
  else launch_fwd_nb<P, 1>(Pl, ch);
  KF_CHECK_LAUNCH();
  Pl.launches++;
}
template <int P>
static void launch_inv(Plan& Pl, const FftChunk& ch) {
  set_smem_attrs<P>();
  k_fft_inv<P><<<(unsigned)ch.nt, 256, FftDims<P>::INV_SMEM, Pl.stream>>>(
      ch.d_tbox, ch.d_tpb, ch.npar, ch.level, Pl.d_cb, Pl.kml, Pl.d_lat, Pl.M, Pl.d_chk, Pl.ldn, Pl.d_wi,
      Pl.d_fpos, Pl.NFP);
  KF_CHECK_LAUNCH();
  Pl.launches++;
}

#define KF_FFT_DISPATCH(FN)                                    \
  switch (Pl.p) {                                              \
    case 3: FN<3>(Pl, ch); break;                              \
    case 4: FN<4>(Pl, ch); break;                              \
    case 5: FN<5>(Pl, ch); break;                              \
    case 6: FN<6>(Pl, ch); break;                              \
    case 7: FN<7>(Pl, ch); break;                              \
    case 8: FN<8>(Pl, ch); break;                              \
    case 10: FN<10>(Pl, ch); break;                            \
    case 12: FN<12>(Pl, ch); break;                            \
    default: throw Error{KAFMM_EINVAL, "FFT M2L: unsupported p"}; \
  }

bool fft_supported_p(int p) { return (p >= 3 && p <= 8) || p == 10 || p == 12; }

#ifndef KF_NT_L
#define KF_NT_L 4
#define KF_NT_G 2
#endif
constexpr int NT_L = KF_NT_L, NT_G = KF_NT_G;  // parent n-tiles per warp (Laplace, Stokes family); measured best (profiles/)

// target children per warp unit of the sparse product: 4 (half parent, 16 warps per SM;
// C5 product 544 ms against 614 ms for whole parents with paired blocks, profiles/r02_C5_product_ab.txt);
// KAFMM_ITEM_NB=4|8 overrides (tuning knob, read at plan setup and launch)
int item_nb() {
  static const int v = getenv("KAFMM_ITEM_NB") ? (atoi(getenv("KAFMM_ITEM_NB")) == 8 ? 8 : 4) : 4;
  return v;
}

// sparse-chunk product: k_m2l_groups (operator reuse across the pairs of one offset;
// default) or k_m2l_items (KAFMM_SPARSE=items, one operator load per pair).  Read at plan
// setup (the stream layout differs) and stored in the chunk.
bool sparse_groups() {
  const char* e = getenv("KAFMM_SPARSE");
  return !(e && std::string(e) == "items");
}
// unit positions per dynamically taken range of k_m2l_groups (host-side layout only);
// KAFMM_GROUP_CHUNK overrides (tests force 1 to get many ranges on small clouds)
static int64_t group_chunk() {
  const char* e = getenv("KAFMM_GROUP_CHUNK");
  return e && atoi(e) > 0 ? atoi(e) : GROUP_CHUNK;
}

void run_m2l_fft(Plan& Pl) {
  for (const FftChunk& ch : Pl.fft_chunks) {
    if (ch.nt == 0 || ch.nq == 0) continue;
    KF_FFT_DISPATCH(launch_fwd);
    const bool pairs = chunk_uses_pairs(Pl, ch);
    prod_mark(Pl);
    if (pairs) {
      // k_m2l_items: grid (CTAs per frequency group, groups); one CTA per SM (the 172 KB
      // operator table of its 32 bins), each warp a run of units of the item stream
      const int NC = Pl.kml == 1 ? 1 : 6;
      const size_t smem = (size_t)N_BASE * NC * 32 * sizeof(double2);
      {
        static std::atomic<uint64_t> attr2{0};
        if (first_on_device(attr2)) {
          for (auto fn : {k_m2l_items<1, 8>, k_m2l_items<1, 4>})
            KF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(N_BASE * 32 * sizeof(double2))));
          for (auto fn : {k_m2l_items<3, 8>, k_m2l_items<3, 4>})
            KF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(N_BASE * 6 * 32 * sizeof(double2))));
        }
        if (ch.groups) {
          static std::atomic<uint64_t> attr3{0};
          if (first_on_device(attr3)) {
            KF_CUDA(cudaFuncSetAttribute(k_m2l_groups<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(N_BASE * 32 * sizeof(double2))));
            KF_CUDA(cudaFuncSetAttribute(k_m2l_groups<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(N_BASE * 6 * 32 * sizeof(double2))));
          }
          const dim3 grid((unsigned)std::max<int64_t>(1, ch.nrange / std::max<int64_t>(1, ch.nper)), (unsigned)Pl.NFG);
          if (Pl.kml == 1)
            k_m2l_groups<1><<<grid, GROUP_WARPS * 32, smem, Pl.stream>>>(
                ch.nq, Pl.NFP, (int)ch.nper, Pl.d_tbase, Pl.d_rslot, Pl.d_ub, Pl.d_cb, ch.d_ioff, ch.d_items,
                ch.d_tpat, ch.d_wrange, ch.d_ord);
          else
            k_m2l_groups<3><<<grid, GROUP_WARPS * 32, smem, Pl.stream>>>(
                ch.nq, Pl.NFP, (int)ch.nper, Pl.d_tbase, Pl.d_rslot, Pl.d_ub, Pl.d_cb, ch.d_ioff, ch.d_items,
                ch.d_tpat, ch.d_wrange, ch.d_ord);
        } else {
          const int nb = item_nb();
          const int wpc = nb == 8 ? ItemCfg<8>::WARPS : ItemCfg<4>::WARPS;
          const dim3 grid((unsigned)std::max<int64_t>(1, (ch.nrange + wpc - 1) / wpc), (unsigned)Pl.NFG);
#define KF_ITEMS(KML, NB)                                                                                      \
  k_m2l_items<KML, NB><<<grid, wpc * 32, smem, Pl.stream>>>(ch.npar, ch.nq, Pl.NFP, (int)ch.nrange, Pl.d_tbase, \
                                                           Pl.d_rslot, Pl.d_ub, Pl.d_cb, ch.d_ioff, ch.d_items,  \
                                                           ch.d_tpat, ch.d_wrange, ch.d_ord)
          if (Pl.kml == 1) {
            if (nb == 8) KF_ITEMS(1, 8);
            else KF_ITEMS(1, 4);
          } else {
            if (nb == 8) KF_ITEMS(3, 8);
            else KF_ITEMS(3, 4);
          }
#undef KF_ITEMS
        }
      }
    } else {
      // parent n-tiles per warp: NT_L / NT_G by default, KAFMM_DMMA_NT=<half> halves them
      // (fewer registers, more resident warps) -- a tuning knob measured in profiles/
      static const bool half = getenv("KAFMM_DMMA_NT") != nullptr;
      const int nt = (Pl.kml == 1 ? NT_L : NT_G) / (half ? 2 : 1);
      const int ppc = DM_WARPS * 8 * nt;
      const int npb = (int)((ch.npar + ppc - 1) / ppc);
      const unsigned grid = (unsigned)((int64_t)npb * Pl.NF);
#define KF_DMMA(KML, NT)                                                                                        \
  k_m2l_dmma<KML, NT><<<grid, DM_WARPS * 32, 0, Pl.stream>>>(ch.npar, ch.nq, npb, Pl.d_that, Pl.d_ub, Pl.d_cb, \
                                                             ch.d_nbr, Pl.d_aidx, Pl.d_fpos, Pl.NFP)
      if (Pl.kml == 1) {
        if (half) KF_DMMA(1, NT_L / 2);
        else KF_DMMA(1, NT_L);
      } else {
        if (half) KF_DMMA(3, NT_G / 2);
        else KF_DMMA(3, NT_G);
      }
#undef KF_DMMA
    }
    KF_CHECK_LAUNCH();
    prod_mark(Pl);
    Pl.launches++;
    KF_FFT_DISPATCH(launch_inv);
  }
}

template <class T>
static T* h2d_vec(Plan& P, const std::vector<T>& h) {
  T* d = dalloc<T>(P, std::max<size_t>(1, h.size()));
  if (!h.empty()) KF_CUDA(cudaMemcpyAsync(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, P.stream));
  return d;
}

template <class T>
static void d2h(Plan& P, std::vector<T>& h, const T* d, int64_t n) {
  h.resize(n);
  if (n) KF_CUDA(cudaMemcpy(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost));
}

// Frequency groups, positions and the reflected-offset tables of the sparse product
// (k_m2l_items).  Orbits of a bin under (fx, fy) -> (+-fx, +-fy) have 4, 2 or 1
// members; they are packed into 8-slot phases (never straddling one) and the phases
// into groups of 32 slots.
static void build_sparse_tables(Plan& P, const int16_t* tab) {
  cudaStream_t st = P.stream;
  const int NG = P.NG, NZ = P.NZ, NF = P.NF;
  auto fid = [&](int fx, int fy, int fz) { return (fx * NG + fy) * NZ + fz; };
  std::vector<std::vector<int>> orb[3];  // by size 4, 2, 1
  std::vector<char> seen(NF, 0);
  for (int fz = 0; fz < NZ; ++fz)
    for (int fx = 0; fx < NG; ++fx)
      for (int fy = 0; fy < NG; ++fy) {
        if (seen[fid(fx, fy, fz)]) continue;
        const int rx = (NG - fx) % NG, ry = (NG - fy) % NG;
        std::vector<int> m;
        for (int f : {fid(fx, fy, fz), fid(rx, fy, fz), fid(fx, ry, fz), fid(rx, ry, fz)})
          if (!seen[f]) {
            seen[f] = 1;
            m.push_back(f);
          }
        orb[m.size() == 4 ? 0 : m.size() == 2 ? 1 : 2].push_back(m);
      }
  std::vector<int> slots;  // frequency per slot, -1 = padding
  for (int k = 0; k < 3; ++k)
    for (const auto& m : orb[k]) {
      if ((int)(slots.size() % 8) + (int)m.size() > 8) slots.resize((slots.size() + 7) / 8 * 8, -1);
      slots.insert(slots.end(), m.begin(), m.end());
    }
  slots.resize((slots.size() + 31) / 32 * 32, -1);
  P.NFG = (int)slots.size() / 32;
  P.NFP = (int)slots.size();
  std::vector<int16_t> fpos(NF, -1);
  for (int i = 0; i < P.NFP; ++i)
    if (slots[i] >= 0) fpos[slots[i]] = (int16_t)i;
  std::vector<int> rslot(P.NFP);
  for (int i = 0; i < P.NFP; ++i) {
    int packed = 0;
    for (int r = 0; r < 4; ++r) {
      int j = i;
      if (slots[i] >= 0) {
        const int f = slots[i], fz = f % NZ, fy = (f / NZ) % NG, fx = f / (NZ * NG);
        const int gx = (r & 1) ? (NG - fx) % NG : fx, gy = (r & 2) ? (NG - fy) % NG : fy;
        j = fpos[fid(gx, gy, fz)];
        if (j / 32 != i / 32) throw Error{KAFMM_ECUDA, "sparse M2L: orbit split across groups"};
      }
      packed |= (j & 31) << (5 * r);
    }
    rslot[i] = packed;
  }
  // base offsets |o| (lexicographic over {0..3}^3, max >= 2) -> offset ids
  std::vector<int16_t> boff;
  int bidx[64];
  for (int a = 0; a < 64; ++a) {
    const int ox = a / 16, oy = (a / 4) % 4, oz = a % 4;
    bidx[a] = -1;
    if (std::max(ox, std::max(oy, oz)) >= 2) {
      bidx[a] = (int)boff.size();
      boff.push_back(tab[(ox + 3) * 49 + (oy + 3) * 7 + (oz + 3)]);
    }
  }
  if ((int)boff.size() != N_BASE) throw Error{KAFMM_ECUDA, "sparse M2L: base offset count"};
  std::vector<uint16_t> info(26 * 64, 0xFFFF);
  for (int dd = 0; dd < 26; ++dd) {
    const int d = dd < 13 ? dd : dd + 1;
    const int dx = d / 9 - 1, dy = (d / 3) % 3 - 1, dz = d % 3 - 1;
    for (int b = 0; b < 8; ++b)
      for (int c = 0; c < 8; ++c) {
        const int ox = 2 * dx + ((c >> 2) & 1) - ((b >> 2) & 1), oy = 2 * dy + ((c >> 1) & 1) - ((b >> 1) & 1),
                  oz = 2 * dz + (c & 1) - (b & 1);
        if (std::max(std::abs(ox), std::max(std::abs(oy), std::abs(oz))) < 2) continue;
        const int sx = ox < 0, sy = oy < 0, sz = oz < 0;
        const int ob = bidx[std::abs(ox) * 16 + std::abs(oy) * 4 + std::abs(oz)];
        const int r = (sx ^ sz) | ((sy ^ sz) << 1);
        info[dd * 64 + b * 8 + c] =
            (uint16_t)(ob | (r << 6) | (sz << 8) | ((sx ^ sy) << 9) | ((sx ^ sz) << 10) | ((sy ^ sz) << 11));
      }
  }
  KF_CUDA(cudaMemcpyToSymbolAsync(c_pinfo, info.data(), info.size() * 2, 0, cudaMemcpyHostToDevice, st));
  {
    std::vector<uint32_t> gr(26 * 2 * 2 * 12, 0u);
    for (int dd = 0; dd < 26; ++dd)
      for (int h = 0; h < 2; ++h)
        for (int cx = 0; cx < 2; ++cx) {
          uint32_t* e = &gr[((size_t)(dd * 2 + h) * 2 + cx) * 12];
          const int d = dd < 13 ? dd : dd + 1;
          const int dx = d / 9 - 1, dy = (d / 3) % 3 - 1, dz = d % 3 - 1;
          const uint32_t S = 0x80000000u;
          const int ox = 2 * dx + cx - h;
          const uint32_t SX = ox < 0 ? S : 0, SYn = dy < 0 ? S : 0, SYm = dy <= 0 ? S : 0, SZn = dz < 0 ? S : 0,
                         SZm = dz <= 0 ? S : 0;
          e[5] = SX, e[6] = SYn, e[7] = SYm, e[8] = SZn, e[9] = SZm, e[10] = SX ^ SZn, e[11] = SX ^ SZm;
          for (int dl = 0; dl < 9; ++dl) {
            const int DY = dl / 3 - 1, DZ = dl % 3 - 1;
            const int oy = 2 * dy + DY, oz = 2 * dz + DZ;
            if (std::max(std::abs(ox), std::max(std::abs(oy), std::abs(oz))) < 2) continue;  // adjacent: never used
            const int sx = ox < 0, sy = oy < 0, sz = oz < 0;
            const int ob = bidx[std::abs(ox) * 16 + std::abs(oy) * 4 + std::abs(oz)];
            const int r = (sx ^ sz) | ((sy ^ sz) << 1);
            e[dl / 2] |= (uint32_t)((ob << 5) | (8 * r)) << (16 * (dl % 2));
          }
        }
    KF_CUDA(cudaMemcpyToSymbolAsync(c_grow, gr.data(), gr.size() * 4, 0, cudaMemcpyHostToDevice, st));
  }
  P.d_fpos = dalloc<int16_t>(P, NF);
  P.d_rslot = dalloc<int>(P, P.NFP);
  KF_CUDA(cudaMemcpyAsync(P.d_fpos, fpos.data(), NF * 2, cudaMemcpyHostToDevice, st));
  KF_CUDA(cudaMemcpyAsync(P.d_rslot, rslot.data(), P.NFP * 4, cudaMemcpyHostToDevice, st));
  int32_t* d_gf;
  int16_t* d_boff;
  KF_CUDA(cudaMalloc(&d_gf, P.NFP * 4));
  KF_CUDA(cudaMalloc(&d_boff, N_BASE * 2));
  KF_CUDA(cudaMemcpyAsync(d_gf, slots.data(), P.NFP * 4, cudaMemcpyHostToDevice, st));
  KF_CUDA(cudaMemcpyAsync(d_boff, boff.data(), N_BASE * 2, cudaMemcpyHostToDevice, st));
  const int nc = P.ncomp;
  P.d_tbase = dalloc<double2>(P, (size_t)P.NFG * N_BASE * nc * 32);
  k_tbase<<<nblk((int64_t)P.NFG * N_BASE * nc * 32), 256, 0, st>>>(P.NFG, nc, d_gf, d_boff, P.d_that, P.d_tbase);
  KF_CHECK_LAUNCH();
  KF_CUDA(cudaStreamSynchronize(st));
  cudaFree(d_gf);
  cudaFree(d_boff);
}

void build_fft_m2l(Plan& P, int64_t budget) {
  if (!fft_supported_p(P.p)) {
    P.m2l_mode = M2L_DENSE;
    return;
  }
  cudaStream_t st = P.stream;
  const int p = P.p, kml = P.kml, R = 8 * kml;
  P.NG = 2 * p - 1;
  P.NZ = P.NG / 2 + 1;
  P.NF = P.NG * P.NG * P.NZ;
  P.ncomp = kml == 1 ? 1 : 6;
  // offset table (same enumeration as the list builder and the dense operators)
  int16_t tab[343];
  std::vector<int8_t> offs;
  int id = 0;
  for (int a = 0; a < 343; ++a) {
    int ox = a / 49 - 3, oy = (a / 7) % 7 - 3, oz = a % 7 - 3;
    if (std::max(std::abs(ox), std::max(std::abs(oy), std::abs(oz))) >= 2) {
      tab[a] = (int16_t)id++;
      offs.push_back((int8_t)ox);
      offs.push_back((int8_t)oy);
      offs.push_back((int8_t)oz);
    } else {
      tab[a] = -1;
    }
  }
  // DMMA A-fragment table: for direction d, k-step ks, m-tile m and lane, the
  // shared-memory index of T_o[sym(a, e)] (or -1 where the child pair is adjacent)
  {
    const int KS = R / 4, NC = P.ncomp;
    const int sym[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
    std::vector<int16_t> ai((size_t)26 * KS * kml * 32);
    for (int dd = 0; dd < 26; ++dd) {
      const int d = dd < 13 ? dd : dd + 1;
      const int dx = d / 9 - 1, dy = (d / 3) % 3 - 1, dz = d % 3 - 1;
      for (int ks = 0; ks < KS; ++ks)
        for (int m = 0; m < kml; ++m)
          for (int lane = 0; lane < 32; ++lane) {
            const int row = m * 8 + (lane >> 2), k = ks * 4 + (lane & 3);
            const int b = row / kml, a = row % kml, c = k / kml, e = k % kml;
            const int ox = 2 * dx + ((c >> 2) & 1) - ((b >> 2) & 1);
            const int oy = 2 * dy + ((c >> 1) & 1) - ((b >> 1) & 1);
            const int oz = 2 * dz + (c & 1) - (b & 1);
            int v = -1;
            if (std::max(std::abs(ox), std::max(std::abs(oy), std::abs(oz))) >= 2)
              v = tab[(ox + 3) * 49 + (oy + 3) * 7 + (oz + 3)] * NC + (kml == 1 ? 0 : sym[a][e]);
            if (v >= 0) v = kml == 1 ? SPOS1[v] : SPOS3[v];  // shared-memory position (kafmm_spos.h)
            ai[((size_t)(dd * KS + ks) * kml + m) * 32 + lane] = (int16_t)v;
          }
    }
    P.d_aidx = dalloc<int16_t>(P, ai.size());
    KF_CUDA(cudaMemcpyAsync(P.d_aidx, ai.data(), ai.size() * 2, cudaMemcpyHostToDevice, st));
  }
  // DFT pass twiddle fragments (see dft_pass): [ks][nt][lane] of the real GEMM
  // matrix B[(i, c_in)][(o, c_out)] = 2x2 real block of w^(s o i) (1x2 for real input)
  {
    const int NG = P.NG, NZ = P.NZ;
    auto table = [&](int nin, int nout, bool cin, double sgn, std::vector<double>& t) {
      const int kc = cin ? 2 : 1, K = kc * nin, N = 2 * nout;
      const int NKS = (K + 3) / 4, NNT = (N + 7) / 8;
      t.assign((size_t)NKS * NNT * 32, 0.0);
      for (int ks = 0; ks < NKS; ++ks)
        for (int nt = 0; nt < NNT; ++nt)
          for (int lane = 0; lane < 32; ++lane) {
            const int k = 4 * ks + (lane & 3), n = 8 * nt + (lane >> 2);
            const int i = k / kc, ci = k % kc, o = n / 2, co = n % 2;
            double v = 0.0;
            if (i < nin && o < nout) {
              const double ang = sgn * 2.0 * M_PI * (double)(((int64_t)o * i) % NG) / NG;
              const double wr = std::cos(ang), wi = std::sin(ang);
              if (!cin) v = co == 0 ? wr : wi;
              else v = (co == 0) ? (ci == 0 ? wr : -wi) : (ci == 0 ? wi : wr);
            }
            t[((size_t)ks * NNT + nt) * 32 + lane] = v;
          }
    };
    std::vector<double> tz, tf, ti;
    table(p, NZ, false, -1.0, tz);
    table(p, NG, true, -1.0, tf);
    table(NG, p, true, +1.0, ti);
    P.d_wz = dalloc<double>(P, tz.size());
    P.d_wf = dalloc<double>(P, tf.size());
    P.d_wi = dalloc<double>(P, ti.size());
    KF_CUDA(cudaMemcpyAsync(P.d_wz, tz.data(), tz.size() * 8, cudaMemcpyHostToDevice, st));
    KF_CUDA(cudaMemcpyAsync(P.d_wf, tf.data(), tf.size() * 8, cudaMemcpyHostToDevice, st));
    KF_CUDA(cudaMemcpyAsync(P.d_wi, ti.data(), ti.size() * 8, cudaMemcpyHostToDevice, st));
  }
  // integer lattice of the surface points (same order as d_surf)
  std::vector<int16_t> lat;
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j)
      for (int k = 0; k < p; ++k)
        if (std::min(i, std::min(j, k)) == 0 || std::max(i, std::max(j, k)) == p - 1) {
          lat.push_back((int16_t)i);
          lat.push_back((int16_t)j);
          lat.push_back((int16_t)k);
        }
  P.d_lat = dalloc<int16_t>(P, lat.size());
  KF_CUDA(cudaMemcpyAsync(P.d_lat, lat.data(), lat.size() * 2, cudaMemcpyHostToDevice, st));
  {  // p^3 lattice -> surface index (or -1), read by the forward z pass
    std::vector<int16_t> lmap((size_t)p * p * p, -1);
    for (size_t m = 0; m < lat.size() / 3; ++m) lmap[((size_t)lat[3 * m] * p + lat[3 * m + 1]) * p + lat[3 * m + 2]] = (int16_t)m;
    P.d_lmap = dalloc<int16_t>(P, lmap.size());
    KF_CUDA(cudaMemcpyAsync(P.d_lmap, lmap.data(), lmap.size() * 2, cudaMemcpyHostToDevice, st));
    KF_CUDA(cudaStreamSynchronize(st));
  }
  // operator spectra at level 0
  {
    const int NG = P.NG, NG3 = NG * NG * NG, nc = P.ncomp;
    int8_t* d_offs;
    double* grid;
    double2* spec;
    KF_CUDA(cudaMalloc(&d_offs, offs.size()));
    KF_CUDA(cudaMemcpy(d_offs, offs.data(), offs.size(), cudaMemcpyHostToDevice));
    KF_CUDA(cudaMalloc(&grid, (size_t)N_OFFSETS * nc * NG3 * 8));
    KF_CUDA(cudaMalloc(&spec, (size_t)N_OFFSETS * nc * P.NF * 16));
    dim3 g(nblk(NG3), N_OFFSETS);
    k_kernel_grid<<<g, 256, 0, st>>>(p, NG, kml, 1.05 / (p - 1), d_offs, grid);
    KF_CHECK_LAUNCH();
    cufftHandle h;
    int n[3] = {NG, NG, NG};
    if (cufftPlanMany(&h, 3, n, nullptr, 1, NG3, nullptr, 1, P.NF, CUFFT_D2Z, N_OFFSETS * nc) != CUFFT_SUCCESS)
      throw Error{KAFMM_ECUDA, "cufftPlanMany failed"};
    cufftSetStream(h, st);
    if (cufftExecD2Z(h, grid, reinterpret_cast<cufftDoubleComplex*>(spec)) != CUFFT_SUCCESS)
      throw Error{KAFMM_ECUDA, "cufftExecD2Z failed"};
    P.d_that = dalloc<double2>(P, (size_t)N_OFFSETS * nc * P.NF);
    k_spectra_transpose<<<nblk((int64_t)N_OFFSETS * nc * P.NF), 256, 0, st>>>(P.NF, nc, spec, P.d_that);
    KF_CHECK_LAUNCH();
    KF_CUDA(cudaStreamSynchronize(st));
    cufftDestroy(h);
    cudaFree(grid);
    cudaFree(spec);
    cudaFree(d_offs);
  }
  build_sparse_tables(P, tab);
  build_fft_chunks(P, budget);
}

// chunks: per level l >= 2, Morton-contiguous runs of target parents at level
// l-1 (only parents whose subtree is active on this rank), sized to the budget
void build_fft_chunks(Plan& P, int64_t budget) {
  if (P.NF == 0) return;
  cudaStream_t st = P.stream;
  const int R = 8 * P.kml;
  P.fft_budget = budget;
  std::vector<int32_t> child, ijk;
  std::vector<uint8_t> leaf;
  std::vector<uint64_t> key;
  d2h(P, child, P.d_child, 8 * P.nbox);
  d2h(P, ijk, P.d_ijk, 3 * P.nbox);
  d2h(P, leaf, P.d_leaf, P.nbox);
  d2h(P, key, P.d_key, P.nbox);
  auto find = [&](int l, int i, int j, int k) -> int64_t {
    int n = 1 << l;
    if (i < 0 || j < 0 || k < 0 || i >= n || j >= n || k >= n) return -1;
    uint64_t kk = 0;
    for (int bit = l - 1; bit >= 0; --bit)
      kk = (kk << 3) | ((uint64_t)((i >> bit) & 1) << 2) | ((uint64_t)((j >> bit) & 1) << 1) | ((k >> bit) & 1);
    auto b = key.begin() + P.levels[l].begin, e = key.begin() + P.levels[l].end;
    auto it = std::lower_bound(b, e, kk);
    return (it != e && *it == kk) ? (int64_t)(it - key.begin()) : -1;
  };
  // V lists by target box (from the (src, tgt) pairs sorted by level/offset)
  std::vector<int2> vp;
  d2h(P, vp, P.d_v_pairs, P.n_v);
  std::vector<int64_t> voff(P.nbox + 1, 0);
  for (const int2& q : vp) voff[q.y + 1]++;
  for (int64_t b = 0; b < P.nbox; ++b) voff[b + 1] += voff[b];
  std::vector<int32_t> vsrc(P.n_v);
  {
    std::vector<int64_t> fill(voff.begin(), voff.end() - 1);
    for (const int2& q : vp) vsrc[fill[q.y]++] = q.x;
  }
  std::vector<int32_t> parent;
  d2h(P, parent, P.d_parent, P.nbox);
  int16_t offid[343];
  {
    int id = 0;
    for (int a = 0; a < 343; ++a) {
      int ox = a / 49 - 3, oy = (a / 7) % 7 - 3, oz = a % 7 - 3;
      offid[a] = (std::max(std::abs(ox), std::max(std::abs(oy), std::abs(oz))) >= 2) ? (int16_t)id++ : (int16_t)-1;
    }
  }
  const int64_t per_block = (int64_t)R * P.NFP * 16;  // one parent block of spectra
  for (FftChunk& c : P.fft_chunks)  // re-planning (kafmm_restrict): release the old lists
    for (void* p : {(void*)c.d_qbox, (void*)c.d_nbr, (void*)c.d_tbox, (void*)c.d_tpb, (void*)c.d_toff,
                    (void*)c.d_tpat, (void*)c.d_ioff, (void*)c.d_items, (void*)c.d_wrange,
                    (void*)c.d_ord})
      dfree(P, p);
  P.fft_chunks.clear();
  P.fft_max_nq = P.fft_max_npar = 0;
  std::vector<int32_t> qlocal(P.nbox, -1);
  for (int l = 2; l <= P.depth; ++l) {
    std::vector<int64_t> parents;
    for (int64_t b = P.levels[l - 1].begin; b < P.levels[l - 1].end; ++b)
      if (!leaf[b] && (P.box_active.empty() || P.box_active[b])) parents.push_back(b);
    size_t i0 = 0;
    while (i0 < parents.size()) {
      std::vector<int32_t> qs, nb;
      size_t i1 = i0;
      while (i1 < parents.size()) {
        const int64_t Pb = parents[i1];
        int64_t cq[26];
        int add = 0;
        for (int dd = 0; dd < 26; ++dd) {
          int d = dd < 13 ? dd : dd + 1;
          int64_t q = find(l - 1, ijk[3 * Pb] + d / 9 - 1, ijk[3 * Pb + 1] + (d / 3) % 3 - 1,
                           ijk[3 * Pb + 2] + d % 3 - 1);
          if (q >= 0 && leaf[q]) q = -1;
          cq[dd] = q;
          if (q >= 0 && qlocal[q] < 0) ++add;
        }
        if (i1 > i0 && ((int64_t)qs.size() + add + (int64_t)(i1 - i0) + 1) * per_block > budget) break;
        for (int dd = 0; dd < 26; ++dd) {
          const int64_t q = cq[dd];
          if (q >= 0 && qlocal[q] < 0) {
            qlocal[q] = (int32_t)qs.size();
            qs.push_back((int32_t)q);
          }
          nb.push_back(q >= 0 ? qlocal[q] : -1);
        }
        ++i1;
      }
      FftChunk ch;
      ch.level = l;
      ch.npar = (int64_t)(i1 - i0);
      ch.nq = (int64_t)qs.size();
      std::vector<int32_t> tb;
      std::vector<int2> tpb;
      std::vector<int32_t> toff(1, 0);
      for (int64_t q = 0; q < ch.npar; ++q) {
        for (int o = 0; o < 8; ++o) {
          const int32_t c = child[8 * parents[i0 + q] + o];
          if (c >= 0 && (P.box_active.empty() || P.box_active[c])) {
            tb.push_back(c);
            tpb.push_back(make_int2((int)q, o));
          }
        }
        toff.push_back((int32_t)tb.size());
      }
      ch.nt = (int64_t)tb.size();
      // child occupancy of the chunk's target and source parents (sparse product), and a
      // check that it reproduces the V lists exactly: every V source of a target is a child
      // of one of the chunk's source parents, and the per-target count equals the existing,
      // non-adjacent children of its parent's non-leaf colleagues
      std::vector<uint8_t> tpat(ch.npar, 0), qpat(ch.nq, 0);
      for (int64_t q = 0; q < ch.npar; ++q)
        for (int o = 0; o < 8; ++o) {
          const int32_t c = child[8 * parents[i0 + q] + o];
          if (c >= 0 && (P.box_active.empty() || P.box_active[c])) tpat[q] |= (uint8_t)(1u << o);
        }
      // a source child counts if it has a UE row here (every child on one GPU; on a rank,
      // the active, shared and ghost boxes -- which include every V source of its targets)
      for (int64_t q = 0; q < ch.nq; ++q)
        for (int o = 0; o < 8; ++o) {
          const int32_t c = child[8 * (int64_t)qs[q] + o];
          if (c >= 0 && (P.h_row.empty() || P.h_row[c] >= 0)) {
            qpat[q] |= (uint8_t)(1u << o);
            ++ch.nsrc_children;
          }
        }
      for (size_t ii = 0; ii < tb.size(); ++ii) {
        const int32_t t = tb[ii];
        for (int64_t e = voff[t]; e < voff[t + 1]; ++e) {
          const int32_t sb = vsrc[e];
          const int32_t q = qlocal[parent[sb]];
          const int ox = ijk[3 * sb] - ijk[3 * t], oy = ijk[3 * sb + 1] - ijk[3 * t + 1],
                    oz = ijk[3 * sb + 2] - ijk[3 * t + 2];
          const int oid = offid[(ox + 3) * 49 + (oy + 3) * 7 + (oz + 3)];
          if (q < 0 || oid < 0) throw Error{KAFMM_ECUDA, "FFT M2L: V source outside the chunk's parent blocks"};
          ++ch.npairs;
        }
        const int64_t Pq = tpb[ii].x;
        const int b = tpb[ii].y;
        int64_t derived = 0;
        for (int dd = 0; dd < 26; ++dd) {
          const int32_t q = nb[Pq * 26 + dd];
          if (q < 0) continue;
          const int d = dd < 13 ? dd : dd + 1;
          for (int c = 0; c < 8; ++c) {
            if (!((qpat[q] >> c) & 1)) continue;
            const int ox = 2 * (d / 9 - 1) + ((c >> 2) & 1) - ((b >> 2) & 1);
            const int oy = 2 * ((d / 3) % 3 - 1) + ((c >> 1) & 1) - ((b >> 1) & 1);
            const int oz = 2 * (d % 3 - 1) + (c & 1) - (b & 1);
            derived += std::max(std::abs(ox), std::max(std::abs(oy), std::abs(oz))) >= 2;
          }
        }
        if (derived != voff[t + 1] - voff[t])
          throw Error{KAFMM_ECUDA, "FFT M2L: child occupancy does not reproduce a V list"};
      }
      if ((int64_t)qs.size() * 8 >= (1 << 22)) throw Error{KAFMM_EINVAL, "FFT M2L chunk too large"};
      {
        int64_t blocks = 0;
        for (int32_t v : nb) blocks += v >= 0;
        ch.block_fill = blocks ? (double)ch.npairs / (64.0 * (double)blocks) : 1.0;
      }
      {  // item stream of the sparse product (k_m2l_items)
        // items of every parent in chunk order
        std::vector<int32_t> cnt(ch.npar, 0);
        std::vector<int2> all;
        for (int64_t q = 0; q < ch.npar; ++q) {
          for (int dd = 0; dd < 26; ++dd) {
            const int32_t qq = nb[q * 26 + dd];
            if (qq < 0) continue;
            const int d = dd < 13 ? dd : dd + 1;
            for (int c = 0; c < 8; ++c) {
              if (!((qpat[qq] >> c) & 1)) continue;
              unsigned vm = 0;
              for (int b = 0; b < 8; ++b) {
                if (!((tpat[q] >> b) & 1)) continue;
                const int ox = 2 * (d / 9 - 1) + ((c >> 2) & 1) - ((b >> 2) & 1);
                const int oy = 2 * ((d / 3) % 3 - 1) + ((c >> 1) & 1) - ((b >> 1) & 1);
                const int oz = 2 * (d % 3 - 1) + (c & 1) - (b & 1);
                if (std::max(std::abs(ox), std::max(std::abs(oy), std::abs(oz))) >= 2) vm |= 1u << b;
              }
              if (vm) {
                // sign pattern of the item (see sparse_apply): bit k set = axis k negative
                const int dv[3] = {d / 9 - 1, (d / 3) % 3 - 1, d % 3 - 1};
                int sp = 0;
                for (int k = 0; k < 3; ++k) {
                  const int ck = (c >> (2 - k)) & 1;
                  if (dv[k] < 0 || (dv[k] == 0 && ck == 0)) sp |= 1 << k;
                }
                const int r = ((sp & 1) ^ (sp >> 2)) | ((((sp >> 1) & 1) ^ (sp >> 2)) << 1);
                const int64_t off = ((int64_t)qq * R + c * P.kml) * 32;
                if (off >= INT32_MAX) throw Error{KAFMM_EINVAL, "FFT M2L chunk too large for the item stream"};
                all.push_back(make_int2((int)off, (int)((unsigned)(dd * 64 + c) | (vm << 11) | ((unsigned)r << 19) |
                                                        ((unsigned)sp << 29))));
                ++cnt[q];
              }
            }
          }
          if (all.size() >= (size_t)INT32_MAX) throw Error{KAFMM_EINVAL, "FFT M2L chunk: too many items"};
        }
        std::vector<int64_t> start(ch.npar + 1, 0);
        for (int64_t q = 0; q < ch.npar; ++q) start[q + 1] = start[q] + cnt[q];
        // processing order: the units (parents, or half parents when item_nb() == 4) dealt
        // round-robin to W warps per frequency group (W = warps per CTA x CTAs per group, >= 4
        // units per warp), warp slot s taking unit positions s, s + W, s + 2W, ...; ord / ioff /
        // items follow that order, wrange cuts it per warp
        const bool grp = sparse_groups();
        const int nbu = grp ? 4 : item_nb(), halves = nbu == 8 ? 1 : 2;
        const int64_t nunit = ch.npar * halves;
        const int64_t wpc = grp ? GROUP_WARPS : nbu == 8 ? ItemCfg<8>::WARPS : ItemCfg<4>::WARPS;
        const int64_t X = std::min<int64_t>(148, std::max<int64_t>(1, (nunit + wpc * 4 - 1) / (wpc * 4)));
        const int64_t W = X * wpc;
        std::vector<int32_t> ord, ioff(1, 0), wr(1, 0);
        std::vector<int2> items;
        ord.reserve(nunit);
        items.reserve(all.size() * halves);
        // k_m2l_groups takes its ranges dynamically: a range is GROUP_CHUNK (4; measured C5 product 8: 431, 4: 425, 16: 435 ms) consecutive
        // positions of one slot, a CTA's ranges ordered chunk-major (all its slots' first
        // chunk, then the second, ...) so that the warps of the whole grid still sweep the
        // same window of Morton-adjacent parents; a warp that finishes early takes the next
        // range of its CTA (ncu, C5 level 9, static ranges: 10.8 of 12 warps active on
        // average, the sub-partitions idle 5% of the cycles).  k_m2l_items keeps one range per
        // warp (chunk = all positions).
        const int64_t npos = (nunit + W - 1) / W;
        const int64_t cpos = grp ? group_chunk() : std::max<int64_t>(1, npos);
        const int64_t nchunk = std::max<int64_t>(1, (npos + cpos - 1) / cpos);
        for (int64_t rg = 0; rg < X * nchunk * wpc; ++rg) {
          // range rg = (CTA x, chunk j, warp slot s) -> slot sl, positions [j cpos, (j + 1) cpos)
          const int64_t x = rg / (nchunk * wpc), j = (rg / wpc) % nchunk, sl = x * wpc + rg % wpc;
          for (int64_t pos = j * cpos; pos < std::min(npos, (j + 1) * cpos); ++pos) {
            const int64_t u = pos * W + sl;
            if (u >= nunit) continue;
            const int64_t q = u / halves;
            const int h = (int)(u % halves);
            ord.push_back((int32_t)(halves == 1 ? q : 2 * q + h));
            if (grp) {  // groups (unit, d, cx) of k_m2l_groups; items arrive in (d, c) order
              int2 cur = make_int2(0, -1);
              for (int64_t e = start[q]; e < start[q + 1]; ++e) {
                const unsigned y = (unsigned)all[e].y;
                const unsigned vm = ((y >> 11) >> (4 * h)) & 15u;
                if (!vm) continue;
                const unsigned dd = (y & 2047u) >> 6, c = y & 7u, cx = c >> 2, cq = c & 3u;
                const unsigned key = (dd * 2 + (unsigned)h) * 2 + cx;  // the c_grow row
                if (cur.y < 0 || ((unsigned)cur.y & 127u) != key) {
                  if (cur.y >= 0) items.push_back(cur);
                  cur = make_int2(all[e].x - (int)(cq * P.kml * 32), (int)key);
                }
                unsigned pm = 0;
                for (int t = 0; t < 4; ++t)
                  if ((vm >> t) & 1u) pm |= 1u << (4 * t + cq);
                cur.y = (int)((unsigned)cur.y | (pm << 7) | (1u << (23 + cq)));
              }
              if (cur.y >= 0) items.push_back(cur);
              ioff.push_back((int32_t)items.size());
              continue;
            }
            for (int64_t e = start[q]; e < start[q + 1]; ++e) {
              int2 it = all[e];
              if (halves == 2) {
                const unsigned vm = (((unsigned)it.y >> 11) >> (4 * h)) & 15u;
                if (!vm) continue;
                it.y = (int)(((unsigned)it.y & ~(255u << 11)) | (vm << 11));
              }
              items.push_back(it);
            }
            ioff.push_back((int32_t)items.size());
          }
          wr.push_back((int32_t)ord.size());
        }
        ch.nitems = (int64_t)items.size();
        ch.groups = grp;
        ch.nrange = X * nchunk * wpc;
        ch.nper = nchunk * wpc;
        ch.d_ioff = dalloc<int32_t>(P, ioff.size());
        ch.d_ord = dalloc<int32_t>(P, std::max<size_t>(1, ord.size()));
        ch.d_wrange = dalloc<int32_t>(P, wr.size());
        ch.d_items = dalloc<int2>(P, std::max<size_t>(1, items.size()));
        KF_CUDA(cudaMemcpyAsync(ch.d_ioff, ioff.data(), ioff.size() * 4, cudaMemcpyHostToDevice, st));
        if (!ord.empty()) KF_CUDA(cudaMemcpyAsync(ch.d_ord, ord.data(), ord.size() * 4, cudaMemcpyHostToDevice, st));
        KF_CUDA(cudaMemcpyAsync(ch.d_wrange, wr.data(), wr.size() * 4, cudaMemcpyHostToDevice, st));
        if (!items.empty())
          KF_CUDA(cudaMemcpyAsync(ch.d_items, items.data(), items.size() * 8, cudaMemcpyHostToDevice, st));
        KF_CUDA(cudaStreamSynchronize(st));
      }
      ch.d_tpat = dalloc<uint8_t>(P, std::max<int64_t>(1, ch.npar));
      KF_CUDA(cudaMemcpyAsync(ch.d_tpat, tpat.data(), ch.npar, cudaMemcpyHostToDevice, st));
      ch.d_qbox = dalloc<int32_t>(P, std::max<int64_t>(1, ch.nq));
      ch.d_nbr = dalloc<int32_t>(P, ch.npar * 26);
      ch.d_tbox = dalloc<int32_t>(P, std::max<int64_t>(1, ch.nt));
      ch.d_tpb = dalloc<int2>(P, std::max<int64_t>(1, ch.nt));
      ch.d_toff = dalloc<int32_t>(P, toff.size());
      KF_CUDA(cudaMemcpyAsync(ch.d_toff, toff.data(), toff.size() * 4, cudaMemcpyHostToDevice, st));
      if (ch.nq) KF_CUDA(cudaMemcpyAsync(ch.d_qbox, qs.data(), ch.nq * 4, cudaMemcpyHostToDevice, st));
      KF_CUDA(cudaMemcpyAsync(ch.d_nbr, nb.data(), ch.npar * 26 * 4, cudaMemcpyHostToDevice, st));
      if (!P.h_row.empty())  // the inverse transform writes CHK rows
        for (int32_t& t : tb) t = P.h_row[t];
      if (ch.nt) {
        KF_CUDA(cudaMemcpyAsync(ch.d_tbox, tb.data(), ch.nt * 4, cudaMemcpyHostToDevice, st));
        KF_CUDA(cudaMemcpyAsync(ch.d_tpb, tpb.data(), ch.nt * 8, cudaMemcpyHostToDevice, st));
      }
      KF_CUDA(cudaStreamSynchronize(st));
      for (int32_t q : qs) qlocal[q] = -1;
      P.fft_max_nq = std::max(P.fft_max_nq, ch.nq);
      P.fft_max_npar = std::max(P.fft_max_npar, ch.npar);
      P.fft_chunks.push_back(ch);
      i0 = i1;
    }
  }
  dfree(P, P.d_ub);
  dfree(P, P.d_cb);
  P.d_ub = dalloc<double2>(P, (size_t)std::max<int64_t>(1, P.fft_max_nq) * R * P.NFP);
  P.d_cb = dalloc<double2>(P, (size_t)std::max<int64_t>(1, P.fft_max_npar) * R * P.NFP);
}

}  // namespace kafmm
