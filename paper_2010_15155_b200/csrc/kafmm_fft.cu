// M2L as a convolution on the regular (2p)^3 lattice grid (SURVEY.md §8(a) a5,
// option b; the paper's M2L cost remark P:633 refers to PVFMM's FFT M2L).
//
// The upward-equivalent surface of a source box C and the downward-check
// surface of a target box B (both radius 1.05 h) are boundary points of p^3
// lattices with the same spacing delta = 2*1.05 h/(p-1).  For C = B + 2h o,
//     check_B(I) = sum_J K(delta (I - J) - 2 h o) ue_C(J),   I, J in [0,p)^3,
// a 3D linear convolution with the kernel grid t_o(D) = K(delta D - 2 h o),
// D in [-(p-1), p-1]^3.  Zero-padded to NG = 2p it is a circular convolution:
//     check_B = IDFT( sum_{C in V(B)} That_o . DFT(ue_C) )  on the lattice.
// This is exactly the dense M2L (up to rounding): same matrices, factored.
//
// Hot path per level and chunk (all on the plan's stream):
//   k_fft_fwd   one CTA per source box: real DFT of ue (p^3 cube, surface only
//               non-zero) -> Uhat[box][comp][NG*NG*(p+1)], staged z, y, x in SMEM
//   k_m2l_had   PVFMM-style blocking: for a frequency f and a target parent P,
//               Chat[children of P](f) = sum over the 26 colleague directions d
//               and the 8x8 (target child, source child) pairs of That_o(f)
//               Uhat(f), o = 2d + oct(c) - oct(b), skipping adjacent pairs;
//               CTA = 16 frequencies x NPB parents, accumulators in registers
//   k_fft_inv   one CTA per target box: inverse DFT, evaluated only at the
//               downward-check surface points, times 2^l / NG^3, added to CHK
// Operator spectra That_o (316 offsets, level 0) are computed once at setup
// with cuFFT (setup only; not on the hot path).
#include <cufft.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <vector>

#include "kafmm_internal.h"

namespace kafmm {

__constant__ int16_t c_fft_off_id[343];  // (ox+3)*49+(oy+3)*7+(oz+3) -> offset id (or -1)

static inline unsigned nblk(int64_t n, int t = 256) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

// ---------------------------------------------------------------------------
// setup: kernel grids t_o and their spectra
// ---------------------------------------------------------------------------
__device__ __forceinline__ int dmap(int g, int p, int NG) { return g < p ? g : (g > p ? g - NG : INT_MIN); }

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
template <int P>
struct FftDims {
  static constexpr int NG = 2 * P, NZ = P + 1, NF = NG * NG * NZ;
  static constexpr int CUBE = (P * P * P + 1) / 2 * 2;  // doubles, keep 16-B alignment after it
  static constexpr size_t FWD_SMEM = (CUBE + 2 * (P * P * NZ + P * NG * NZ + NG)) * sizeof(double);
  static constexpr size_t INV_SMEM = 2 * (P * NG * NZ + P * P * NZ + NG) * sizeof(double);
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ void cmac(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
}

template <int P>
__global__ void __launch_bounds__(256)
    k_fft_fwd(const int32_t* __restrict__ src, const double* __restrict__ ue, int ldn, int kml,
              const int16_t* __restrict__ lat, int M, double2* __restrict__ uhat) {
  using D = FftDims<P>;
  constexpr int NG = D::NG, NZ = D::NZ, NF = D::NF;
  extern __shared__ __align__(16) double sm[];
  double* cube = sm;
  double2* A = reinterpret_cast<double2*>(sm + D::CUBE);  // [x][y][fz]
  double2* B = A + P * P * NZ;                              // [x][fy][fz]
  double2* tw = B + P * NG * NZ;                            // w^j = exp(-2 pi i j / NG)
  const int s = blockIdx.x, tid = threadIdx.x, bd = blockDim.x;
  const int64_t box = src[s];
  for (int j = tid; j < NG; j += bd) {
    double sn, cs;
    sincospi(2.0 * j / NG, &sn, &cs);
    tw[j] = make_double2(cs, -sn);
  }
  for (int e = 0; e < kml; ++e) {
    for (int i = tid; i < P * P * P; i += bd) cube[i] = 0.0;
    __syncthreads();
    for (int m = tid; m < M; m += bd)
      cube[(lat[3 * m] * P + lat[3 * m + 1]) * P + lat[3 * m + 2]] = ue[box * ldn + m * kml + e];
    __syncthreads();
    for (int idx = tid; idx < P * P * NZ; idx += bd) {  // z: real -> half spectrum
      int xy = idx / NZ, fz = idx - xy * NZ;
      const double* c = cube + xy * P;
      double re = 0.0, im = 0.0;
      int k = 0;
#pragma unroll
      for (int z = 0; z < P; ++z) {
        re = fma(c[z], tw[k].x, re);
        im = fma(c[z], tw[k].y, im);
        k += fz;
        if (k >= NG) k -= NG;
      }
      A[idx] = make_double2(re, im);
    }
    __syncthreads();
    for (int idx = tid; idx < P * NG * NZ; idx += bd) {  // y
      int x = idx / (NG * NZ), r = idx - x * NG * NZ, fy = r / NZ, fz = r - fy * NZ;
      const double2* a = A + x * P * NZ + fz;
      double2 acc = make_double2(0.0, 0.0);
      int k = 0;
#pragma unroll
      for (int y = 0; y < P; ++y) {
        cmac(acc, a[y * NZ], tw[k]);
        k += fy;
        if (k >= NG) k -= NG;
      }
      B[idx] = acc;
    }
    __syncthreads();
    double2* out = uhat + ((int64_t)s * kml + e) * NF;
    for (int idx = tid; idx < NF; idx += bd) {  // x
      int fx = idx / (NG * NZ), r = idx - fx * NG * NZ;
      const double2* b = B + r;
      double2 acc = make_double2(0.0, 0.0);
      int k = 0;
#pragma unroll
      for (int x = 0; x < P; ++x) {
        cmac(acc, b[x * NG * NZ], tw[k]);
        k += fx;
        if (k >= NG) k -= NG;
      }
      out[idx] = acc;
    }
    __syncthreads();
  }
}

template <int P>
__global__ void __launch_bounds__(256)
    k_fft_inv(int64_t t0, const int32_t* __restrict__ level, const double2* __restrict__ chat, int kml,
              const int16_t* __restrict__ lat, int M, double* __restrict__ chk, int ldn) {
  using D = FftDims<P>;
  constexpr int NG = D::NG, NZ = D::NZ, NF = D::NF;
  extern __shared__ __align__(16) double sm[];
  double2* Dx = reinterpret_cast<double2*>(sm);  // [x][fy][fz]
  double2* E = Dx + P * NG * NZ;                  // [x][y][fz]
  double2* tw = E + P * P * NZ;                   // exp(+2 pi i j / NG)
  const int t = blockIdx.x, tid = threadIdx.x, bd = blockDim.x;
  const int64_t box = t0 + t;
  const double scale = ldexp(1.0, level[box]) / (double)(NG * NG * NG);
  for (int j = tid; j < NG; j += bd) {
    double sn, cs;
    sincospi(2.0 * j / NG, &sn, &cs);
    tw[j] = make_double2(cs, sn);
  }
  __syncthreads();
  for (int a = 0; a < kml; ++a) {
    const double2* c = chat + ((int64_t)t * kml + a) * NF;
    for (int idx = tid; idx < P * NG * NZ; idx += bd) {  // x: only x in [0, P)
      int x = idx / (NG * NZ), r = idx - x * NG * NZ;
      double2 acc = make_double2(0.0, 0.0);
      int k = 0;
#pragma unroll 4
      for (int fx = 0; fx < NG; ++fx) {
        cmac(acc, c[fx * NG * NZ + r], tw[k]);
        k += x;
        if (k >= NG) k -= NG;
      }
      Dx[idx] = acc;
    }
    __syncthreads();
    for (int idx = tid; idx < P * P * NZ; idx += bd) {  // y: only y in [0, P)
      int x = idx / (P * NZ), r = idx - x * P * NZ, y = r / NZ, fz = r - y * NZ;
      const double2* d = Dx + x * NG * NZ + fz;
      double2 acc = make_double2(0.0, 0.0);
      int k = 0;
#pragma unroll 4
      for (int fy = 0; fy < NG; ++fy) {
        cmac(acc, d[fy * NZ], tw[k]);
        k += y;
        if (k >= NG) k -= NG;
      }
      E[idx] = acc;
    }
    __syncthreads();
    double* o = chk + box * ldn;
    for (int m = tid; m < M; m += bd) {  // z: half spectrum -> real, only at surface points
      int x = lat[3 * m], y = lat[3 * m + 1], z = lat[3 * m + 2];
      const double2* e = E + (x * P + y) * NZ;
      double v = e[0].x;
      int k = z;
      for (int fz = 1; fz < P; ++fz) {
        v += 2.0 * (e[fz].x * tw[k].x - e[fz].y * tw[k].y);
        k += z;
        if (k >= NG) k -= NG;
      }
      v += e[P].x * ((z & 1) ? -1.0 : 1.0);  // Nyquist bin
      o[m * kml + a] += scale * v;
    }
    __syncthreads();
  }
}

constexpr int HAD_THREADS = 128;
constexpr int HAD_FPB = HAD_THREADS / 8;  // frequencies per block (8 target children per frequency)

template <int KML, int NPB>
__global__ void __launch_bounds__(HAD_THREADS)
    k_m2l_had(int NF, int npar, const double2* __restrict__ that, const double2* __restrict__ uhat,
              double2* __restrict__ chat, const int2* __restrict__ par, const int2* __restrict__ nbr) {
  constexpr int NC = KML == 1 ? 1 : 6;
  __shared__ int2 s_nbr[NPB * 26];
  __shared__ int2 s_par[NPB];
  const int nbp = (npar + NPB - 1) / NPB;
  const int pb = blockIdx.x % nbp, fc = blockIdx.x / nbp;
  const int b = threadIdx.x & 7, fi = threadIdx.x >> 3;
  const int f = fc * HAD_FPB + fi;
  const bool fok = f < NF;
  const int fs = fok ? f : NF - 1;
  const int P0 = pb * NPB;
  for (int i = threadIdx.x; i < NPB * 26; i += HAD_THREADS) {
    int pp = P0 + i / 26;
    s_nbr[i] = pp < npar ? nbr[(int64_t)P0 * 26 + i] : make_int2(0, 0);
  }
  for (int i = threadIdx.x; i < NPB; i += HAD_THREADS) s_par[i] = (P0 + i < npar) ? par[P0 + i] : make_int2(0, 0);
  __syncthreads();
  double2 acc[NPB][KML];
#pragma unroll
  for (int q = 0; q < NPB; ++q)
#pragma unroll
    for (int a = 0; a < KML; ++a) acc[q][a] = make_double2(0.0, 0.0);
  const int bx = (b >> 2) & 1, by = (b >> 1) & 1, bz = b & 1;
  const double2* tf = that + (int64_t)fs * N_OFFSETS * NC;
  for (int dd = 0; dd < 26; ++dd) {
    const int d = dd < 13 ? dd : dd + 1;  // skip the centre (0,0,0)
    const int dx = d / 9 - 1, dy = (d / 3) % 3 - 1, dz = d % 3 - 1;
    for (int c = 0; c < 8; ++c) {
      const int ox = 2 * dx + ((c >> 2) & 1) - bx, oy = 2 * dy + ((c >> 1) & 1) - by, oz = 2 * dz + (c & 1) - bz;
      if (max(abs(ox), max(abs(oy), abs(oz))) < 2) continue;  // adjacent: U list, not V
      const int oid = c_fft_off_id[(ox + 3) * 49 + (oy + 3) * 7 + (oz + 3)];
      double2 T[NC];
#pragma unroll
      for (int i = 0; i < NC; ++i) T[i] = tf[oid * NC + i];
      const int lowmask = (1 << c) - 1;
#pragma unroll
      for (int q = 0; q < NPB; ++q) {
        const int2 nb = s_nbr[q * 26 + dd];
        if ((nb.y >> c) & 1) {
          const int64_t s = nb.x + __popc(nb.y & lowmask);
          if (KML == 1) {
            cmac(acc[q][0], T[0], uhat[s * NF + fs]);
          } else {
            const double2 u0 = uhat[(s * 3 + 0) * NF + fs];
            const double2 u1 = uhat[(s * 3 + 1) * NF + fs];
            const double2 u2 = uhat[(s * 3 + 2) * NF + fs];
            cmac(acc[q][0], T[0], u0);
            cmac(acc[q][0], T[1], u1);
            cmac(acc[q][0], T[2], u2);
            cmac(acc[q][KML > 1 ? 1 : 0], T[1], u0);
            cmac(acc[q][KML > 1 ? 1 : 0], T[3], u1);
            cmac(acc[q][KML > 1 ? 1 : 0], T[4], u2);
            cmac(acc[q][KML > 2 ? 2 : 0], T[2], u0);
            cmac(acc[q][KML > 2 ? 2 : 0], T[4], u1);
            cmac(acc[q][KML > 2 ? 2 : 0], T[5], u2);
          }
        }
      }
    }
  }
  if (!fok) return;
#pragma unroll
  for (int q = 0; q < NPB; ++q) {
    const int2 pp = s_par[q];
    if ((pp.y >> b) & 1) {
      const int64_t t = pp.x + __popc(pp.y & ((1 << b) - 1));
#pragma unroll
      for (int a = 0; a < KML; ++a) chat[(t * KML + a) * NF + f] = acc[q][a];
    }
  }
}

// ---------------------------------------------------------------------------
// host
// ---------------------------------------------------------------------------
template <int P>
static void set_smem_attrs() {
  static bool done = false;
  if (done) return;
  KF_CUDA(cudaFuncSetAttribute(k_fft_fwd<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)FftDims<P>::FWD_SMEM));
  KF_CUDA(cudaFuncSetAttribute(k_fft_inv<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)FftDims<P>::INV_SMEM));
  done = true;
}

template <int P>
static void launch_fwd(Plan& Pl, const FftChunk& ch) {
  set_smem_attrs<P>();
  k_fft_fwd<P><<<(unsigned)ch.ns, 256, FftDims<P>::FWD_SMEM, Pl.stream>>>(ch.d_src, Pl.d_ue, Pl.ldn, Pl.kml,
                                                                           Pl.d_lat, Pl.M, Pl.d_uhat);
  KF_CHECK_LAUNCH();
  Pl.launches++;
}
template <int P>
static void launch_inv(Plan& Pl, const FftChunk& ch) {
  set_smem_attrs<P>();
  k_fft_inv<P><<<(unsigned)ch.nt, 256, FftDims<P>::INV_SMEM, Pl.stream>>>(ch.t0, Pl.d_level, Pl.d_chat, Pl.kml,
                                                                           Pl.d_lat, Pl.M, Pl.d_chk, Pl.ldn);
  KF_CHECK_LAUNCH();
  Pl.launches++;
}

static void dispatch_fwd(Plan& Pl, const FftChunk& ch) {
  switch (Pl.p) {
    case 4: launch_fwd<4>(Pl, ch); break;
    case 5: launch_fwd<5>(Pl, ch); break;
    case 6: launch_fwd<6>(Pl, ch); break;
    case 7: launch_fwd<7>(Pl, ch); break;
    case 8: launch_fwd<8>(Pl, ch); break;
    case 10: launch_fwd<10>(Pl, ch); break;
    case 12: launch_fwd<12>(Pl, ch); break;
    default: throw Error{KAFMM_EINVAL, "FFT M2L: unsupported p"};
  }
}
static void dispatch_inv(Plan& Pl, const FftChunk& ch) {
  switch (Pl.p) {
    case 4: launch_inv<4>(Pl, ch); break;
    case 5: launch_inv<5>(Pl, ch); break;
    case 6: launch_inv<6>(Pl, ch); break;
    case 7: launch_inv<7>(Pl, ch); break;
    case 8: launch_inv<8>(Pl, ch); break;
    case 10: launch_inv<10>(Pl, ch); break;
    case 12: launch_inv<12>(Pl, ch); break;
    default: throw Error{KAFMM_EINVAL, "FFT M2L: unsupported p"};
  }
}

bool fft_supported_p(int p) { return p == 4 || p == 5 || p == 6 || p == 7 || p == 8 || p == 10 || p == 12; }

void run_m2l_fft(Plan& Pl) {
  for (const FftChunk& ch : Pl.fft_chunks) {
    if (ch.nt == 0 || ch.ns == 0) continue;
    dispatch_fwd(Pl, ch);
    const int nbp_1 = (int)((ch.npar + 15) / 16), nbp_3 = (int)((ch.npar + 3) / 4);
    const int nfc = (Pl.NF + HAD_FPB - 1) / HAD_FPB;
    if (Pl.kml == 1)
      k_m2l_had<1, 16><<<(unsigned)((int64_t)nbp_1 * nfc), HAD_THREADS, 0, Pl.stream>>>(
          Pl.NF, (int)ch.npar, Pl.d_that, Pl.d_uhat, Pl.d_chat, ch.d_par, ch.d_nbr);
    else
      k_m2l_had<3, 4><<<(unsigned)((int64_t)nbp_3 * nfc), HAD_THREADS, 0, Pl.stream>>>(
          Pl.NF, (int)ch.npar, Pl.d_that, Pl.d_uhat, Pl.d_chat, ch.d_par, ch.d_nbr);
    KF_CHECK_LAUNCH();
    Pl.launches++;
    dispatch_inv(Pl, ch);
  }
}

template <class T>
static void d2h(Plan& P, std::vector<T>& h, const T* d, int64_t n) {
  h.resize(n);
  if (n) KF_CUDA(cudaMemcpy(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost));
}

void build_fft_m2l(Plan& P, int64_t budget) {
  if (!fft_supported_p(P.p)) {
    P.m2l_mode = M2L_DENSE;
    return;
  }
  cudaStream_t st = P.stream;
  const int p = P.p;
  P.NG = 2 * p;
  P.NZ = p + 1;
  P.NF = P.NG * P.NG * P.NZ;
  P.ncomp = P.kml == 1 ? 1 : 6;
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
  KF_CUDA(cudaMemcpyToSymbol(c_fft_off_id, tab, sizeof(tab)));
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
    k_kernel_grid<<<g, 256, 0, st>>>(p, NG, P.kml, 1.05 / (p - 1), d_offs, grid);
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
  // chunks: per level l >= 2, Morton-contiguous target parents at level l-1
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
  const int64_t per_box = (int64_t)P.kml * P.NF * 16;
  P.fft_chunks.clear();
  P.fft_max_ns = P.fft_max_nt = 0;
  for (int l = 2; l <= P.depth; ++l) {
    const int64_t lb = P.levels[l].begin, le = P.levels[l].end;
    std::vector<int32_t> local(le - lb, -1);
    std::vector<int64_t> parents;
    for (int64_t b = P.levels[l - 1].begin; b < P.levels[l - 1].end; ++b)
      if (!leaf[b]) parents.push_back(b);
    size_t i0 = 0;
    while (i0 < parents.size()) {
      // grow the chunk until the source + target spectra exceed the budget
      std::vector<int64_t> nbrs;  // (26 per parent) colleague ids or -1
      std::vector<int32_t> srcs;
      int64_t nt = 0;
      size_t i1 = i0;
      while (i1 < parents.size()) {
        const int64_t Pb = parents[i1];
        int64_t add_src = 0;
        int64_t qs[26];
        for (int dd = 0; dd < 26; ++dd) {
          int d = dd < 13 ? dd : dd + 1;
          int64_t q = find(l - 1, ijk[3 * Pb] + d / 9 - 1, ijk[3 * Pb + 1] + (d / 3) % 3 - 1, ijk[3 * Pb + 2] + d % 3 - 1);
          if (q >= 0 && leaf[q]) q = -1;
          qs[dd] = q;
          if (q >= 0) {
            int64_t c0 = -1;
            for (int o = 0; o < 8; ++o)
              if (child[8 * q + o] >= 0) {
                c0 = child[8 * q + o];
                break;
              }
            if (local[c0 - lb] < 0) {
              for (int o = 0; o < 8; ++o) add_src += child[8 * q + o] >= 0;
            }
          }
        }
        int64_t add_t = 0;
        for (int o = 0; o < 8; ++o) add_t += child[8 * Pb + o] >= 0;
        if (i1 > i0 && ((int64_t)srcs.size() + add_src + nt + add_t) * per_box > budget) break;
        for (int dd = 0; dd < 26; ++dd) {
          int64_t q = qs[dd];
          nbrs.push_back(q);
          if (q >= 0) {
            for (int o = 0; o < 8; ++o) {
              int64_t c = child[8 * q + o];
              if (c >= 0 && local[c - lb] < 0) {
                local[c - lb] = 0;  // mark; final local indices after sorting
                srcs.push_back((int32_t)c);
              }
            }
          }
        }
        nt += add_t;
        ++i1;
      }
      std::sort(srcs.begin(), srcs.end());
      for (size_t s = 0; s < srcs.size(); ++s) local[srcs[s] - lb] = (int32_t)s;
      FftChunk ch;
      ch.level = l;
      ch.npar = (int64_t)(i1 - i0);
      ch.ns = (int64_t)srcs.size();
      ch.nt = nt;
      // targets: children of parents[i0..i1) form one contiguous id range
      int64_t t0 = -1;
      for (int o = 0; o < 8 && t0 < 0; ++o)
        if (child[8 * parents[i0] + o] >= 0) t0 = child[8 * parents[i0] + o];
      ch.t0 = t0;
      std::vector<int2> hpar(ch.npar), hnbr(ch.npar * 26);
      for (int64_t q = 0; q < ch.npar; ++q) {
        const int64_t Pb = parents[i0 + q];
        int mask = 0, first = -1;
        for (int o = 0; o < 8; ++o)
          if (child[8 * Pb + o] >= 0) {
            mask |= 1 << o;
            if (first < 0) first = child[8 * Pb + o];
          }
        hpar[q] = make_int2((int)(first - t0), mask);
        for (int dd = 0; dd < 26; ++dd) {
          int64_t Q = nbrs[q * 26 + dd];
          int m2 = 0, f2 = -1;
          if (Q >= 0)
            for (int o = 0; o < 8; ++o)
              if (child[8 * Q + o] >= 0) {
                m2 |= 1 << o;
                if (f2 < 0) f2 = child[8 * Q + o];
              }
          hnbr[q * 26 + dd] = (Q >= 0) ? make_int2(local[f2 - lb], m2) : make_int2(0, 0);
        }
      }
      ch.d_src = dalloc<int32_t>(P, std::max<int64_t>(1, ch.ns));
      ch.d_par = dalloc<int2>(P, ch.npar);
      ch.d_nbr = dalloc<int2>(P, ch.npar * 26);
      if (ch.ns) KF_CUDA(cudaMemcpyAsync(ch.d_src, srcs.data(), ch.ns * 4, cudaMemcpyHostToDevice, st));
      KF_CUDA(cudaMemcpyAsync(ch.d_par, hpar.data(), ch.npar * 8, cudaMemcpyHostToDevice, st));
      KF_CUDA(cudaMemcpyAsync(ch.d_nbr, hnbr.data(), ch.npar * 26 * 8, cudaMemcpyHostToDevice, st));
      KF_CUDA(cudaStreamSynchronize(st));
      for (int32_t s : srcs) local[s - lb] = -1;
      P.fft_max_ns = std::max(P.fft_max_ns, ch.ns);
      P.fft_max_nt = std::max(P.fft_max_nt, ch.nt);
      P.fft_chunks.push_back(ch);
      i0 = i1;
    }
  }
  P.d_uhat = dalloc<double2>(P, (size_t)std::max<int64_t>(1, P.fft_max_ns) * P.kml * P.NF);
  P.d_chat = dalloc<double2>(P, (size_t)std::max<int64_t>(1, P.fft_max_nt) * P.kml * P.NF);
}

}  // namespace kafmm
