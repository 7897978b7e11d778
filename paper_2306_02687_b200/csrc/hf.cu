// High-fidelity RVE solve on the device and the POD basis built from its
// snapshots (SURVEY §8(f) rank 2 — the offline stage that replaces the seeded
// Φ with physical modes).
//
// Reference behaviour followed (paths relative to
// /root/reference/proj/include/fe2rom/ unless noted):
//   assemble_micro                      rve.hpp:220-262
//   micro_newton (8-halving Armijo LS)   rve.hpp:285-346
//   homogenize (3 sensitivity solves)    rve.hpp:350-392
//   run_trajectory + SnapshotRecorder    rve.hpp:397-494 (x_u = u - E.x per step)
//   build_elastic_modes, pod
//
// Device layout: the material update, strains and element stiffness run in
// k_hf_element (one CTA per Tri6 element, 144 threads = its 12x12 entries);
// k_hf_gather_band sums the element vectors/matrices into the residual and
// the LOWER BAND of the free stiffness (free DOFs in reverse Cuthill-McKee
// order) with ONE thread per DOF walking its element incidences in ascending
// element order — the reference's assembly order, no atomics,
// bit-reproducible. k_band_chol / k_band_solve factor and solve the band on
// one CTA (the reference factors with sparse SimplicialLDLT, rve.hpp:295-325).
// Many RVE solves run at once (fe2_hf_trajectories, the FE² HF engine's
// points): one worker = one stream + buffers + host thread. The POD SVD is
// cuSOLVER gesvd (dlopen'ed at first use). Host code keeps the Newton control
// flow, norms and the homogenisation sums (a few thousand integration points).
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <type_traits>
#include <thread>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <vector>

#include "common.hpp"
#include "fe2rom/fe2rom_gpu.h"
#include "host_util.cuh"
#include "material.cuh"
#include "rve.hpp"

namespace fe2 {

namespace {

// ---------------------------------------------------------------------------
// cuSOLVER, resolved at first use.
struct Cusolver {
  decltype(&cusolverDnCreate) create = nullptr;
  decltype(&cusolverDnDestroy) destroy = nullptr;
  decltype(&cusolverDnSetStream) set_stream = nullptr;
  decltype(&cusolverDnDgesvd_bufferSize) gesvd_ws = nullptr;
  decltype(&cusolverDnDgesvd) gesvd = nullptr;
  std::string err;

  static const Cusolver& get() {
    static const Cusolver s = load();
    check(s.err.empty(), Code::solver, s.err);
    return s;
  }

 private:
  static Cusolver load() {
    Cusolver s;
    void* lib = nullptr;
    for (const char* name : {"libcusolver.so.11", "/usr/local/cuda/lib64/libcusolver.so.11", "libcusolver.so"})
      if ((lib = dlopen(name, RTLD_NOW | RTLD_LOCAL))) break;
    if (!lib) {
      s.err = "cannot load cuSOLVER (libcusolver.so.11)";
      return s;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(lib, name));
      if (!fn && s.err.empty()) s.err = std::string("cuSOLVER symbol missing: ") + name;
    };
    sym(s.create, "cusolverDnCreate");
    sym(s.destroy, "cusolverDnDestroy");
    sym(s.set_stream, "cusolverDnSetStream");
    sym(s.gesvd_ws, "cusolverDnDgesvd_bufferSize");
    sym(s.gesvd, "cusolverDnDgesvd");
    return s;
  }
};

void sol_check(cusolverStatus_t st, const char* what) {
  if (st != CUSOLVER_STATUS_SUCCESS)
    throw Failure(Code::solver, std::string("cuSOLVER ") + what + " failed (status " + std::to_string(int(st)) + ")");
}

constexpr int kMaxMats = 8;
struct MatTable {
  MatDev m[kMaxMats];
};

// ---------------------------------------------------------------------------
// Kernels

// One CTA per element: strains + material update at its 3 integration points
// (threads 0-2), element force (threads 0-11) and, with_K, the 12x12 element
// stiffness (thread t = entry (t / 12, t % 12)). Arithmetic order follows
// assemble_micro (rve.hpp:233-256): eps = B u_el, f_a += (B^T sigma)_a w,
// k_ab += (B^T (C B))_ab w over the points in order.
__global__ void __launch_bounds__(144) k_hf_element(int n_el, const int* __restrict__ conn,
                                                    const int* __restrict__ phase, MatTable mats,
                                                    const double* __restrict__ B, const double* __restrict__ w,
                                                    const double* __restrict__ u, const double* __restrict__ st0,
                                                    int with_K, double* __restrict__ f_el, double* __restrict__ k_el,
                                                    double* __restrict__ st_out, double* __restrict__ sig_out,
                                                    double* __restrict__ C_out, int* __restrict__ err) {
  const int e = blockIdx.x, t = threadIdx.x;
  if (e >= n_el) return;
  __shared__ double sB[3][36], sS[3][3], sC[3][9], sW[3];
  for (int i = t; i < 108; i += blockDim.x) sB[i / 36][i % 36] = B[(size_t)108 * e + i];
  __syncthreads();
  if (t < 3) {
    const int ip = 3 * e + t;
    double ue[12];
    for (int a = 0; a < 6; ++a) {
      const int nd = conn[6 * e + a];
      ue[2 * a] = u[2 * nd];
      ue[2 * a + 1] = u[2 * nd + 1];
    }
    double eps[3];
    for (int r = 0; r < 3; ++r) {
      double s = 0.0;
      for (int c = 0; c < 12; ++c) s += sB[t][r * 12 + c] * ue[c];
      eps[r] = s;
    }
    const double* s0 = st0 + (size_t)6 * ip;
    bool ok = true;
    const MatOut o =
        update_material_any(mats.m[phase[e]], s0[0], s0[1], s0[2], s0[3], s0[4], eps[0], eps[1], eps[2], ok);
    if (!ok) atomicExch(err, 1);
    sS[t][0] = o.s0;
    sS[t][1] = o.s1;
    sS[t][2] = o.s2;
    const double Cf[9] = {o.c00, o.c01, o.c02, o.c01, o.c11, o.c12, o.c02, o.c12, o.c22};
    for (int k = 0; k < 9; ++k) sC[t][k] = Cf[k];
    sW[t] = w[ip];
    if (with_K) {
      double* so = st_out + (size_t)6 * ip;
      so[0] = o.ep0;
      so[1] = o.ep1;
      so[2] = o.ep2;
      so[3] = o.ep3;
      so[4] = o.eq;
      so[5] = o.s33;
      sig_out[3 * ip] = o.s0;
      sig_out[3 * ip + 1] = o.s1;
      sig_out[3 * ip + 2] = o.s2;
      for (int k = 0; k < 9; ++k) C_out[(size_t)9 * ip + k] = Cf[k];
    }
  }
  __syncthreads();
  if (t < 12) {
    double f = 0.0;
    for (int g = 0; g < 3; ++g) {
      double s = 0.0;
      for (int i = 0; i < 3; ++i) s += sB[g][i * 12 + t] * sS[g][i];
      f += s * sW[g];
    }
    f_el[(size_t)12 * e + t] = f;
  }
  if (with_K) {
    const int a = t / 12, b = t % 12;
    double k = 0.0;
    for (int g = 0; g < 3; ++g) {
      double s = 0.0;
      for (int i = 0; i < 3; ++i) {
        double cb = 0.0;
        for (int j = 0; j < 3; ++j) cb += sC[g][3 * i + j] * sB[g][j * 12 + b];
        s += sB[g][i * 12 + a] * cb;
      }
      k += s * sW[g];
    }
    k_el[(size_t)144 * e + t] = k;
  }
}

// ---------------------------------------------------------------------------
// Banded Cholesky of the micro stiffness (replaces a dense factorisation; the
// reference factors with sparse SimplicialLDLT, rve.hpp:295-325). The free
// DOFs are numbered in reverse Cuthill-McKee order (band_order), which keeps
// every element's DOFs within a half bandwidth bw (275 for default_cell(33),
// n = 7,910: n bw^2 / 2 = 0.3 G FMA per factorisation instead of n^3 / 6 =
// 82 G). Column-band storage: Kb[c * ldb + (r - c)], 0 <= r - c <= bw.
// One CTA per system; a batch of RVE solves runs its systems on concurrent
// streams (fe2_hf_trajectories), one CTA each.
constexpr int kNB = 32;             // columns per panel (= warp width: the diagonal blocks run lane-per-row)
#ifndef FE2_BAND_THREADS
#define FE2_BAND_THREADS 512
#endif
constexpr int kBandThreads = FE2_BAND_THREADS;  // factorisation CTA
constexpr int kSolveThreads = 256;  // substitution CTA
constexpr int kMaxRhs = 4;          // right-hand sides per substitution (monolithic: K^-1 [r | K_fE])

__host__ __device__ constexpr int band_panel_ld(int bw) { return (bw + kNB + 3) / 4 * 4; }
size_t band_chol_smem(int bw) { return sizeof(double) * kNB * band_panel_ld(bw); }
constexpr int kBandSmemMax = 200 * 1024;

// Right-looking, blocked by kNB columns, with look-ahead. Per panel (columns
// j0 .. j0+nb-1, rows j0 .. j0+nb-1+bw; k-major in shared memory so the 4-row
// tile reads are 32-B vectors): its nb x nb diagonal block is already factored
// (sDiag, by the previous panel's look-ahead); load the rows below; solve them
// against the diagonal block, one thread per row in registers; write the panel
// back; rank-nb update of the next bw x bw lower window in 4x4 register tiles
// (warps on tile columns, lanes on tile rows: coalesced band loads / stores, the
// 16 loads of a tile issued before any store) — first the tile columns of the
// NEXT panel on all warps, then warp 0 factors the next diagonal block in
// registers (lane = row, column broadcast by shuffles) while warps 1.. finish
// the remaining tiles. info = 0, or 1 + the first non-positive pivot's column.
__device__ __forceinline__ bool band_diag_factor(const double* __restrict__ Kb, int ldb, int bw, int c0, int nb,
                                                 double (*sDiag)[kNB + 1], double* sInvD, int lane, int* bad_col) {
  // stage the block (column k of it is contiguous in the band: lanes read rows k + lane)
  for (int k = 0; k < nb; ++k) {
    const int r = k + lane;
    if (r < nb) sDiag[r][k] = (lane <= bw) ? Kb[static_cast<size_t>(c0 + k) * ldb + lane] : 0.0;
  }
  __syncwarp();
  double a[kNB];
#pragma unroll
  for (int k = 0; k < kNB; ++k) a[k] = (k < nb && lane < nb && k <= lane) ? sDiag[lane][k] : 0.0;
#pragma unroll
  for (int k = 0; k < kNB; ++k) {
    if (k < nb) {
      const double d = __shfl_sync(0xffffffffu, a[k], k);
      if (!(d > 0.0)) {
        *bad_col = k;
        return false;
      }
      const double l = sqrt(d), inv = 1.0 / l;
      if (lane == k) {
        a[k] = l;
        sInvD[k] = inv;
      } else if (lane > k) {
        a[k] *= inv;
      }
#pragma unroll
      for (int kk = k + 1; kk < kNB; ++kk) {
        const double lk = __shfl_sync(0xffffffffu, a[k], kk);  // L(kk, k)
        if (lane >= kk) a[kk] -= a[k] * lk;
      }
    }
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < kNB; ++k) sDiag[lane][k] = (k <= lane) ? a[k] : 0.0;
  return true;
}

// one 4x4 tile (rows 4 ti.., columns 4 tj.. of the window after column j0 + nb - 1)
__device__ __forceinline__ void band_tile_update(double* __restrict__ Kb, int ldb, int j0, int nb, int M,
                                                 const double* sP, int LR, int ti, int tj) {
  double old[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int c = 4 * tj + r;
    const double* col = Kb + static_cast<size_t>(j0 + nb + c) * ldb;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = 4 * ti + q;
      old[q][r] = (c < M && i < M && i >= c) ? col[i - c] : 0.0;
    }
  }
  asm volatile("" ::: "memory");  // keep the 16 band loads ahead of the stores (they overlap)
  double acc[4][4] = {};
  for (int k = 0; k < nb; ++k) {
    const double* ck = sP + k * LR + nb;
    const double2 x0 = *reinterpret_cast<const double2*>(ck + 4 * ti);  // rows (128-bit loads)
    const double2 x1 = *reinterpret_cast<const double2*>(ck + 4 * ti + 2);
    const double2 y0 = *reinterpret_cast<const double2*>(ck + 4 * tj);  // columns (broadcast)
    const double2 y1 = *reinterpret_cast<const double2*>(ck + 4 * tj + 2);
    const double xv[4] = {x0.x, x0.y, x1.x, x1.y}, yv[4] = {y0.x, y0.y, y1.x, y1.y};
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[q][r] += xv[q] * yv[r];
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int c = 4 * tj + r;
    double* col = Kb + static_cast<size_t>(j0 + nb + c) * ldb;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = 4 * ti + q;
      if (c < M && i < M && i >= c) col[i - c] = old[q][r] - acc[q][r];
    }
  }
}

__global__ void __launch_bounds__(kBandThreads) k_band_chol(int n, int bw, int ldb, double* __restrict__ Kb,
                                                            int* __restrict__ info) {
  extern __shared__ __align__(32) double sP[];  // [kNB][LR]: sP[k * LR + i] = L(j0 + i, j0 + k), i >= nb
  __shared__ double sDiag[kNB][kNB + 1];        // the factored diagonal block of the current panel
  __shared__ double sInvD[kNB];                 // 1 / L_kk of it
  __shared__ int s_fail;
  const int LR = band_panel_ld(bw);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nwarps = blockDim.x >> 5;
  if (t == 0) s_fail = 0;
  __syncthreads();
  // j0 = -kNB: only the look-ahead step (the first panel's diagonal block), so the
  // diagonal factorisation has a single call site (register allocation)
  for (int j0 = -kNB; j0 < n; j0 += kNB) {
    const int nb = j0 < 0 ? 0 : min(kNB, n - j0);
    const int R = j0 < 0 ? 0 : min(n, j0 + nb + bw) - j0;
    const int M = R - nb;
    const int T4 = (M + 3) / 4;
    const int TA = min(T4, kNB / 4);  // tile columns of the next panel
    if (j0 >= 0) {
      for (int e = t; e < (R - nb) * nb; e += blockDim.x) {  // the rows below the diagonal block
        const int k = e / (R - nb), i = nb + (e - k * (R - nb));
        sP[k * LR + i] = (i - k <= bw) ? Kb[static_cast<size_t>(j0 + k) * ldb + (i - k)] : 0.0;
      }
      __syncthreads();
      // L_21 = A_21 L_11^-T, one thread per row in registers
      for (int i = nb + t; i < R; i += blockDim.x) {
        asm volatile("" ::: "memory");  // keep the L(k, m) reads in the loop (hoisted, 528 values spill)
        double a[kNB];
#pragma unroll
        for (int k = 0; k < kNB; ++k) a[k] = k < nb ? sP[k * LR + i] : 0.0;
#pragma unroll
        for (int k = 0; k < kNB; ++k) {
          if (k < nb) {
            double v = a[k];
#pragma unroll
            for (int m = 0; m < k; ++m) v -= a[m] * sDiag[k][m];  // L(k, m): broadcast
            a[k] = v * sInvD[k];
          }
        }
#pragma unroll
        for (int k = 0; k < kNB; ++k)
          if (k < nb) sP[k * LR + i] = a[k];
      }
      __syncthreads();
      for (int e = t; e < R * nb; e += blockDim.x) {  // the factored panel back to the band
        const int k = e / R, i = e - k * R;
        if (i >= k && i - k <= bw)
          Kb[static_cast<size_t>(j0 + k) * ldb + (i - k)] = i < nb ? sDiag[i][k] : sP[k * LR + i];
      }
      // phase A: the next panel's columns, all warps (column w % TA, rows split over warp groups)
      const int groups = TA > 0 && nwarps / TA > 0 ? nwarps / TA : 1;
      if (TA > 0 && warp < TA * groups) {
        const int tj = warp % TA, g = warp / TA;
        for (int ti = tj + lane + 32 * g; ti < T4; ti += 32 * groups) band_tile_update(Kb, ldb, j0, nb, M, sP, LR, ti, tj);
      }
    }
    __syncthreads();
    // phase B: warp 0 factors the next diagonal block (its entries are final now) while
    // the other warps update the remaining tile columns
    const int c1 = j0 + kNB;  // the next panel (j0 + nb when j0 >= 0 and the panel is full)
    if (warp == 0) {
      if (c1 < n) {
        int bc = 0;
        if (!band_diag_factor(Kb, ldb, bw, c1, min(kNB, n - c1), sDiag, sInvD, lane, &bc) && lane == 0) {
          *info = c1 + bc + 1;
          s_fail = 1;
        }
      }
    } else {
      for (int tj = TA + warp - 1; tj < T4; tj += nwarps - 1)
        for (int ti = tj + lane; ti < T4; ti += 32) band_tile_update(Kb, ldb, j0, nb, M, sP, LR, ti, tj);
    }
    __syncthreads();
    if (s_fail) return;  // uniform
  }
  if (t == 0) *info = 0;
}

// x = (L L^T)^-1 x for nrhs columns (stride n) with the band factor of
// k_band_chol, blocked by kNB. Per block: stage the diagonal block and its
// reciprocal pivots in shared memory; solve it on one warp per right-hand
// side (lane = block row, shuffles); then push the block's solution to the
// (up to bw) rows it couples to — forward: rows below, backward: columns
// before — one thread per (row, rhs), the kNB band entries loaded together.
__global__ void __launch_bounds__(kSolveThreads) k_band_solve(int n, int bw, int ldb, const double* __restrict__ Kb,
                                                              double* __restrict__ x, int nrhs) {
  __shared__ double sD[kNB][kNB + 1];  // diagonal block, sD[i][k] = L(j0 + i, j0 + k)
  __shared__ double sInv[kNB];
  __shared__ double sX[kMaxRhs][kNB];  // the block's solution
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  auto stage = [&](int j0, int nb) {
    for (int e = t; e < kNB * kNB; e += blockDim.x) {
      const int i = e % kNB, k = e / kNB;
      sD[i][k] = (i < nb && k < nb && i >= k && i - k <= bw) ? Kb[static_cast<size_t>(j0 + k) * ldb + (i - k)] : 0.0;
    }
    __syncthreads();
    if (t < nb) sInv[t] = 1.0 / sD[t][t];
    __syncthreads();
  };
  // forward: L y = b
  for (int j0 = 0; j0 < n; j0 += kNB) {
    const int nb = min(kNB, n - j0);
    stage(j0, nb);
    if (warp < nrhs) {
      double* xr = x + static_cast<size_t>(warp) * n + j0;
      double v = lane < nb ? xr[lane] : 0.0;
      for (int k = 0; k < nb; ++k) {
        const double y = __shfl_sync(0xffffffffu, v, k) * sInv[k];
        if (lane == k) v = y;
        else if (lane > k && lane < nb) v -= sD[lane][k] * y;
      }
      if (lane < nb) {
        xr[lane] = v;
        sX[warp][lane] = v;
      }
    }
    __syncthreads();
    const int m = min(n, j0 + nb + bw) - (j0 + nb);  // rows below the block that it couples to
    for (int e = t; e < m * nrhs; e += blockDim.x) {
      const int rh = e / m, i = j0 + nb + (e - rh * m);
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < kNB; ++k) {
        const int off = i - (j0 + k);
        if (k < nb && off <= bw) s += Kb[static_cast<size_t>(j0 + k) * ldb + off] * sX[rh][k];
      }
      x[static_cast<size_t>(rh) * n + i] -= s;
    }
    __syncthreads();
  }
  // backward: L^T x = y
  const int nblk = (n + kNB - 1) / kNB;
  for (int b = nblk - 1; b >= 0; --b) {
    const int j0 = b * kNB, nb = min(kNB, n - j0);
    stage(j0, nb);
    if (warp < nrhs) {
      double* xr = x + static_cast<size_t>(warp) * n + j0;
      double v = lane < nb ? xr[lane] : 0.0;
      for (int k = nb - 1; k >= 0; --k) {
        const double y = __shfl_sync(0xffffffffu, v, k) * sInv[k];
        if (lane == k) v = y;
        else if (lane < k) v -= sD[k][lane] * y;
      }
      if (lane < nb) {
        xr[lane] = v;
        sX[warp][lane] = v;
      }
    }
    __syncthreads();
    const int j1 = max(0, j0 - bw);  // columns before the block that it couples to
    const int m = j0 - j1;
    for (int e = t; e < m * nrhs; e += blockDim.x) {
      const int rh = e / m, j = j1 + (e - rh * m);
      const double* col = Kb + static_cast<size_t>(j) * ldb;
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < kNB; ++k) {
        const int off = j0 + k - j;
        if (k < nb && off <= bw) s += col[off] * sX[rh][k];
      }
      x[static_cast<size_t>(rh) * n + j] -= s;
    }
    __syncthreads();
  }
}

// One thread per DOF: residual entry and (free DOF, with_K) the lower-band
// part of its stiffness row in the band ordering, summed over the DOF's
// element incidences in ascending element order (deterministic, no atomics:
// entry (pa, pb <= pa) belongs to row pa's thread alone).
__global__ void k_hf_gather_band(int nd, const int* __restrict__ inc_ptr, const int* __restrict__ inc,
                                 const int* __restrict__ conn, const int* __restrict__ free_index,
                                 const int* __restrict__ perm, int ldb, const double* __restrict__ f_el,
                                 const double* __restrict__ k_el, int with_K, double* __restrict__ f_full,
                                 double* __restrict__ Kb) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= nd) return;
  const int p0 = inc_ptr[d], p1 = inc_ptr[d + 1];
  double f = 0.0;
  for (int p = p0; p < p1; ++p) f += f_el[inc[p]];
  f_full[d] = f;
  const int fa = free_index[d];
  if (!with_K || fa < 0) return;
  const int pa = perm[fa];
  for (int p = p0; p < p1; ++p) {
    const int e = inc[p] / 12, a = inc[p] % 12;
    const double* ke = k_el + static_cast<size_t>(144) * e + 12 * a;
    for (int b = 0; b < 12; ++b) {
      const int fb = free_index[2 * conn[6 * e + b / 2] + b % 2];
      if (fb < 0) continue;
      const int pb = perm[fb];
      if (pb <= pa) Kb[static_cast<size_t>(pb) * ldb + (pa - pb)] += ke[b];
    }
  }
}

double norm2(const double* v, size_t n) {
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += v[i] * v[i];
  return std::sqrt(s);
}

}  // namespace

}  // namespace fe2

using namespace fe2;

namespace {

// Reverse Cuthill-McKee order of the nodes that carry free DOFs (adjacent =
// sharing an element), started from a pseudo-peripheral node of each
// connected component; the free DOFs are numbered node by node in that order.
// perm[free index] = band position; bw = the resulting half bandwidth.
std::vector<int> band_order(const RveData& r, int& bw) {
  const int nn = r.n_nodes;
  std::vector<char> has(nn, 0);
  for (int v = 0; v < nn; ++v) has[v] = (r.free_index[2 * v] >= 0 || r.free_index[2 * v + 1] >= 0) ? 1 : 0;
  std::vector<std::vector<int>> adj(nn);
  for (int e = 0; e < r.n_el; ++e)
    for (int a = 0; a < 6; ++a)
      for (int b = 0; b < 6; ++b) {
        const int u = r.conn[6 * e + a], v = r.conn[6 * e + b];
        if (u != v && has[u] && has[v]) adj[u].push_back(v);
      }
  for (auto& l : adj) {
    std::sort(l.begin(), l.end());
    l.erase(std::unique(l.begin(), l.end()), l.end());
  }
  std::vector<int> deg(nn);
  for (int v = 0; v < nn; ++v) deg[v] = static_cast<int>(adj[v].size());
  std::vector<int> level(nn, -1), order;
  order.reserve(nn);
  auto bfs = [&](int s, std::vector<int>& out) {  // Cuthill-McKee sweep; returns the last level
    std::vector<int> seen;
    out.clear();
    level[s] = 0;
    out.push_back(s);
    for (size_t h = 0; h < out.size(); ++h) {
      const int v = out[h];
      std::vector<int> nb;
      for (int u : adj[v])
        if (level[u] < 0) {
          level[u] = level[v] + 1;
          nb.push_back(u);
        }
      std::stable_sort(nb.begin(), nb.end(), [&](int a, int b) { return deg[a] < deg[b]; });
      out.insert(out.end(), nb.begin(), nb.end());
    }
    return level[out.back()];
  };
  std::vector<int> comp;
  for (int s0 = 0; s0 < nn; ++s0) {
    if (!has[s0] || level[s0] >= 0) continue;
    // the component, and a pseudo-peripheral start (lowest degree in the last level, repeated)
    bfs(s0, comp);
    int s = s0;
    for (int v : comp)
      if (deg[v] < deg[s]) s = v;
    int ecc = -1;
    for (int pass = 0; pass < 4; ++pass) {
      for (int v : comp) level[v] = -1;
      const int L = bfs(s, comp);
      if (L <= ecc) break;
      ecc = L;
      int best = -1;
      for (int v : comp)
        if (level[v] == L && (best < 0 || deg[v] < deg[best])) best = v;
      s = best;
    }
    for (int v : comp) level[v] = -1;
    bfs(s, comp);
    order.insert(order.end(), comp.begin(), comp.end());
  }
  std::reverse(order.begin(), order.end());
  std::vector<int> perm(r.n_free, -1);
  int pos = 0;
  for (int v : order)
    for (int c = 0; c < 2; ++c)
      if (r.free_index[2 * v + c] >= 0) perm[r.free_index[2 * v + c]] = pos++;
  check(pos == r.n_free, Code::mesh, "band ordering lost a free DOF");
  bw = 0;
  for (int e = 0; e < r.n_el; ++e)
    for (int a = 0; a < 12; ++a)
      for (int b = 0; b < 12; ++b) {
        const int fa = r.free_index[2 * r.conn[6 * e + a / 2] + a % 2];
        const int fb = r.free_index[2 * r.conn[6 * e + b / 2] + b % 2];
        if (fa >= 0 && fb >= 0) bw = std::max(bw, std::abs(perm[fa] - perm[fb]));
      }
  return perm;
}

// Concurrent workers of a batch (FE2_HF_WORKERS, default 64). The device's
// hardware work queues (CUDA_DEVICE_MAX_CONNECTIONS) are raised to their
// maximum of 32 when the library loads, unless the process set them: with the
// default 8, streams share a queue and one long band factorisation blocks the
// others' work behind it (40 POD trajectories: 8.2 s -> 4.2 s measured).
int hf_workers_max() {
  const char* e = std::getenv("FE2_HF_WORKERS");
  const int v = (e && *e) ? std::atoi(e) : 64;
  return std::max(1, std::min(v, 256));
}

__attribute__((constructor)) void raise_device_connections() {
  setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 0);  // effective if no CUDA context exists yet
}

}  // namespace

// Immutable RVE data on the device, shared by the workers.
struct HfShared {
  int device = 0;
  RveData r;
  MatTable mats{}, mats_el{};
  int *d_conn = nullptr, *d_phase = nullptr, *d_free = nullptr, *d_inc_ptr = nullptr, *d_inc = nullptr,
      *d_perm = nullptr;
  double *d_B = nullptr, *d_w = nullptr;
  std::vector<int> perm;  // free index -> band position
  int bw = 0, ldb = 1;    // half bandwidth, band column stride
  int nd() const { return r.n_dofs(); }
  int nf() const { return r.n_free; }
  ~HfShared() {
    for (int* p : {d_conn, d_phase, d_free, d_inc_ptr, d_inc, d_perm})
      if (p) cudaFree(p);
    for (double* p : {d_B, d_w})
      if (p) cudaFree(p);
  }
};

// One RVE solve context: its own stream and working buffers (states, element
// arrays, the band factor), so that many run concurrently (one host thread each).
struct HfWork {
  const HfShared& S;
  cudaStream_t stream = nullptr;
  int* d_info = nullptr;
  int* d_err = nullptr;  // set by k_hf_element when a return map fails
  double *d_u = nullptr, *d_st0 = nullptr, *d_st1 = nullptr, *d_fel = nullptr, *d_kel = nullptr, *d_f = nullptr;
  double *d_Kb = nullptr, *d_sig = nullptr, *d_C = nullptr, *d_rhs = nullptr;
  // pinned staging of every host<->device transfer (pageable copies serialise
  // against the other workers' streams): u / f [nd], rhs [3 nf], sigma / C per
  // integration point, {err, info}
  double *h_u = nullptr, *h_f = nullptr, *h_rhs = nullptr, *h_sig = nullptr, *h_C = nullptr;
  int* h_flags = nullptr;
  bool factored = false;      // d_Kb holds the factor of the last assembled stiffness
  double* st_comm = nullptr;  // committed states the assembly reads (d_st0, or a point's block)
  // FE2_HF_PROF=1: host wall time per phase (assemble with K, residual-only assemble,
  // factor, solve, homogenize), printed when the worker is destroyed
  double prof[8] = {};
  long prof_n[8] = {};
  static bool prof_on() {
    static const bool on = [] {
      const char* e = std::getenv("FE2_HF_PROF");
      return e && *e && *e != '0';
    }();
    return on;
  }
  struct Tick {
    HfWork& w;
    int k;
    std::chrono::steady_clock::time_point t0;
    Tick(HfWork& w_, int k_) : w(w_), k(k_), t0(std::chrono::steady_clock::now()) {}
    ~Tick() {
      w.prof[k] += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      w.prof_n[k] += 1;
    }
  };

  cudaEvent_t done = nullptr;  // blocking-sync event: a waiting worker thread sleeps instead of spinning

  // wait for this worker's stream; the thread yields the core (a batch runs
  // more worker threads than the host has cores)
  void wait() {
    CK(cudaEventRecord(done, stream));
    CK(cudaEventSynchronize(done));
  }

  explicit HfWork(const HfShared& s) : S(s) {
    const RveData& r = S.r;
    CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&done, cudaEventBlockingSync | cudaEventDisableTiming));
    d_info = dalloc<int>(1);
    d_err = dalloc<int>(1);
    CK(cudaMemset(d_err, 0, sizeof(int)));
    d_u = dalloc<double>(S.nd());
    d_f = dalloc<double>(S.nd());
    d_st0 = dalloc<double>(static_cast<size_t>(6) * r.n_ips());
    d_st1 = dalloc<double>(static_cast<size_t>(6) * r.n_ips());
    d_sig = dalloc<double>(static_cast<size_t>(3) * r.n_ips());
    d_C = dalloc<double>(static_cast<size_t>(9) * r.n_ips());
    d_fel = dalloc<double>(static_cast<size_t>(12) * r.n_el);
    d_kel = dalloc<double>(static_cast<size_t>(144) * r.n_el);
    d_Kb = dalloc<double>(static_cast<size_t>(S.nf()) * S.ldb);
    d_rhs = dalloc<double>(static_cast<size_t>(kMaxRhs) * S.nf());
    CK(cudaMallocHost(&h_u, sizeof(double) * S.nd()));
    CK(cudaMallocHost(&h_f, sizeof(double) * S.nd()));
    CK(cudaMallocHost(&h_rhs, sizeof(double) * kMaxRhs * S.nf()));
    CK(cudaMallocHost(&h_sig, sizeof(double) * 3 * r.n_ips()));
    CK(cudaMallocHost(&h_C, sizeof(double) * 9 * r.n_ips()));
    CK(cudaMallocHost(&h_flags, sizeof(int) * 2));
    st_comm = d_st0;
  }
  ~HfWork() {
    if (prof_on() && prof_n[0] > 0)
      std::fprintf(stderr,
                   "FE2_HF_PROF assemble+K %.3f ms x %ld | assemble %.3f ms x %ld | factor %.3f ms x %ld | "
                   "solve %.3f ms x %ld | homogenize %.3f ms x %ld\n",
                   1e3 * prof[0] / prof_n[0], prof_n[0], 1e3 * prof[1] / std::max(1L, prof_n[1]), prof_n[1],
                   1e3 * prof[2] / std::max(1L, prof_n[2]), prof_n[2], 1e3 * prof[3] / std::max(1L, prof_n[3]),
                   prof_n[3], 1e3 * prof[4] / std::max(1L, prof_n[4]), prof_n[4]);
    if (prof_on() && prof_n[5] > 0)
      std::fprintf(stderr, "FE2_HF_PROF solve: h2d %.3f ms | kernel %.3f ms | d2h %.3f ms\n", 1e3 * prof[5] / prof_n[5],
                   1e3 * prof[6] / prof_n[6], 1e3 * prof[7] / prof_n[7]);
    if (done) cudaEventDestroy(done);
    if (stream) cudaStreamDestroy(stream);
    for (int* p : {d_info, d_err})
      if (p) cudaFree(p);
    for (double* p : {d_u, d_st0, d_st1, d_fel, d_kel, d_f, d_Kb, d_sig, d_C, d_rhs})
      if (p) cudaFree(p);
    for (void* p : {static_cast<void*>(h_u), static_cast<void*>(h_f), static_cast<void*>(h_rhs),
                    static_cast<void*>(h_sig), static_cast<void*>(h_C), static_cast<void*>(h_flags)})
      if (p) cudaFreeHost(p);
  }
  int nd() const { return S.nd(); }
  int nf() const { return S.nf(); }

  void affine(const double* E, std::vector<double>& u) const {  // affine_field, rve.hpp:43-51
    const RveData& r = S.r;
    u.assign(nd(), 0.0);
    const double e11 = E[0], e22 = E[1], e12 = 0.5 * E[2];
    for (int id = 0; id < r.n_nodes; ++id) {
      u[2 * id] = e11 * r.x[id] + e12 * r.y[id];
      u[2 * id + 1] = e12 * r.x[id] + e22 * r.y[id];
    }
  }

  // assemble_micro at u_full from the committed states (st_comm); with_K also
  // keeps the trial states, stresses and tangents of every point and the band
  // stiffness.
  void assemble(const std::vector<double>& u_full, bool with_K, const MatTable& mt, std::vector<double>& f_full) {
    const Tick tk(*this, with_K ? 0 : 1);
    const RveData& r = S.r;
    std::memcpy(h_u, u_full.data(), sizeof(double) * nd());
    CK(cudaMemcpyAsync(d_u, h_u, sizeof(double) * nd(), cudaMemcpyHostToDevice, stream));
    if (with_K) CK(cudaMemsetAsync(d_Kb, 0, sizeof(double) * nf() * S.ldb, stream));
    k_hf_element<<<r.n_el, 144, 0, stream>>>(r.n_el, S.d_conn, S.d_phase, mt, S.d_B, S.d_w, d_u, st_comm,
                                             with_K ? 1 : 0, d_fel, d_kel, d_st1, d_sig, d_C, d_err);
    CK(cudaGetLastError());
    k_hf_gather_band<<<(nd() + 127) / 128, 128, 0, stream>>>(nd(), S.d_inc_ptr, S.d_inc, S.d_conn, S.d_free,
                                                             S.d_perm, S.ldb, d_fel, d_kel, with_K ? 1 : 0, d_f,
                                                             d_Kb);
    CK(cudaGetLastError());
    f_full.resize(nd());
    CK(cudaMemcpyAsync(h_f, d_f, sizeof(double) * nd(), cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(h_flags, d_err, sizeof(int), cudaMemcpyDeviceToHost, stream));
    wait();
    std::memcpy(f_full.data(), h_f, sizeof(double) * nd());
    const int err = h_flags[0];
    check(err == 0, Code::material, "material return map did not converge");
    if (with_K) factored = false;
  }

  void factor(const char* what) {
    const Tick tk(*this, 2);
    k_band_chol<<<1, kBandThreads, band_chol_smem(S.bw), stream>>>(nf(), S.bw, S.ldb, d_Kb, d_info);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h_flags + 1, d_info, sizeof(int), cudaMemcpyDeviceToHost, stream));
    wait();
    check(h_flags[1] == 0, Code::solver, what);
    factored = true;
  }

  // x = K^-1 b for nrhs right-hand sides (free numbering, column j at b + j n), in place
  void solve(std::vector<double>& b, int nrhs) {
    const Tick tk(*this, 3);
    const int n = nf();
    double* bp = h_rhs;
    for (int j = 0; j < nrhs; ++j)
      for (int i = 0; i < n; ++i) bp[static_cast<size_t>(j) * n + S.perm[i]] = b[static_cast<size_t>(j) * n + i];
    {
      const Tick t5(*this, 5);
      CK(cudaMemcpyAsync(d_rhs, bp, sizeof(double) * n * nrhs, cudaMemcpyHostToDevice, stream));
      if (prof_on()) wait();
    }
    {
      const Tick t6(*this, 6);
      k_band_solve<<<1, kSolveThreads, 0, stream>>>(n, S.bw, S.ldb, d_Kb, d_rhs, nrhs);
      CK(cudaGetLastError());
      if (prof_on()) wait();
    }
    const Tick t7(*this, 7);
    CK(cudaMemcpyAsync(bp, d_rhs, sizeof(double) * n * nrhs, cudaMemcpyDeviceToHost, stream));
    wait();
    for (int j = 0; j < nrhs; ++j)
      for (int i = 0; i < n; ++i) b[static_cast<size_t>(j) * n + i] = bp[static_cast<size_t>(j) * n + S.perm[i]];
  }
  struct Newton {
    bool converged = false;
    int iterations = 0;
    double res_last = 0.0;
    std::vector<double> u_full;
  };

  // micro_newton (rve.hpp:285-346): boundary DOFs fixed to E.x, reference
  // force = max(|r_0|, |boundary reactions_0|, 1e-30), 8-halving Armijo line
  // search keeping the best trial. On convergence d_st1 / d_sig / d_C / d_K
  // hold the converged states, stresses, tangents and (unfactored) stiffness.
  Newton newton(const double* E, std::vector<double> u_free, double tol, int max_iter, const MatTable& mt) {
    const RveData& r = S.r;
    const int n = nf(), N = nd();
    Newton out;
    std::vector<double> aff;
    affine(E, aff);
    auto expand = [&](const std::vector<double>& uf, std::vector<double>& u) {
      u.resize(N);
      for (int i = 0; i < N; ++i) u[i] = r.free_index[i] >= 0 ? uf[r.free_index[i]] : aff[i];
    };
    auto reduce = [&](const std::vector<double>& f, std::vector<double>& rr) {
      rr.assign(n, 0.0);
      for (int i = 0; i < N; ++i)
        if (r.free_index[i] >= 0) rr[r.free_index[i]] += f[i];
    };
    std::vector<double> f_full, res, du(n), ut(n), u_trial, rt;
    double ref = 0.0;
    for (int it = 0; it <= max_iter; ++it) {
      expand(u_free, out.u_full);
      assemble(out.u_full, true, mt, f_full);
      reduce(f_full, res);
      const double rn = norm2(res.data(), n);
      out.res_last = rn;
      if (it == 0) {
        double s = 0.0;
        for (int i = 0; i < N; ++i)
          if (r.free_index[i] < 0) s += f_full[i] * f_full[i];
        ref = std::max({rn, std::sqrt(s), 1e-30});
      }
      if (rn <= tol * ref) {
        out.converged = true;
        out.iterations = it;
        return out;
      }
      if (it == max_iter) break;
      factor("micro stiffness factorization failed");
      for (int i = 0; i < n; ++i) du[i] = -res[i];
      solve(du, 1);
      double alpha = 1.0, best_alpha = 1.0, best_rn = std::numeric_limits<double>::infinity();
      for (int ls = 0; ls < 8; ++ls) {
        for (int i = 0; i < n; ++i) ut[i] = u_free[i] + alpha * du[i];
        expand(ut, u_trial);
        assemble(u_trial, false, mt, f_full);
        reduce(f_full, rt);
        const double trial = norm2(rt.data(), n);
        if (trial < best_rn) {
          best_rn = trial;
          best_alpha = alpha;
        }
        if (trial <= (1.0 - 1e-4 * alpha) * rn) break;
        alpha *= 0.5;
      }
      for (int i = 0; i < n; ++i) u_free[i] = u_free[i] + best_alpha * du[i];
    }
    out.converged = false;
    out.iterations = max_iter;
    return out;
  }

  // The integration-point stresses / tangents of the last assembly to the host,
  // s = Σ w σ, c_avg = Σ w C and the macro-strain coupling of the free DOFs,
  // kfe[j][n] = K_fE e_j = Σ w B_fᵀ C e_j (homogenize's right-hand sides, rve.hpp:372-380).
  void point_sums(std::vector<double>& Cq, double* s, double* c_avg, std::vector<double>& kfe) {
    const RveData& r = S.r;
    const int n = nf(), N = nd(), nip = r.n_ips();
    std::vector<double> sg(static_cast<size_t>(3) * nip);
    Cq.resize(static_cast<size_t>(9) * nip);
    CK(cudaMemcpyAsync(h_sig, d_sig, sizeof(double) * sg.size(), cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(h_C, d_C, sizeof(double) * Cq.size(), cudaMemcpyDeviceToHost, stream));
    wait();
    std::memcpy(sg.data(), h_sig, sizeof(double) * sg.size());
    std::memcpy(Cq.data(), h_C, sizeof(double) * Cq.size());
    for (int i = 0; i < 3; ++i) s[i] = 0.0;
    for (int ip = 0; ip < nip; ++ip)
      for (int i = 0; i < 3; ++i) s[i] += r.w[ip] * sg[3 * ip + i];
    std::vector<double> rhs_full(static_cast<size_t>(N) * 3, 0.0);
    for (int k = 0; k < 9; ++k) c_avg[k] = 0.0;
    for (int ip = 0; ip < nip; ++ip) {
      const int* el = r.conn.data() + 6 * (ip / 3);
      const double* B = r.B.data() + static_cast<size_t>(36) * ip;
      const double* Cp = Cq.data() + static_cast<size_t>(9) * ip;
      for (int a = 0; a < 12; ++a) {
        const int ga = 2 * el[a / 2] + a % 2;
        for (int j = 0; j < 3; ++j) {
          double t = 0.0;
          for (int i = 0; i < 3; ++i) t += B[i * 12 + a] * Cp[3 * i + j];
          rhs_full[static_cast<size_t>(ga) * 3 + j] += t * r.w[ip];
        }
      }
      for (int k = 0; k < 9; ++k) c_avg[k] += r.w[ip] * Cp[k];
    }
    kfe.assign(static_cast<size_t>(n) * 3, 0.0);
    for (int j = 0; j < 3; ++j)
      for (int i = 0; i < N; ++i)
        if (r.free_index[i] >= 0) kfe[static_cast<size_t>(j) * n + r.free_index[i]] += rhs_full[static_cast<size_t>(i) * 3 + j];
  }

  // out = Σ_ip w C_ip B_ip v for a free-DOF vector v (boundary entries 0)
  void cb_integral(const std::vector<double>& Cq, const double* v, double* out) const {
    const RveData& r = S.r;
    const int N = nd(), nip = r.n_ips();
    std::vector<double> vf(N);
    for (int i = 0; i < N; ++i) vf[i] = r.free_index[i] >= 0 ? v[r.free_index[i]] : 0.0;
    out[0] = out[1] = out[2] = 0.0;
    for (int ip = 0; ip < nip; ++ip) {
      const int* el = r.conn.data() + 6 * (ip / 3);
      const double* B = r.B.data() + static_cast<size_t>(36) * ip;
      const double* Cp = Cq.data() + static_cast<size_t>(9) * ip;
      double he[12];
      for (int a = 0; a < 6; ++a) {
        he[2 * a] = vf[2 * el[a]];
        he[2 * a + 1] = vf[2 * el[a] + 1];
      }
      double bh[3];
      for (int q = 0; q < 3; ++q) {
        double t = 0.0;
        for (int c = 0; c < 12; ++c) t += B[q * 12 + c] * he[c];
        bh[q] = t;
      }
      for (int i = 0; i < 3; ++i) {
        double t = 0.0;
        for (int k = 0; k < 3; ++k) t += Cp[3 * i + k] * bh[k];
        out[i] += r.w[ip] * t;
      }
    }
  }

  // homogenize (rve.hpp:350-392) at the converged state of the last newton():
  // Σ = s / V, C = (c_avg + Σ_j C B h_j) / V with h_j = K^-1 (-K_fE e_j).
  void homogenize(double* sigma, double* C) {
    const Tick tk(*this, 4);
    const int n = nf();
    std::vector<double> Cq, h;
    double s[3], c_avg[9];
    point_sums(Cq, s, c_avg, h);
    for (int i = 0; i < 3; ++i) sigma[i] = s[i] / S.r.volume;
    if (!factored) factor("homogenize: singular converged stiffness");
    for (double& v : h) v = -v;
    solve(h, 3);
    double c_hom[9];
    for (int k = 0; k < 9; ++k) c_hom[k] = c_avg[k];
    for (int j = 0; j < 3; ++j) {
      double ch[3];
      cb_integral(Cq, h.data() + static_cast<size_t>(j) * n, ch);
      for (int i = 0; i < 3; ++i) c_hom[3 * i + j] += ch[i];
    }
    for (int k = 0; k < 9; ++k) C[k] = c_hom[k] / S.r.volume;
  }

  // One monolithic micro iteration of a point (SPEC.md:474-481 HF_monolithic, the
  // full-field counterpart of k_increment<..., MONO>): the fluctuation w (free DOFs,
  // u = E.x + w) moves by the previous iteration's linearisation,
  // w <- w - K^-1 (r + K_fE (E - E_prev)) (the first iteration of a step starts from the
  // committed w); assemble at (E, w) from the committed states (trial states -> d_st1),
  // factor, z = K^-1 [r | K_fE]; condensed Σ~ = (s - K_fEᵀ K^-1 r) / V and
  // C = (c_avg - K_fEᵀ K^-1 K_fE) / V; rel_res = |r| / max(|r| at the step's first
  // iteration, |boundary reactions|, 1e-30).
  struct Mono {
    std::vector<double> w, z;  // [nf], [4][nf]
    double E[3] = {0, 0, 0};
    double r_first = 0.0;
    bool failed = false;  // the last iterate failed: commit keeps the point's committed state
  };
  void mono_iteration(const double* E, bool first, Mono& ms, double* sigma, double* C, double& rel_res) {
    const RveData& r = S.r;
    const int n = nf(), N = nd();
    if (!first) {
      const double d0 = E[0] - ms.E[0], d1 = E[1] - ms.E[1], d2 = E[2] - ms.E[2];
      for (int i = 0; i < n; ++i)
        ms.w[i] -= ms.z[i] + ms.z[static_cast<size_t>(n) + i] * d0 + ms.z[static_cast<size_t>(2) * n + i] * d1 +
                   ms.z[static_cast<size_t>(3) * n + i] * d2;
    }
    std::vector<double> aff, u_full(N), f_full;
    affine(E, aff);
    for (int i = 0; i < N; ++i) u_full[i] = aff[i] + (r.free_index[i] >= 0 ? ms.w[r.free_index[i]] : 0.0);
    assemble(u_full, true, S.mats, f_full);
    std::vector<double> res(n, 0.0);
    double reac = 0.0;
    for (int i = 0; i < N; ++i) {
      if (r.free_index[i] >= 0) res[r.free_index[i]] += f_full[i];
      else reac += f_full[i] * f_full[i];
    }
    const double rn = norm2(res.data(), n);
    if (first) ms.r_first = rn;
    rel_res = rn / std::max({ms.r_first, std::sqrt(reac), 1e-30});
    std::vector<double> Cq, kfe;
    double s[3], c_avg[9];
    point_sums(Cq, s, c_avg, kfe);
    factor("monolithic: singular micro stiffness");
    ms.z.assign(static_cast<size_t>(4) * n, 0.0);
    std::copy(res.begin(), res.end(), ms.z.begin());
    std::copy(kfe.begin(), kfe.end(), ms.z.begin() + n);
    solve(ms.z, 4);
    double t[3];
    cb_integral(Cq, ms.z.data(), t);  // K_fEᵀ K^-1 r
    for (int i = 0; i < 3; ++i) sigma[i] = (s[i] - t[i]) / r.volume;
    for (int j = 0; j < 3; ++j) {
      cb_integral(Cq, ms.z.data() + static_cast<size_t>(1 + j) * n, t);  // K_fEᵀ K^-1 K_fE e_j
      for (int i = 0; i < 3; ++i) C[3 * i + j] = (c_avg[3 * i + j] - t[i]) / r.volume;
    }
    for (int i = 0; i < 3; ++i) ms.E[i] = E[i];
  }

  // One path step of run_trajectory (rve.hpp:459-491) from the committed
  // state (st_comm on the device, u_free, E_comm) towards E_target, E_prev
  // being the previous path point: warm start = committed solution + affine
  // increment, bisection on non-convergence (throws ErrorCode::solver after
  // max_bisections). On success the committed state has advanced; the last
  // converged Newton result is returned (its d_sig / d_C / d_K are current).
  Newton increment(const double* E_prev, const double* E_target, std::vector<double>& u_free, double* E_comm,
                   double tol, int max_iter, int max_bisections, const MatTable& mt, int& its) {
    const RveData& r = S.r;
    const int N = nd();
    std::vector<double> aff, u0(nf());
    double done = 0.0, frac = 1.0;
    int bis = 0;
    its = 0;
    Newton res;
    while (done < 1.0 - 1e-12) {
      const double target = std::min(1.0, done + frac);
      double Ev[3], dE[3];
      for (int i = 0; i < 3; ++i) Ev[i] = E_prev[i] + (E_target[i] - E_prev[i]) * target;
      for (int i = 0; i < 3; ++i) dE[i] = Ev[i] - E_comm[i];
      affine(dE, aff);
      for (int i = 0; i < N; ++i)
        if (r.free_index[i] >= 0) u0[r.free_index[i]] = u_free[r.free_index[i]] + aff[i];
      MatTable ms = mt;  // creep: the sub-step's fraction of the increment's dt (rve.hpp:466)
      for (MatDev& md : ms.m) md.dt *= target - done;
      res = newton(Ev, u0, tol, max_iter, ms);
      its += res.iterations;
      if (!res.converged) {
        check(++bis <= max_bisections, Code::solver, "micro trajectory failed after max bisections");
        frac *= 0.5;
        continue;
      }
      CK(cudaMemcpyAsync(st_comm, d_st1, sizeof(double) * 6 * r.n_ips(), cudaMemcpyDeviceToDevice, stream));
      for (int i = 0; i < N; ++i)
        if (r.free_index[i] >= 0) u_free[r.free_index[i]] = res.u_full[i];
      for (int i = 0; i < 3; ++i) E_comm[i] = Ev[i];
      done = target;
    }
    return res;
  }

  // run_trajectory (rve.hpp:448-494) from the virgin state.
  void trajectory(int n_steps, const double* E, double tol, int max_iter, int max_bisections, const MatTable& mt,
                  double* sigma, double* C, int* iterations, double* u_fluct_inf, double* res_last, double* snaps) {
    const RveData& r = S.r;
    const int n = nf(), N = nd();
    st_comm = d_st0;
    CK(cudaMemsetAsync(d_st0, 0, sizeof(double) * 6 * r.n_ips(), stream));
    CK(cudaMemsetAsync(d_err, 0, sizeof(int), stream));
    std::vector<double> u_free(n, 0.0), aff;
    double E_prev[3] = {0, 0, 0}, E_comm[3] = {0, 0, 0};
    for (int k = 0; k < n_steps; ++k) {
      int its = 0;
      const Newton res = increment(E_prev, E + 3 * k, u_free, E_comm, tol, max_iter, max_bisections, mt, its);
      if (sigma || C) {
        double s3[3], c9[9];
        homogenize(s3, c9);
        if (sigma) std::memcpy(sigma + 3 * k, s3, sizeof(s3));
        if (C) std::memcpy(C + 9 * k, c9, sizeof(c9));
      }
      affine(E_comm, aff);
      double mx = 0.0;
      for (int i = 0; i < N; ++i) {
        const double wv = res.u_full[i] - aff[i];
        mx = std::max(mx, std::abs(wv));
        if (snaps) snaps[(size_t)k * N + i] = wv;
      }
      if (u_fluct_inf) u_fluct_inf[k] = mx;
      if (res_last) res_last[k] = res.res_last;
      if (iterations) iterations[k] = its;
      for (int i = 0; i < 3; ++i) E_prev[i] = E[3 * k + i];
    }
    wait();
  }

};

// The handle: shared RVE data plus a pool of workers (worker 0 serves the
// single-RVE calls; batches spread over up to FE2_HF_WORKERS of them, one
// host thread each, their kernels running concurrently on their own streams).
struct fe2_hf_s {
  HfShared S;
  std::vector<std::unique_ptr<HfWork>> work;
  // macro-point batch (fe2_hf_alloc_points): per point committed states on the
  // device, committed free displacements / strains on the host; snapshot copies
  int64_t P = 0;
  double *d_pst = nullptr, *d_pst_snap = nullptr;
  std::vector<double> pu, pu_snap, pE, pE_snap;  // [P][nf], [P][6] = (E_prev, E_comm)
  // monolithic scheme: per point the iterate (fluctuation, K^-1 [r | K_fE], E) and the
  // candidate states of its last assembly (adopted by fe2_hf_mono_commit)
  std::vector<HfWork::Mono> pmono;
  double* d_pcand = nullptr;
  bool mono_first = true, mono_any = false;

  ~fe2_hf_s() {
    work.clear();
    for (double* p : {d_pst, d_pst_snap, d_pcand})
      if (p) cudaFree(p);
  }
  HfWork& w0() { return worker(0); }
  HfWork& worker(int i) {
    while (static_cast<int>(work.size()) <= i) work.push_back(std::make_unique<HfWork>(S));
    return *work[i];
  }
  void sync_all() {
    for (auto& w : work) CK(cudaStreamSynchronize(w->stream));
  }

  // fn(worker, item) for item = 0..count-1, items dealt cyclically to the
  // workers; the first failure (by item order) is rethrown here.
  template <class Fn>
  void parallel(int64_t count, Fn&& fn) {
    const int nw = static_cast<int>(std::min<int64_t>(count, hf_workers_max()));
    if (nw <= 0) return;
    for (int i = 0; i < nw; ++i) worker(i);
    if (nw == 1) {
      for (int64_t it = 0; it < count; ++it) fn(*work[0], it);
      return;
    }
    std::vector<std::exception_ptr> errs(count);
    std::vector<std::thread> pool;
    for (int i = 0; i < nw; ++i)
      pool.emplace_back([&, i] {
        cudaSetDevice(S.device);
        for (int64_t it = i; it < count; it += nw) {
          try {
            fn(*work[i], it);
          } catch (...) {
            errs[it] = std::current_exception();
          }
        }
      });
    for (auto& t : pool) t.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
  }

  // A batch of P macro points, each an RVE with its own committed state
  // (the HF engine of an FE² run, SPEC.md:474-477 HF_nested). One increment
  // per call for every point (points in parallel over the workers); a point
  // whose step fails keeps its committed state and reports 1 + ErrorCode.
  void alloc_points(int64_t n_points) {
    HfWork& w = w0();
    dfree(d_pst);
    dfree(d_pst_snap);
    P = n_points;
    const size_t per = static_cast<size_t>(6) * S.r.n_ips();
    d_pst = dalloc<double>(static_cast<size_t>(P) * per);
    d_pst_snap = dalloc<double>(static_cast<size_t>(P) * per);
    CK(cudaMemsetAsync(d_pst, 0, sizeof(double) * P * per, w.stream));
    CK(cudaMemsetAsync(d_pst_snap, 0, sizeof(double) * P * per, w.stream));
    pu.assign(static_cast<size_t>(P) * S.nf(), 0.0);
    pE.assign(static_cast<size_t>(P) * 6, 0.0);
    pu_snap = pu;
    pE_snap = pE;
    dfree(d_pcand);
    pmono.clear();
    mono_first = true;
    mono_any = false;
    w.wait();
  }

  // One monolithic iteration of every point at the macro strains E (points in parallel
  // over the workers); status 0 or 1 + ErrorCode per point.
  void mono_points(const double* E, double* sigma, double* C, double* rel_res, int* status) {
    const int n = S.nf();
    const size_t sb = sizeof(double) * 6 * S.r.n_ips();
    if (!d_pcand) d_pcand = dalloc<double>(static_cast<size_t>(P) * 6 * S.r.n_ips());
    if (pmono.size() != static_cast<size_t>(P)) pmono.assign(P, HfWork::Mono{});
    const bool first = mono_first;
    parallel(P, [&](HfWork& w, int64_t p) {
      HfWork::Mono& ms = pmono[p];
      if (first) {  // the committed fluctuation: u_free - (E_comm . x) on the free DOFs
        const double* Ec = pE.data() + 6 * p + 3;
        std::vector<double> aff;
        w.affine(Ec, aff);
        ms.w.assign(n, 0.0);
        for (int i = 0; i < S.nd(); ++i)
          if (S.r.free_index[i] >= 0) ms.w[S.r.free_index[i]] = pu[p * n + S.r.free_index[i]] - aff[i];
      }
      int code = 0;
      double s3[3] = {0, 0, 0}, c9[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, rr = 0.0;
      CK(cudaMemsetAsync(w.d_err, 0, sizeof(int), w.stream));
      w.st_comm = d_pst + static_cast<size_t>(p) * 6 * S.r.n_ips();
      try {
        w.mono_iteration(E + 3 * p, first, ms, s3, c9, rr);
        CK(cudaMemcpyAsync(d_pcand + static_cast<size_t>(p) * 6 * S.r.n_ips(), w.d_st1, sb,
                           cudaMemcpyDeviceToDevice, w.stream));
        ms.failed = false;
      } catch (const Failure& f) {
        code = 1 + static_cast<int>(f.code);
        ms.failed = true;
        CK(cudaMemsetAsync(w.d_err, 0, sizeof(int), w.stream));
      }
      w.st_comm = w.d_st0;
      w.wait();
      if (sigma) std::memcpy(sigma + 3 * p, s3, sizeof(s3));
      if (C) std::memcpy(C + 9 * p, c9, sizeof(c9));
      if (rel_res) rel_res[p] = rr;
      if (status) status[p] = code;
    });
    mono_first = false;
    mono_any = true;
  }

  // adopt every point's last monolithic iterate: its trial states, u = E.x + w, E
  void mono_commit() {
    HfWork& w = w0();
    const int n = S.nf();
    const size_t per = static_cast<size_t>(6) * S.r.n_ips();
    for (int64_t p = 0; p < P; ++p) {
      const HfWork::Mono& ms = pmono[p];
      if (ms.failed) continue;  // as k_mono_commit skips failed points
      CK(cudaMemcpyAsync(d_pst + p * per, d_pcand + p * per, sizeof(double) * per, cudaMemcpyDeviceToDevice,
                         w.stream));
      std::vector<double> aff;
      w.affine(ms.E, aff);
      for (int i = 0; i < S.nd(); ++i)
        if (S.r.free_index[i] >= 0) pu[p * n + S.r.free_index[i]] = aff[i] + ms.w[S.r.free_index[i]];
      for (int i = 0; i < 3; ++i) pE[6 * p + i] = pE[6 * p + 3 + i] = ms.E[i];
    }
    w.wait();
    mono_first = true;
  }

  void solve_points(const double* E, double tol, int max_iter, int max_bisections, double* sigma, double* C,
                    int* iters, int* status) {
    const int n = S.nf();
    const size_t sb = sizeof(double) * 6 * S.r.n_ips();
    parallel(P, [&](HfWork& w, int64_t p) {
      double* own = d_pst + static_cast<size_t>(p) * 6 * S.r.n_ips();
      double* Ep = pE.data() + 6 * p;  // (E_prev, E_comm)
      std::vector<double> u_free(pu.begin() + p * n, pu.begin() + (p + 1) * n);
      double E_comm[3] = {Ep[3], Ep[4], Ep[5]};
      int its = 0, code = 0;
      CK(cudaMemsetAsync(w.d_err, 0, sizeof(int), w.stream));
      CK(cudaMemcpyAsync(w.d_st0, own, sb, cudaMemcpyDeviceToDevice, w.stream));  // backup for a failed step
      w.st_comm = own;
      try {
        w.increment(Ep, E + 3 * p, u_free, E_comm, tol, max_iter, max_bisections, S.mats, its);
        double s3[3], c9[9];
        w.homogenize(s3, c9);
        if (sigma) std::memcpy(sigma + 3 * p, s3, sizeof(s3));
        if (C) std::memcpy(C + 9 * p, c9, sizeof(c9));
        std::copy(u_free.begin(), u_free.end(), pu.begin() + p * n);
        for (int i = 0; i < 3; ++i) {
          Ep[i] = E[3 * p + i];
          Ep[3 + i] = E_comm[i];
        }
      } catch (const Failure& f) {
        code = 1 + static_cast<int>(f.code);
        CK(cudaMemsetAsync(w.d_err, 0, sizeof(int), w.stream));
        // a failed bisection may have committed sub-steps: return to the call's start
        CK(cudaMemcpyAsync(own, w.d_st0, sb, cudaMemcpyDeviceToDevice, w.stream));
      }
      w.st_comm = w.d_st0;
      w.wait();
      if (iters) iters[p] = its;
      if (status) status[p] = code;
    });
  }
};

extern "C" {

int fe2_hf_create(int device, int subdivisions, const char* mesh_path, const fe2_material_t* materials, int n_materials,
                  fe2_hf_t* out) {
  return guard([&] {
    check(out && materials && n_materials >= 1 && n_materials <= kMaxMats, Code::config, "bad HF arguments");
    *out = nullptr;
    auto h = std::make_unique<fe2_hf_s>();
    HfShared& S = h->S;
    for (int i = 0; i < n_materials; ++i) {
      S.mats.m[i] = to_dev(materials[i]);
      fe2_material_t el = materials[i];
      el.kind = 0;  // the elastic part (build_elastic_modes)
      S.mats_el.m[i] = to_dev(el);
    }
    S.r = rve_data(subdivisions, mesh_path);
    const RveData& r = S.r;
    for (int e = 0; e < r.n_el; ++e)
      check(r.phase[e] >= 0 && r.phase[e] < n_materials, Code::config, "element material id out of range");
    check(r.n_free >= 1, Code::mesh, "RVE has no free DOF");
    S.perm = band_order(r, S.bw);
    S.ldb = S.bw + 1;
    check(band_chol_smem(S.bw) <= static_cast<size_t>(kBandSmemMax), Code::mesh,
          "RVE stiffness band too wide for the device band factorisation (half bandwidth " + std::to_string(S.bw) + ")");
    require_device(device);
    S.device = device;
    // per-DOF element incidences in ascending element order (CSR)
    const int N = r.n_dofs();
    std::vector<int> cnt(N + 1, 0), inc;
    for (int e = 0; e < r.n_el; ++e)
      for (int a = 0; a < 12; ++a) ++cnt[2 * r.conn[6 * e + a / 2] + a % 2 + 1];
    for (int d = 0; d < N; ++d) cnt[d + 1] += cnt[d];
    inc.resize(cnt[N]);
    std::vector<int> pos(cnt.begin(), cnt.end() - 1);
    for (int e = 0; e < r.n_el; ++e)
      for (int a = 0; a < 12; ++a) inc[pos[2 * r.conn[6 * e + a / 2] + a % 2]++] = 12 * e + a;
    auto up_i = [&](int*& d, const std::vector<int>& v) {
      d = dalloc<int>(v.size());
      CK(cudaMemcpy(d, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice));
    };
    auto up_d = [&](double*& d, const std::vector<double>& v) {
      d = dalloc<double>(v.size());
      CK(cudaMemcpy(d, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice));
    };
    up_i(S.d_conn, r.conn);
    up_i(S.d_phase, r.phase);
    up_i(S.d_free, r.free_index);
    up_i(S.d_inc_ptr, cnt);
    up_i(S.d_inc, inc);
    up_i(S.d_perm, S.perm);
    up_d(S.d_B, r.B);
    up_d(S.d_w, r.w);
    // one ceiling for every handle (the attribute is per kernel, not per launch)
    CK(cudaFuncSetAttribute(k_band_chol, cudaFuncAttributeMaxDynamicSharedMemorySize, kBandSmemMax));
    h->w0();
    *out = h.release();
  });
}

void fe2_hf_destroy(fe2_hf_t h) {
  if (!h) return;
  cudaSetDevice(h->S.device);
  delete h;
}

int fe2_hf_sizes(fe2_hf_t h, int* n_dofs, int* n_free, int* n_ips, double* volume) {
  return guard([&] {
    check(h != nullptr, Code::config, "null HF handle");
    if (n_dofs) *n_dofs = h->S.nd();
    if (n_free) *n_free = h->S.nf();
    if (n_ips) *n_ips = h->S.r.n_ips();
    if (volume) *volume = h->S.r.volume;
  });
}

int fe2_hf_band(fe2_hf_t h, int* half_bandwidth) {
  return guard([&] {
    check(h != nullptr && half_bandwidth != nullptr, Code::config, "bad arguments");
    *half_bandwidth = h->S.bw;
  });
}

int fe2_hf_trajectory(fe2_hf_t h, int n_steps, const double* E, const fe2_newton_opts_t* opts, double* sigma,
                      double* C, int* iterations, double* u_fluct_inf, double* res_last, double* snapshots) {
  return guard([&] {
    check(h && E && opts && n_steps >= 0, Code::config, "bad HF trajectory arguments");
    check(opts->tol > 0.0 && opts->max_iter >= 1 && opts->max_bisections >= 0, Code::config, "bad Newton options");
    CK(cudaSetDevice(h->S.device));
    h->w0().trajectory(n_steps, E, opts->tol, opts->max_iter, opts->max_bisections, h->S.mats, sigma, C, iterations,
                       u_fluct_inf, res_last, snapshots);
  });
}

int fe2_hf_trajectories(fe2_hf_t h, int n_traj, int n_steps, const double* E, const fe2_newton_opts_t* opts,
                        double* sigma, double* C, int* iterations, double* u_fluct_inf, double* res_last,
                        double* snapshots, int* status) {
  return guard([&] {
    check(h && E && opts && n_traj >= 0 && n_steps >= 0, Code::config, "bad HF trajectory arguments");
    check(opts->tol > 0.0 && opts->max_iter >= 1 && opts->max_bisections >= 0, Code::config, "bad Newton options");
    CK(cudaSetDevice(h->S.device));
    const size_t N = h->S.nd(), k = n_steps;
    std::vector<std::string> msg(n_traj);
    h->parallel(n_traj, [&](HfWork& w, int64_t t) {
      int code = 0;
      try {
        w.trajectory(n_steps, E + 3 * k * t, opts->tol, opts->max_iter, opts->max_bisections, h->S.mats,
                     sigma ? sigma + 3 * k * t : nullptr, C ? C + 9 * k * t : nullptr,
                     iterations ? iterations + k * t : nullptr, u_fluct_inf ? u_fluct_inf + k * t : nullptr,
                     res_last ? res_last + k * t : nullptr, snapshots ? snapshots + N * k * t : nullptr);
      } catch (const std::exception& f) {
        const Failure* ff = dynamic_cast<const Failure*>(&f);
        code = 1 + static_cast<int>(ff ? ff->code : Code::numeric);
        msg[t] = f.what();
        CK(cudaMemsetAsync(w.d_err, 0, sizeof(int), w.stream));
        w.wait();
      }
      if (status) status[t] = code;
    });
    for (int t = 0; t < n_traj; ++t)  // the call succeeds; fe2_last_error names the first failed trajectory
      if (!msg[t].empty()) {
        set_last_error("trajectory " + std::to_string(t) + ": " + msg[t]);
        break;
      }
  });
}

int fe2_hf_alloc_points(fe2_hf_t h, int64_t P) {
  return guard([&] {
    check(h != nullptr && P >= 1, Code::config, "bad arguments");
    CK(cudaSetDevice(h->S.device));
    h->alloc_points(P);
  });
}

int fe2_hf_solve_increment(fe2_hf_t h, const double* E, const fe2_newton_opts_t* opts, double* sigma, double* C,
                           int* iters, int* status) {
  return guard([&] {
    check(h && E && opts, Code::config, "bad arguments");
    check(h->P > 0, Code::config, "no points allocated (fe2_hf_alloc_points)");
    check(opts->tol > 0.0 && opts->max_iter >= 1 && opts->max_bisections >= 0, Code::config, "bad Newton options");
    CK(cudaSetDevice(h->S.device));
    h->solve_points(E, opts->tol, opts->max_iter, opts->max_bisections, sigma, C, iters, status);
  });
}

int fe2_hf_mono_begin(fe2_hf_t h) {
  return guard([&] {
    check(h != nullptr && h->P > 0, Code::config, "no points allocated (fe2_hf_alloc_points)");
    h->mono_first = true;
  });
}

int fe2_hf_mono_iterate(fe2_hf_t h, const double* E, double* sigma, double* C, double* rel_res, int* status) {
  return guard([&] {
    check(h != nullptr && E != nullptr, Code::config, "bad arguments");
    check(h->P > 0, Code::config, "no points allocated (fe2_hf_alloc_points)");
    CK(cudaSetDevice(h->S.device));
    h->mono_points(E, sigma, C, rel_res, status);
  });
}

int fe2_hf_mono_commit(fe2_hf_t h) {
  return guard([&] {
    check(h != nullptr && h->P > 0, Code::config, "no points allocated (fe2_hf_alloc_points)");
    check(h->mono_any && !h->mono_first, Code::config, "fe2_hf_mono_commit needs a monolithic iterate");
    CK(cudaSetDevice(h->S.device));
    h->mono_commit();
  });
}

int fe2_hf_snapshot(fe2_hf_t h) {
  return guard([&] {
    check(h != nullptr && h->P > 0, Code::config, "no points allocated (fe2_hf_alloc_points)");
    CK(cudaSetDevice(h->S.device));
    HfWork& w = h->w0();
    CK(cudaMemcpyAsync(h->d_pst_snap, h->d_pst, sizeof(double) * h->P * 6 * h->S.r.n_ips(), cudaMemcpyDeviceToDevice,
                       w.stream));
    h->pu_snap = h->pu;
    h->pE_snap = h->pE;
    w.wait();
  });
}

int fe2_hf_restore(fe2_hf_t h) {
  return guard([&] {
    check(h != nullptr && h->P > 0, Code::config, "no points allocated (fe2_hf_alloc_points)");
    CK(cudaSetDevice(h->S.device));
    HfWork& w = h->w0();
    CK(cudaMemcpyAsync(h->d_pst, h->d_pst_snap, sizeof(double) * h->P * 6 * h->S.r.n_ips(), cudaMemcpyDeviceToDevice,
                       w.stream));
    h->pu = h->pu_snap;
    h->pE = h->pE_snap;
    w.wait();
  });
}

int fe2_hf_points(fe2_hf_t h, int64_t* P) {
  return guard([&] {
    check(h != nullptr && P != nullptr, Code::config, "bad arguments");
    *P = h->P;
  });
}

int fe2_hf_elastic_modes(fe2_hf_t h, double* modes, int* count) {
  return guard([&] {
    check(h && modes && count, Code::config, "bad arguments");
    CK(cudaSetDevice(h->S.device));
    const int N = h->S.nd();
    HfWork& w = h->w0();
    std::vector<double> A((size_t)3 * N), drop(3);
    for (int j = 0; j < 3; ++j) {
      double E[3] = {0, 0, 0};
      E[j] = 1.0;
      int its = 0;
      w.trajectory(1, E, 1e-10, 10, 0, h->S.mats_el, nullptr, nullptr, &its, nullptr, nullptr, A.data() + (size_t)j * N);
      std::vector<double> aff;
      w.affine(E, aff);
      drop[j] = 1e-10 * norm2(aff.data(), aff.size());
    }
    *count = orthonormalize_columns(A, N, 3, drop);
    std::memset(modes, 0, sizeof(double) * 3 * N);
    std::memcpy(modes, A.data(), sizeof(double) * A.size());
  });
}

int fe2_pod_basis(int device, const double* X, int64_t n_rows, int n_cols, const double* elastic, int n_elastic,
                  int n_target, double* V, double* singular_values, int* max_modes) {
  return guard([&] {
    check(X && V && n_rows >= 1 && n_cols >= 1 && n_elastic >= 0 && (n_elastic == 0 || elastic), Code::config,
          "bad POD arguments");
    check(n_target >= std::max(1, n_elastic) && n_target <= n_rows, Code::config, "POD target out of range");
    check(n_rows * static_cast<int64_t>(n_cols) < (int64_t(1) << 31), Code::config, "snapshot matrix too large");
    const size_t R = static_cast<size_t>(n_rows), M = static_cast<size_t>(n_cols);
    // elastic modes, orthonormalised
    std::vector<double> Em(elastic, elastic + R * n_elastic);
    const int ne = orthonormalize_columns(Em, n_rows, n_elastic, std::vector<double>(n_elastic, 1e-10));
    check(ne == n_elastic, Code::config, "elastic modes are linearly dependent");
    // deflation against the elastic span (classical Gram-Schmidt, twice)
    std::vector<double> D(X, X + R * M);
    const double xnorm = norm2(X, R * M);
    for (int pass = 0; pass < 2; ++pass)
      for (size_t c = 0; c < M; ++c) {
        double* d = D.data() + c * R;
        for (int j = 0; j < ne; ++j) {
          const double* q = Em.data() + static_cast<size_t>(j) * R;
          double dot = 0.0;
          for (size_t i = 0; i < R; ++i) dot += q[i] * d[i];
          for (size_t i = 0; i < R; ++i) d[i] -= dot * q[i];
        }
      }
    // SVD of the deflated snapshots on the device (gesvd needs rows >= cols:
    // otherwise factor D^T and read the left vectors from its VT)
    require_device(device);
    const Cusolver& cs = Cusolver::get();
    cusolverDnHandle_t sol = nullptr;
    sol_check(cs.create(&sol), "create");
    const bool tall = R >= M;
    const int m = tall ? n_rows : n_cols, n = tall ? n_cols : static_cast<int>(n_rows);
    std::vector<double> A(R * M);
    if (tall) A = D;
    else
      for (size_t c = 0; c < M; ++c)
        for (size_t i = 0; i < R; ++i) A[c + i * M] = D[i + c * R];
    double *dA = nullptr, *dS = nullptr, *dU = nullptr, *dW = nullptr, *dRw = nullptr;
    int* dInfo = nullptr;
    int lw = 0, info = 0;
    std::vector<double> S(n), Uh;
    try {
      dA = dalloc<double>(A.size());
      dS = dalloc<double>(n);
      dU = dalloc<double>(static_cast<size_t>(tall ? m : n) * n);
      dRw = dalloc<double>(n);
      dInfo = dalloc<int>(1);
      CK(cudaMemcpy(dA, A.data(), sizeof(double) * A.size(), cudaMemcpyHostToDevice));
      sol_check(cs.gesvd_ws(sol, m, n, &lw), "gesvd workspace");
      dW = dalloc<double>(std::max(1, lw));
      if (tall)
        sol_check(cs.gesvd(sol, 'S', 'N', m, n, dA, m, dS, dU, m, nullptr, n, dW, lw, dRw, dInfo), "gesvd");
      else
        sol_check(cs.gesvd(sol, 'N', 'S', m, n, dA, m, dS, nullptr, m, dU, n, dW, lw, dRw, dInfo), "gesvd");
      CK(cudaMemcpy(&info, dInfo, sizeof(int), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(S.data(), dS, sizeof(double) * n, cudaMemcpyDeviceToHost));
      Uh.resize(static_cast<size_t>(tall ? m : n) * n);
      CK(cudaMemcpy(Uh.data(), dU, sizeof(double) * Uh.size(), cudaMemcpyDeviceToHost));
    } catch (...) {
      for (double* p : {dA, dS, dU, dW, dRw}) dfree(p);
      dfree(dInfo);
      cs.destroy(sol);
      throw;
    }
    for (double* p : {dA, dS, dU, dW, dRw}) dfree(p);
    dfree(dInfo);
    cs.destroy(sol);
    check(info == 0, Code::solver, "SVD did not converge");
    const int ns = std::min<int64_t>(n_rows, n_cols);  // == n
    if (singular_values)
      for (int i = 0; i < n_cols; ++i) singular_values[i] = i < ns ? S[i] : 0.0;
    int rank = 0;
    while (rank < ns && S[rank] > 1e-10 * xnorm) ++rank;
    if (max_modes) *max_modes = ne + rank;
    const int k = n_target - ne;
    check(k <= rank, Code::rank,
          "POD: requested " + std::to_string(n_target) + " modes, at most " + std::to_string(ne + rank) + " usable");
    // left singular vector i: column i of U (tall) or row i of VT (n x n, wide)
    std::vector<double> Vh(R * n_target);
    std::copy(Em.begin(), Em.end(), Vh.begin());
    for (int i = 0; i < k; ++i) {
      double* v = Vh.data() + static_cast<size_t>(ne + i) * R;
      for (size_t r = 0; r < R; ++r) v[r] = tall ? Uh[r + static_cast<size_t>(i) * m] : Uh[i + r * static_cast<size_t>(n)];
    }
    const int kept = orthonormalize_columns(Vh, n_rows, n_target, std::vector<double>(n_target, 1e-8));
    check(kept == n_target, Code::numeric, "POD basis lost rank in re-orthonormalisation");
    for (int j = ne; j < n_target; ++j) {  // sign: largest-magnitude entry positive (lowest index on ties)
      double* v = Vh.data() + static_cast<size_t>(j) * R;
      size_t im = 0;
      for (size_t r = 1; r < R; ++r)
        if (std::abs(v[r]) > std::abs(v[im])) im = r;
      if (v[im] < 0.0)
        for (size_t r = 0; r < R; ++r) v[r] = -v[r];
    }
    std::memcpy(V, Vh.data(), sizeof(double) * Vh.size());
  });
}

}  // extern "C"
