// otdr_kernels.cuh -- sm_100a kernels of the RDROT iteration.
//
// One DR iteration (solver.cpp:95-102 + :23-38) is three launches:
//   sweep   one pass over (C, X): X <- prox([((X - rho C) + phi_i) + psi_j]_+),
//           plus fixed-order row/column partial sums of the new X  (HBM-bound)
//   reduce  partial sums -> r = X1 - p, S = X^T 1, sum r, sum r^2, sum X
//           (the n+3 "exchange" vector NCCL all-reduces across row shards)
//   update  s = S - q, eta, shift, phi/psi/a/b/theta recurrence, r_primal and
//           the solve loop's stopping logic, all on device (no host round trip)
// plus, only on check iterations that need it, the duality certificate
// (duality.cpp:9-24) and the objective (problem.cpp:76-85).
//
// All arithmetic is fp64 in registers. With fp64 storage (EXACT) every
// element-wise operation uses the reference's association order with
// round-to-nearest intrinsics (no FMA contraction), so plan entries are
// bit-identical to the reference given identical inputs; only the order of the
// row/column sums differs (fixed, deterministic, not Eigen's).
#pragma once
#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace otdrk {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

enum RegKind { REG_NONE = 0, REG_QUAD = 1, REG_GL = 2 };
enum Termination { TERM_CONVERGED = 0, TERM_MAXITER = 1, TERM_STALLED = 2, TERM_NONFINITE = 3 };

// Per-solve parameters (device resident so captured graphs stay valid when
// rho / tolerances change).
struct Params {
  double rho;
  double quad_d;    // 1 + rho*alpha                regularizers.cpp:54
  double quad_inv;  // 1 / (1 + rho*alpha)          (fp32-storage fast path)
  double alpha;
  double lambda;
  double gl_thr;    // rho*lambda                   regularizers.cpp:86
  double tol_primal;
  double tol_gap;
  long long max_iter;
  long long check_every;
  int has_tol_gap;
  int record_trace;
  int deterministic;
  int fused;
  int solving;      // stopping logic active (solve) vs raw step()
  long long trace_cap;
};

// Device control block: the solver's scalar state and loop bookkeeping.
struct Ctl {
  double theta[2];  // double-buffered by k parity (readers vs the finalizer)
  double eta;
  double r_primal;
  double best;
  long long k;                 // SolverState::k
  long long k0;                // k at solve start
  long long last_improvement;  // solve-relative iteration
  int done;
  int termination;
  int want_cert;
  int fused_shifted;           // X buffer holds B = X - rho C (even/odd path)
  unsigned int cnt_reduce;
  unsigned int cnt_update;
  unsigned int cnt_cert;
  int supp_changed;
  unsigned long long supp_count;
  long long support_last_change;
  long long trace_len;
  unsigned long long t0_ns;
  double objective, gap, dual_value, dres;
  long long last_support;
  // Monotonic 64-bit arrival counters of the software grid barriers; each is
  // used by exactly one kernel with a fixed grid size, so between launches it
  // always holds a multiple of that grid size.
  unsigned long long bar_fin;  // cooperative finalize kernel
  unsigned long long bar_res;  // resident solve kernel
  unsigned long long bar_str;  // streaming solve kernel
  unsigned int tile_ctr;       // streaming kernel: tiles claimed this sweep
  unsigned int gl_ctr;         // pipelined group-lasso sweep: items claimed
  unsigned int gl_done;        //   CTAs finished (the last one resets both)
  unsigned int pad_;
  unsigned long long bar_gls;  // persistent group-lasso solve kernel
  unsigned long long bar_tst;  // TMA-producer streaming solve kernel
};

struct TraceRow {
  long long iter;
  double r_primal, gap, dual_residual;
  long long support;
  double elapsed_ms;
};

// ---------------------------------------------------------------- helpers
template <typename T> struct Vec;
template <> struct Vec<float> { using type = float4; static constexpr int N = 4; };
template <> struct Vec<double> { using type = double2; static constexpr int N = 2; };

__device__ __forceinline__ void unpack(const float4& v, double* o) {
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}
__device__ __forceinline__ void unpack(const double2& v, double* o) { o[0] = v.x; o[1] = v.y; }
__device__ __forceinline__ float4 pack4(const double* o) {
  return make_float4(__double2float_rn(o[0]), __double2float_rn(o[1]),
                     __double2float_rn(o[2]), __double2float_rn(o[3]));
}
__device__ __forceinline__ double2 pack2(const double* o) { return make_double2(o[0], o[1]); }
template <typename T> __device__ __forceinline__ typename Vec<T>::type pack(const double* o);
template <> __device__ __forceinline__ float4 pack<float>(const double* o) { return pack4(o); }
template <> __device__ __forceinline__ double2 pack<double>(const double* o) { return pack2(o); }

// Streaming loads: C is read-only for the whole launch (non-coherent path);
// X is read then overwritten by the same thread (coherent path).
template <typename V> __device__ __forceinline__ V ld_ro(const V* p) { return __ldg(p); }
template <typename V> __device__ __forceinline__ V ld_rw(const V* p) { return *p; }

// RN(x / d) for the quadratic prox X /= (1 + rho alpha) (regularizers.cpp:54):
// x finite >= 0, d = 1 + rho alpha >= 1, inv = RN(1 / d) (host). q0 = RN(x inv)
// is within one ulp of x / d, the residual x - q0 d is exact in one FMA, and one
// correction q0 + r inv rounds to the correctly rounded quotient (Markstein).
// Three fp64 ops instead of the __ddiv_rn sequence; bitwise equal to the
// reference's true division (tests/test_gpu_parity.py::test_first_step_bitwise).
__device__ __forceinline__ double div_rn_by(double x, double d, double inv) {
  const double q0 = __dmul_rn(x, inv);
  const double r = __fma_rn(-q0, d, x);
  return __fma_rn(r, inv, q0);
}

// max(v, 0) with std::max's NaN propagation (solver.cpp:99 cwiseMax).
__device__ __forceinline__ double clamp0(double v) { return v < 0.0 ? 0.0 : v; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Fixed-order block sum (butterfly within warps, then warp 0 sums in order).
// Result valid in thread 0. red must hold kWarps doubles.
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kWarps; ++i) t += red[i];
  return t;
}

// block_sum for NW warps (result valid in thread 0).
template <int NW>
__device__ __forceinline__ double block_sum_n(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < NW; ++i) t += red[i];
  return t;
}

// Reduce-scatter of 8 row partials across a warp: lane l ends with the full
// sum of row row8_of(l) (lanes with equal bits 2..4 share a row). 9 double
// shuffles per 8 rows instead of 5 per row; the summation tree is fixed.
__device__ __forceinline__ int row8_of(int lane) {
  return ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
}
__device__ __forceinline__ double reduce8_rows(const double (&rs)[8], int lane) {
  double a4[4];
  const bool hi16 = (lane & 16) != 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const double keep = hi16 ? rs[4 + t] : rs[t];
    const double send = hi16 ? rs[t] : rs[4 + t];
    a4[t] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  double a2[2];
  const bool hi8 = (lane & 8) != 0;
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const double keep = hi8 ? a4[2 + t] : a4[t];
    const double send = hi8 ? a4[t] : a4[2 + t];
    a2[t] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  const bool hi4 = (lane & 4) != 0;
  double a1 = (hi4 ? a2[1] : a2[0]) + __shfl_xor_sync(0xffffffffu, hi4 ? a2[0] : a2[1], 4);
  a1 += __shfl_xor_sync(0xffffffffu, a1, 2);
  a1 += __shfl_xor_sync(0xffffffffu, a1, 1);
  return a1;
}

// ---------------------------------------------------------------- sweep
// Row-major C, X with leading dimension ld (multiple of the vector width;
// padded columns hold X = 0 and psi = -inf so they stay exactly 0).
// CTA (blockIdx.x = stripe, blockIdx.y = row group) owns columns
// [stripe*TN, stripe*TN+TN) of rows [rg*rows_per_cta, ...). Lane l holds NV
// vectors at columns stripe*TN + v*32*VEC + l*VEC (coalesced 512 B per warp
// per vector slot). Row partials: warp butterfly -> rowpart[row][stripe].
// Column partials: registers over the CTA's rows, then a fixed-order
// cross-warp smem sum -> colpart[rg][col].
template <typename T>
struct SweepArgs {
  T* X;
  const T* C;
  const double* phi;
  const double* psi;
  double* rowpart;  // [m][stripes]
  double* colpart;  // [rowgroups][ld]
  const Params* prm;
  Ctl* ctl;
  long long m, ld;
  int rows_per_cta;
  int sums_only;    // make_state: only the sums of the current X
};

enum SweepMode { MODE_NORMAL = 0, MODE_EVEN = 1, MODE_ODD = 2, MODE_SUMS = 3 };

template <typename T, int REG, bool EXACT, bool TRACK, int NV, int U>
__global__ void __launch_bounds__(kThreads, 2) sweep_kernel(SweepArgs<T> a) {
  using V = typename Vec<T>::type;
  constexpr int VEC = Vec<T>::N;
  constexpr int TN = 32 * VEC * NV;
  const Ctl* ctl = a.ctl;
  if (ctl->done) return;
  const Params& prm = *a.prm;
  int mode = MODE_NORMAL;
  if (a.sums_only) mode = MODE_SUMS;
  else if (prm.fused) mode = ctl->fused_shifted ? MODE_ODD : MODE_EVEN;
  const double rho = prm.rho;
  const double qd = prm.quad_d, qinv = prm.quad_inv;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long stripe = blockIdx.x;
  const long long col0 = stripe * TN;
  const long long r_begin = (long long)blockIdx.y * a.rows_per_cta;
  long long r_end = r_begin + a.rows_per_cta;
  if (r_end > a.m) r_end = a.m;

  long long cols[NV];
  bool cok[NV];
  double psi_r[NV][VEC];
  double cacc[NV][VEC];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    cols[v] = col0 + v * 32 * VEC + lane * VEC;
    cok[v] = cols[v] < a.ld;
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      psi_r[v][e] = cok[v] ? a.psi[cols[v] + e] : 0.0;
      cacc[v][e] = 0.0;
    }
  }
  const bool need_c = (mode == MODE_NORMAL || mode == MODE_EVEN) || (TRACK && mode == MODE_ODD);
  unsigned long long supp = 0;
  int changed = 0;

  for (long long i0 = r_begin + warp; i0 < r_end; i0 += (long long)kWarps * U) {
    V xv[U][NV], cv[U][NV];
    double phv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = i0 + (long long)u * kWarps;
      if (i < r_end) {
        phv[u] = a.phi[i];
        const V* xrow = reinterpret_cast<const V*>(a.X + i * a.ld);
        const V* crow = reinterpret_cast<const V*>(a.C + i * a.ld);
#pragma unroll
        for (int v = 0; v < NV; ++v)
          if (cok[v]) {
            xv[u][v] = ld_rw(xrow + cols[v] / VEC);
            if (need_c) cv[u][v] = ld_ro(crow + cols[v] / VEC);
          }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = i0 + (long long)u * kWarps;
      if (i >= r_end) break;  // warp-uniform
      double rs = 0.0;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        if (!cok[v]) continue;
        double x[VEC], c[VEC], o[VEC];
        unpack(xv[u][v], x);
        if (need_c) unpack(cv[u][v], c);
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          double nx;
          if (mode == MODE_SUMS) {
            nx = x[e];
          } else {
            double val;
            if (mode == MODE_ODD) {  // B + phi + psi (solver.cpp:170-172)
              val = EXACT ? __dadd_rn(__dadd_rn(x[e], phv[u]), psi_r[v][e])
                          : (x[e] + phv[u]) + psi_r[v][e];
            } else {                 // ((X - rho C) + phi) + psi (solver.cpp:97-99)
              val = EXACT ? __dadd_rn(__dadd_rn(__dsub_rn(x[e], __dmul_rn(rho, c[e])), phv[u]),
                                      psi_r[v][e])
                          : (fma(-rho, c[e], x[e]) + phv[u]) + psi_r[v][e];
            }
            nx = clamp0(val);
            if (REG == REG_QUAD) nx = EXACT ? div_rn_by(nx, qd, qinv) : nx * qinv;
            if (TRACK) {
              double xold = x[e];
              if (mode == MODE_ODD) xold = __dadd_rn(x[e], __dmul_rn(rho, c[e]));
              changed |= ((xold > 0.0) != (nx > 0.0));
              supp += (nx > 0.0);
            }
          }
          cacc[v][e] += nx;
          rs += nx;
          if (mode == MODE_EVEN)  // B = (-rho C) + X_{k+1}  (solver.cpp:162,167)
            o[e] = EXACT ? __dadd_rn(-__dmul_rn(rho, c[e]), nx) : nx - rho * c[e];
          else
            o[e] = nx;
        }
        if (mode != MODE_SUMS)
          reinterpret_cast<V*>(a.X + i * a.ld)[cols[v] / VEC] = pack<T>(o);
      }
      rs = warp_sum(rs);
      if (lane == 0) a.rowpart[i * (long long)gridDim.x + stripe] = rs;
    }
  }

  // Column partials: fixed-order cross-warp sum through shared memory.
  __shared__ double red[kWarps][TN];
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int e = 0; e < VEC; ++e) red[warp][v * 32 * VEC + lane * VEC + e] = cacc[v][e];
  __syncthreads();
  for (int t = threadIdx.x; t < TN; t += kThreads) {
    const long long col = col0 + t;
    if (col < a.ld) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) s += red[w][t];
      a.colpart[(long long)blockIdx.y * a.ld + col] = s;
    }
  }
  if (TRACK && mode != MODE_SUMS) {
    const unsigned long long ws = __reduce_add_sync(0xffffffffu, (unsigned)supp);
    const int wc = __any_sync(0xffffffffu, changed);
    if (lane == 0) {
      if (ws) atomicAdd(&a.ctl->supp_count, ws);
      if (wc) atomicOr(&a.ctl->supp_changed, 1);
    }
  }
}

// ------------------------------------------------------- group-lasso sweep
// One CTA per (row segment, column stripe). After the class-sort permutation
// every group (column j, class c) of column_class_blocks (groups.cpp:37-60) is
// the contiguous row segment of class c in column j, so the group norm is a
// per-column reduction over the CTA's rows. Phase 1 accumulates ||v_g||^2 per
// column; phase 2 re-reads the tile (the CTA's own tile, typically L2-hot),
// scales by [1 - rho*lambda/||v_g||]_+ (regularizers.cpp:85-99), stores, and
// produces the row/column partials like the plain sweep.
struct Segment {
  long long begin, end;
  int grouped;  // 0: rows in no group (label -1): plain clamp
  int pad;
};

template <typename T>
struct GLArgs {
  T* X;
  const T* C;
  const double* phi;
  const double* psi;
  double* rowpart;  // [m][stripes]
  double* colpart;  // [segments][ld]
  const Segment* seg;
  const Params* prm;
  Ctl* ctl;
  long long m, ld;
};

template <typename T, bool EXACT, bool TRACK, int NV>
__global__ void __launch_bounds__(kThreads) gl_sweep_kernel(GLArgs<T> a) {
  using V = typename Vec<T>::type;
  constexpr int VEC = Vec<T>::N;
  constexpr int TN = 32 * VEC * NV;
  const Ctl* ctl = a.ctl;
  if (ctl->done) return;
  const Params& prm = *a.prm;
  const int mode = prm.fused ? (ctl->fused_shifted ? MODE_ODD : MODE_EVEN) : MODE_NORMAL;
  const double rho = prm.rho, thr = prm.gl_thr;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long stripe = blockIdx.x;
  const long long col0 = stripe * TN;
  const Segment sg = a.seg[blockIdx.y];

  long long cols[NV];
  bool cok[NV];
  double psi_r[NV][VEC];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    cols[v] = col0 + v * 32 * VEC + lane * VEC;
    cok[v] = cols[v] < a.ld;
#pragma unroll
    for (int e = 0; e < VEC; ++e) psi_r[v][e] = cok[v] ? a.psi[cols[v] + e] : 0.0;
  }
  const bool need_c = mode != MODE_ODD || TRACK;

  auto pre_prox = [&](double x, double c, double ph, double ps) -> double {
    double val;
    if (mode == MODE_ODD)
      val = EXACT ? __dadd_rn(__dadd_rn(x, ph), ps) : (x + ph) + ps;
    else
      val = EXACT ? __dadd_rn(__dadd_rn(__dsub_rn(x, __dmul_rn(rho, c)), ph), ps)
                  : (fma(-rho, c, x) + ph) + ps;
    return clamp0(val);
  };

  __shared__ double red[kWarps][TN];
  __shared__ double sigma[TN];
  double sc[NV][VEC];
  if (sg.grouped) {
    double sq[NV][VEC];
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int e = 0; e < VEC; ++e) sq[v][e] = 0.0;
    for (long long i = sg.begin + warp; i < sg.end; i += kWarps) {
      const double ph = a.phi[i];
      const V* xrow = reinterpret_cast<const V*>(a.X + i * a.ld);
      const V* crow = reinterpret_cast<const V*>(a.C + i * a.ld);
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        if (!cok[v]) continue;
        double x[VEC], c[VEC];
        unpack(ld_rw(xrow + cols[v] / VEC), x);
        if (mode != MODE_ODD) unpack(ld_ro(crow + cols[v] / VEC), c);
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          const double val = pre_prox(x[e], c[e], ph, psi_r[v][e]);
          sq[v][e] += val * val;
        }
      }
    }
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int e = 0; e < VEC; ++e) red[warp][v * 32 * VEC + lane * VEC + e] = sq[v][e];
    __syncthreads();
    for (int t = threadIdx.x; t < TN; t += kThreads) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) s += red[w][t];
      const double nrm = sqrt(s);
      sigma[t] = (nrm <= thr) ? 0.0 : (EXACT ? __dsub_rn(1.0, __ddiv_rn(thr, nrm)) : 1.0 - thr / nrm);
    }
    __syncthreads();
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int e = 0; e < VEC; ++e) sc[v][e] = sigma[v * 32 * VEC + lane * VEC + e];
  } else {
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int e = 0; e < VEC; ++e) sc[v][e] = 1.0;
  }

  double cacc[NV][VEC];
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int e = 0; e < VEC; ++e) cacc[v][e] = 0.0;
  unsigned long long supp = 0;
  int changed = 0;
  for (long long i = sg.begin + warp; i < sg.end; i += kWarps) {
    const double ph = a.phi[i];
    V* xrow = reinterpret_cast<V*>(a.X + i * a.ld);
    const V* crow = reinterpret_cast<const V*>(a.C + i * a.ld);
    double rs = 0.0;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if (!cok[v]) continue;
      double x[VEC], c[VEC], o[VEC];
      unpack(ld_rw(xrow + cols[v] / VEC), x);
      if (need_c) unpack(ld_ro(crow + cols[v] / VEC), c);
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        double nx = pre_prox(x[e], c[e], ph, psi_r[v][e]);
        if (sg.grouped) nx = EXACT ? __dmul_rn(nx, sc[v][e]) : nx * sc[v][e];
        if (TRACK) {
          const double xold = (mode == MODE_ODD) ? __dadd_rn(x[e], __dmul_rn(rho, c[e])) : x[e];
          changed |= ((xold > 0.0) != (nx > 0.0));
          supp += (nx > 0.0);
        }
        cacc[v][e] += nx;
        rs += nx;
        o[e] = (mode == MODE_EVEN)
                   ? (EXACT ? __dadd_rn(-__dmul_rn(rho, c[e]), nx) : nx - rho * c[e])
                   : nx;
      }
      xrow[cols[v] / VEC] = pack<T>(o);
    }
    rs = warp_sum(rs);
    if (lane == 0) a.rowpart[i * (long long)gridDim.x + stripe] = rs;
  }
  __syncthreads();
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int e = 0; e < VEC; ++e) red[warp][v * 32 * VEC + lane * VEC + e] = cacc[v][e];
  __syncthreads();
  for (int t = threadIdx.x; t < TN; t += kThreads) {
    const long long col = col0 + t;
    if (col < a.ld) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) s += red[w][t];
      a.colpart[(long long)blockIdx.y * a.ld + col] = s;
    }
  }
  if (TRACK) {
    const unsigned long long ws = __reduce_add_sync(0xffffffffu, (unsigned)supp);
    const int wc = __any_sync(0xffffffffu, changed);
    if (lane == 0) {
      if (ws) atomicAdd(&a.ctl->supp_count, ws);
      if (wc) atomicOr(&a.ctl->supp_changed, 1);
    }
  }
}

// ------------------------------------------------ TMA / mbarrier helpers
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
// try_wait's suspend-time hint: a waiting warp sleeps until the phase
// completes (or the hint elapses) instead of re-issuing the probe -- spinning
// consumers otherwise take issue slots from the warps that compute
constexpr unsigned kMbarSuspendNs = 0x989680;
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(phase), "r"(kMbarSuspendNs)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(smem_addr(bar))
      : "memory");
}

// ---------------------------------------------------------------- reduce
// Blocks [0, RB): rows. R_i = sum_s rowpart[s][i] (stripe order), r_i = R_i - p_i,
// block partials (sum r, sum r^2, sum R); the last row block folds them in
// block order into exch[n..n+2]. Blocks [RB, RB+CB): S_j = sum_g colpart[g][j].
struct ReduceArgs {
  const double* rowpart;
  const double* colpart;
  const double* p;
  double* r;
  double* exch;     // [n + 3]
  double* bpart;    // [RB * 3]
  Ctl* ctl;
  long long m, n, ld;
  int stripes, groups, RB;
};

__global__ void __launch_bounds__(kThreads) reduce_kernel(ReduceArgs a) {
  Ctl* ctl = a.ctl;
  if (ctl->done) return;
  __shared__ double red[kWarps];
  __shared__ bool last;
  if ((int)blockIdx.x < a.RB) {
    const long long i = (long long)blockIdx.x * kThreads + threadIdx.x;
    double R = 0.0, r = 0.0;
    if (i < a.m) {
      for (int s = 0; s < a.stripes; ++s) R += a.rowpart[i * a.stripes + s];
      r = R - a.p[i];
      a.r[i] = r;
    }
    const double s1 = block_sum(r, red);
    const double s2 = block_sum(r * r, red);
    const double s3 = block_sum(R, red);
    if (threadIdx.x == 0) {
      a.bpart[blockIdx.x * 3 + 0] = s1;
      a.bpart[blockIdx.x * 3 + 1] = s2;
      a.bpart[blockIdx.x * 3 + 2] = s3;
      __threadfence();
      last = atomicAdd(&ctl->cnt_reduce, 1u) == (unsigned)(a.RB - 1);
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
      __threadfence();
      double t1 = 0.0, t2 = 0.0, t3 = 0.0;
      for (int b = 0; b < a.RB; ++b) {
        t1 += __ldcg(a.bpart + b * 3 + 0);
        t2 += __ldcg(a.bpart + b * 3 + 1);
        t3 += __ldcg(a.bpart + b * 3 + 2);
      }
      a.exch[a.n + 0] = t1;
      a.exch[a.n + 1] = t2;
      a.exch[a.n + 2] = t3;
      ctl->cnt_reduce = 0;
    }
  } else {
    const long long j = (long long)(blockIdx.x - a.RB) * kThreads + threadIdx.x;
    if (j < a.n) {
      double S = 0.0;
      for (int g = 0; g < a.groups; ++g) S += a.colpart[(long long)g * a.ld + j];
      a.exch[j] = S;
    }
  }
}

// ---------------------------------------------------------------- update
// solver.cpp:28-37 with the stopping logic of solver.cpp:179-235.
struct UpdateArgs {
  const double* exch;  // all-reduced [S(n) | sum r | sum r^2 | sum X]
  const double* q;
  const double* r;
  double* s;
  double* phi;
  double* psi;
  double* a;
  double* b;
  double* bpart;       // [RB + CB]
  const Params* prm;
  Ctl* ctl;
  TraceRow* trace;
  long long m_local, m_global, n;
  int RB, CB;
  cudaGraphConditionalHandle cond;
  int use_cond;
  int cert_follows;    // a certificate kernel pair runs after this one
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Stall/termination bookkeeping after convergence has been decided.
__device__ __forceinline__ void finish_iteration(Ctl* ctl, const Params& prm, long long kk,
                                                 bool converged) {
  if (converged) {
    ctl->done = 1;
    ctl->termination = TERM_CONVERGED;
  } else if (kk - ctl->last_improvement >= 10000) {  // solver.cpp:17, :232-235
    ctl->done = 1;
    ctl->termination = TERM_STALLED;
  } else if (kk >= prm.max_iter) {
    ctl->done = 1;
    ctl->termination = TERM_MAXITER;
  }
}

// Bookkeeping after X_{k+1} and the residual norms: theta/eta/k, trace
// support counters, and the solve loop's stopping logic (solver.cpp:179-235).
__device__ void finish_solve_iteration(Ctl* ctl, const Params& prm, long long k, double theta,
                                       double eta, double rp, int cert_follows,
                                       cudaGraphConditionalHandle cond, int use_cond) {
  ctl->theta[(k + 1) & 1] = __dsub_rn(theta, eta);
  ctl->eta = eta;
  ctl->k = k + 1;
  ctl->r_primal = rp;
  if (prm.fused) ctl->fused_shifted ^= 1;
  const long long kk = k + 1 - ctl->k0;
  if (prm.record_trace) {
    if (ctl->supp_changed) ctl->support_last_change = kk;
    ctl->last_support = (long long)ctl->supp_count;
    ctl->supp_changed = 0;
    ctl->supp_count = 0;
  }
  if (prm.solving) {
    if (!(rp - rp == 0.0)) {  // !isfinite  solver.cpp:181-185
      ctl->done = 1;
      ctl->termination = TERM_NONFINITE;
    } else {
      if (rp < ctl->best * (1.0 - 1e-14)) {  // solver.cpp:200-203
        ctl->best = rp;
        ctl->last_improvement = kk;
      }
      const bool at_check = (kk % prm.check_every) == 0;
      const bool want_cert = (at_check && prm.has_tol_gap && rp <= prm.tol_primal) ||
                             (prm.record_trace && (at_check || kk == prm.max_iter));
      if (want_cert && cert_follows) {
        ctl->want_cert = 1;  // the certificate kernels finish this iteration
      } else {
        const bool converged = at_check && rp <= prm.tol_primal && !prm.has_tol_gap;
        finish_iteration(ctl, prm, kk, converged);
      }
    }
    if (use_cond) cudaGraphSetConditional(cond, ctl->done ? 0u : 1u);
  }
}

__global__ void __launch_bounds__(kThreads) update_kernel(UpdateArgs a) {
  Ctl* ctl = a.ctl;
  if (ctl->done) return;
  const Params& prm = *a.prm;
  const long long k = ctl->k;
  const double theta = ctl->theta[k & 1];
  const double mn = (double)(a.m_global + a.n);
  const double eta = __ddiv_rn(a.exch[a.n], mn);
  const double shift = __dsub_rn(2.0 * eta, theta);
  const double dn = (double)a.n, dm = (double)a.m_global;
  __shared__ double red[kWarps];
  __shared__ bool last;
  double ssq = 0.0;
  if ((int)blockIdx.x < a.RB) {
    const long long i = (long long)blockIdx.x * kThreads + threadIdx.x;
    if (i < a.m_local) {
      const double ri = a.r[i], ai = a.a[i];
      a.phi[i] = __ddiv_rn(__dadd_rn(__dsub_rn(ai, 2.0 * ri), shift), dn);
      a.a[i] = __dsub_rn(ai, ri);
    }
  } else {
    const long long j = (long long)(blockIdx.x - a.RB) * kThreads + threadIdx.x;
    if (j < a.n) {
      const double sj = __dsub_rn(a.exch[j], a.q[j]);
      const double bj = a.b[j];
      a.s[j] = sj;
      a.psi[j] = __ddiv_rn(__dadd_rn(__dsub_rn(bj, 2.0 * sj), shift), dm);
      a.b[j] = __dsub_rn(bj, sj);
      ssq = sj * sj;
    }
  }
  const double bs = block_sum(ssq, red);
  if (threadIdx.x == 0) {
    a.bpart[blockIdx.x] = bs;
    __threadfence();
    last = atomicAdd(&ctl->cnt_update, 1u) == (unsigned)(a.RB + a.CB - 1);
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  double tssq = 0.0;
  for (int b = a.RB; b < a.RB + a.CB; ++b) tssq += __ldcg(a.bpart + b);
  const double rsq = a.exch[a.n + 1];
  // std::max(||r||, ||s||) with its NaN behaviour (solver.cpp:179).
  const double nr = sqrt(rsq), ns = sqrt(tssq);
  const double rp = (nr < ns) ? ns : nr;
  ctl->cnt_update = 0;
  finish_solve_iteration(ctl, prm, k, theta, eta, rp, a.cert_follows, a.cond, a.use_cond);
}

// ------------------------------------------------------------ grid barrier
__device__ __forceinline__ void grid_barrier(unsigned long long* counter) {
  // Arrival number a belongs to generation a / gridDim.x; wait until the
  // counter reaches the end of that generation (one atomic + one polled word).
  // The arrival is a gpu-scope release (cumulative over the CTA's writes that
  // bar.sync ordered before it), the poll a gpu-scope acquire: no separate
  // full fences on either side.
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long arrived;
    asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(arrived) : "l"(counter) : "memory");
    const unsigned long long target = (arrived / gridDim.x + 1ull) * gridDim.x;
    unsigned long long cur;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(cur) : "l"(counter) : "memory");
    } while (cur < target);
  }
  __syncthreads();
}

__device__ void finish_solve_iteration(Ctl* ctl, const Params& prm, long long k, double theta,
                                       double eta, double rp, int cert_follows,
                                       cudaGraphConditionalHandle cond, int use_cond);

// ------------------------------------------------------ certificate / objective
// duality.cpp:9-24 + problem.cpp:76-85. Tiled like the group-lasso sweep (one
// CTA per (segment, stripe)) so group norms of X and of U = [Xbar - X]_+ are
// CTA-local. Per-CTA partial vector (fixed order):
//   0 <C,X>  1 ||X||^2  2 ||U||^2 over ungrouped cells  3 sum_g ||X_g||
//   4 sum_g (||U_g|| - lambda)_+^2   5 <p,phi> (block 0 only)
constexpr int kCertVals = 6;

template <typename T>
struct CertArgs {
  const T* X;
  const T* C;
  const double* phi;
  const double* psi;
  const double* p;
  const Segment* seg;
  double* cpart;   // [num_ctas * kCertVals]
  double* csum;    // [kCertVals]  (all-reduced across ranks when sharded)
  const Params* prm;
  Ctl* ctl;
  long long m, ld;
  int reg;
  int objective_only;  // 1: run unconditionally (end of solve / objective)
};

template <typename T, int NV>
__global__ void __launch_bounds__(kThreads) cert_partial_kernel(CertArgs<T> a) {
  using V = typename Vec<T>::type;
  constexpr int VEC = Vec<T>::N;
  constexpr int TN = 32 * VEC * NV;
  Ctl* ctl = a.ctl;
  if (!a.objective_only && (ctl->done || !ctl->want_cert)) return;
  const Params& prm = *a.prm;
  const double rho = prm.rho, lam = prm.lambda;
  const bool shifted = prm.fused && ctl->fused_shifted;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long stripe = blockIdx.x;
  const long long col0 = stripe * TN;
  const Segment sg = a.seg[blockIdx.y];
  const bool gl = (a.reg == REG_GL) && sg.grouped;

  long long cols[NV];
  bool cok[NV];
  double psi_r[NV][VEC], gx[NV][VEC], gu[NV][VEC];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    cols[v] = col0 + v * 32 * VEC + lane * VEC;
    cok[v] = cols[v] < a.ld;
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      psi_r[v][e] = cok[v] ? a.psi[cols[v] + e] : 0.0;
      gx[v][e] = 0.0;
      gu[v][e] = 0.0;
    }
  }
  double lin = 0.0, xsq = 0.0, usq = 0.0;
  for (long long i = sg.begin + warp; i < sg.end; i += kWarps) {
    const double ph = a.phi[i];
    const V* xrow = reinterpret_cast<const V*>(a.X + i * a.ld);
    const V* crow = reinterpret_cast<const V*>(a.C + i * a.ld);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if (!cok[v]) continue;
      double x[VEC], c[VEC];
      unpack(xrow[cols[v] / VEC], x);
      unpack(ld_ro(crow + cols[v] / VEC), c);
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        if (cols[v] + e >= a.ld) continue;
        const double rc = __dmul_rn(rho, c[e]);
        const double xx = shifted ? __dadd_rn(x[e], rc) : x[e];
        const double xbar = clamp0(__dadd_rn(__dadd_rn(__dsub_rn(xx, rc), ph), psi_r[v][e]));
        const double u = clamp0(__dsub_rn(xbar, xx));
        lin += c[e] * xx;
        xsq += xx * xx;
        if (gl) {
          gx[v][e] += xx * xx;
          gu[v][e] += u * u;
        } else {
          usq += u * u;
        }
      }
    }
  }
  __shared__ double red[kWarps][TN];
  __shared__ double wred[kWarps];
  double glx = 0.0, glu = 0.0;
  if (gl) {
    for (int pass = 0; pass < 2; ++pass) {
      __syncthreads();
#pragma unroll
      for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int e = 0; e < VEC; ++e)
          red[warp][v * 32 * VEC + lane * VEC + e] = pass == 0 ? gx[v][e] : gu[v][e];
      __syncthreads();
      for (int t = threadIdx.x; t < TN; t += kThreads) {
        if (col0 + t >= a.ld) continue;
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) s += red[w][t];
        const double nrm = sqrt(s);
        if (pass == 0) {
          glx += nrm;
        } else {
          const double d = nrm - lam;
          glu += d > 0.0 ? d * d : 0.0;
        }
      }
    }
  }
  double vals[kCertVals] = {lin, xsq, usq, glx, glu, 0.0};
  const long long cta = (long long)blockIdx.y * gridDim.x + blockIdx.x;
  for (int q = 0; q < 5; ++q) {
    const double t = block_sum(vals[q], wred);
    if (threadIdx.x == 0) a.cpart[cta * kCertVals + q] = t;
  }
  // <p, phi> over local rows, done once by CTA 0.
  double pp = 0.0;
  if (cta == 0)
    for (long long i = threadIdx.x; i < a.m; i += kThreads) pp += a.p[i] * a.phi[i];
  const double tp = block_sum(pp, wred);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    a.cpart[cta * kCertVals + 5] = tp;
    __threadfence();
    last = atomicAdd(&ctl->cnt_cert, 1u) == (unsigned)(gridDim.x * gridDim.y - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    const long long nct = (long long)gridDim.x * gridDim.y;
    for (int q = 0; q < kCertVals; ++q) {
      double t = 0.0;
      for (long long b = 0; b < nct; ++b) t += __ldcg(a.cpart + b * kCertVals + q);
      a.csum[q] = t;
    }
    ctl->cnt_cert = 0;
  }
}

struct CertFinalArgs {
  const double* csum;
  const double* q;
  const double* psi;
  const Params* prm;
  Ctl* ctl;
  TraceRow* trace;
  long long n;
  int reg;
  int objective_only;
  cudaGraphConditionalHandle cond;
  int use_cond;
};

// Single block: <q,psi>, gap, dual residual, convergence decision, trace row.
__global__ void __launch_bounds__(kThreads) cert_final_kernel(CertFinalArgs a) {
  Ctl* ctl = a.ctl;
  if (!a.objective_only && (ctl->done || !ctl->want_cert)) return;
  const Params& prm = *a.prm;
  __shared__ double wred[kWarps];
  double qp = 0.0;
  for (long long j = threadIdx.x; j < a.n; j += kThreads) qp += a.q[j] * a.psi[j];
  const double tq = block_sum(qp, wred);
  if (threadIdx.x != 0) return;
  const double lin = a.csum[0], xsq = a.csum[1], usq = a.csum[2], glx = a.csum[3],
               glu = a.csum[4], pphi = a.csum[5];
  double h = 0.0, conj = 0.0, dres = 0.0;
  if (a.reg == REG_QUAD) {
    h = 0.5 * prm.alpha * xsq;                            // regularizers.cpp:50
    conj = usq / (2.0 * prm.alpha * prm.rho * prm.rho);   // regularizers.cpp:61
    dres = 0.0;
  } else if (a.reg == REG_GL) {
    h = prm.lambda * glx;                                 // regularizers.cpp:75-83
    dres = sqrt(glu + usq);                               // regularizers.cpp:28-37
  } else {
    dres = sqrt(usq);
  }
  const double primal = lin + h;
  ctl->objective = primal;
  if (a.objective_only) return;
  const double dual_value = (pphi + tq) / prm.rho - conj;  // duality.cpp:17-19
  const double gap = primal - dual_value;
  ctl->gap = gap;
  ctl->dres = dres;
  ctl->dual_value = dual_value;
  ctl->want_cert = 0;
  const long long kk = ctl->k - ctl->k0;
  const bool at_check = (kk % prm.check_every) == 0;
  bool converged = false;
  if (at_check && ctl->r_primal <= prm.tol_primal)
    converged = !prm.has_tol_gap || (fabs(gap) <= prm.tol_gap && dres <= prm.tol_gap);
  if (prm.record_trace && (at_check || converged || kk == prm.max_iter)) {
    if (ctl->trace_len < prm.trace_cap) {
      TraceRow& row = a.trace[ctl->trace_len];
      row.iter = kk;
      row.r_primal = ctl->r_primal;
      row.gap = gap;
      row.dual_residual = dres;
      row.support = ctl->last_support;
      row.elapsed_ms = prm.deterministic ? 0.0 : (double)(globaltimer_ns() - ctl->t0_ns) * 1e-6;
    }
    ctl->trace_len += 1;
  }
  finish_iteration(ctl, prm, kk, converged);
  if (a.use_cond) cudaGraphSetConditional(a.cond, ctl->done ? 0u : 1u);
}

// ---------------------------------------------------------------- utilities
__global__ void stamp_t0_kernel(Ctl* c) { c->t0_ns = globaltimer_ns(); }

// Moves whole rows (16-byte units): dst row dst_row[h] <- src row src_row[h].
__global__ void move_rows_kernel(uint4* dst, const uint4* src, const long long* dst_row,
                                 const long long* src_row, long long rows, long long units) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < rows * units;
       t += (long long)gridDim.x * blockDim.x) {
    const long long h = t / units, u = t - h * units;
    dst[dst_row[h] * units + u] = src[src_row[h] * units + u];
  }
}
// X = B + rho C: materialise the plan after an even fused iteration.
template <typename T>
__global__ void unshift_kernel(T* X, const T* C, const Params* prm, long long count) {
  const double rho = prm->rho;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < count;
       t += (long long)gridDim.x * blockDim.x)
    X[t] = (T)__dadd_rn((double)X[t], __dmul_rn(rho, (double)C[t]));
}

// Host-order rows (fp64, or already in the storage type) -> device-order
// storage rows (with the GL permutation).
template <typename T, typename S = double>
__global__ void scatter_rows_kernel(T* dst, const S* src, const long long* dev_row,
                                    long long rows, long long n, long long ld) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < rows * n;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = t / n, j = t - i * n;
    dst[dev_row[i] * ld + j] = (T)src[t];
  }
}

// Device-order storage rows -> host-order rows (fp64, or the storage type).
template <typename T, typename S = double>
__global__ void gather_rows_kernel(S* dst, const T* src, const long long* dev_row,
                                   long long rows, long long n, long long ld) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < rows * n;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = t / n, j = t - i * n;
    dst[t] = (S)src[dev_row[i] * ld + j];
  }
}

// make_state tail (solver.cpp:83-91): a = n phi + r, b = m psi + s,
// theta = (sum X - 1)/(m+n). exch holds the all-reduced sums of X0.
struct SeedArgs {
  const double* exch;
  const double* q;
  const double* r;
  const double* phi;
  const double* psi;
  double* s;
  double* a;
  double* b;
  Ctl* ctl;
  long long m_local, m_global, n;
};

__global__ void seed_state_kernel(SeedArgs a) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const double dn = (double)a.n, dm = (double)a.m_global;
  if (t < a.m_local) a.a[t] = __dadd_rn(__dmul_rn(dn, a.phi[t]), a.r[t]);
  if (t < a.n) {
    const double sj = __dsub_rn(a.exch[t], a.q[t]);
    a.s[t] = sj;
    a.b[t] = __dadd_rn(__dmul_rn(dm, a.psi[t]), sj);
  }
  if (t == 0) {
    a.ctl->theta[0] = __ddiv_rn(__dsub_rn(a.exch[a.n + 2], 1.0), (double)(a.m_global + a.n));
    a.ctl->theta[1] = a.ctl->theta[0];
    a.ctl->eta = 0.0;
    a.ctl->k = 0;
  }
}

// squared_distance_cost (datagen.cpp:43-54) in fp64; pass 0 reduces the max
// (normalize_cost, problem.cpp:68-74), pass 1 divides and stores.
template <typename T>
__global__ void sqdist_kernel(T* C, const double* src, const double* tgt, int d,
                              long long m, long long n, long long ld, const double* mx_in,
                              unsigned long long* mx_bits, int pass) {
  double local_max = 0.0;
  const double mx = pass ? *mx_in : 0.0;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < m * n;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = t / n, j = t - i * n;
    double sq = 0.0;
    for (int e = 0; e < d; ++e) {
      const double diff = __dsub_rn(src[i * d + e], tgt[j * d + e]);
      sq = __dadd_rn(sq, __dmul_rn(diff, diff));
    }
    const double c = __dmul_rn(0.5, sq);
    if (pass == 0) {
      local_max = fmax(local_max, c);
    } else {
      C[i * ld + j] = (T)(mx > 0.0 ? __ddiv_rn(c, mx) : c);
    }
  }
  if (pass == 0) {
    // non-negative doubles order like their bit patterns
    unsigned long long bits = (unsigned long long)__double_as_longlong(local_max);
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long ob = __shfl_xor_sync(0xffffffffu, bits, o);
      bits = ob > bits ? ob : bits;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(mx_bits, bits);
  }
}

}  // namespace otdrk
