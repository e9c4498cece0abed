// otdr_resident.cuh -- on-chip resident solve loop for plans that fit in the
// aggregate shared memory of the GPU (grid mode) or of one thread-block
// cluster (cluster mode, one problem per cluster: the batched entry point).
//
// Each CTA keeps its R rows of C and X in shared memory for the WHOLE solve:
// HBM is touched once to load C/X and once to write the final plan back. One
// DR iteration (solver.cpp:95-102, :23-38) per loop trip:
//   1. sweep own rows in smem: clamp + prox, row sums (complete), per-CTA
//      column sums; publish column sums + (sum r, sum r^2, sum X) partials
//   2. exchange barrier
//   3. column owner phase: CTA g owns a column slice, folds the G column
//      partials in rank order, updates s, psi, b; every CTA folds the scalar
//      partials (same order -> same eta/shift everywhere) and updates its phi/a
//   4. exchange barrier; every CTA gathers psi and the sum s^2 partials, forms
//      r_primal and runs the stopping logic (identical in every CTA)
// Grid mode exchanges through global scratch (L2) with a software grid
// barrier over co-resident CTAs (cooperative launch); cluster mode exchanges
// through distributed shared memory with cluster barriers.
#pragma once
#include "otdr_kernels.cuh"

#include <type_traits>

namespace otdrk {

constexpr int kRT = 512;       // threads per resident CTA
constexpr int kRW = kRT / 32;  // warps per resident CTA

// Fixed-order block sum over kRW warps (result valid in thread 0).
__device__ __forceinline__ double block_sum_r(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kRW; ++i) t += red[i];
  return t;
}

struct ResidentArgs {
  void* X;             // problem b at X + b * mat_stride (elements)
  const void* C;
  long long mat_stride;
  double* phi;         // per-problem row vectors, stride m
  double* a;
  double* r;
  const double* p;
  double* psi;         // per-problem column vectors, stride n
  double* b;
  double* s;
  const double* q;
  Ctl* ctl;            // per problem
  const Params* prm;
  double* gscratch;    // grid mode: [G][n + 4] exchange rows
  long long m, n, ld;
  int R;               // rows per CTA
  int G;               // CTAs per problem (grid size or cluster size)
  int reg;             // REG_NONE / REG_QUAD
  long long iters;     // raw mode: iterations to run (prm.solving == 0)
};

// Shared-memory layout (dynamic): C tile [R][ld] T | X tile [R][ld] T |
// xrow: this CTA's exchange row [n + 4] doubles (column sums | sr | sr2 | sR | ssq)
// | psi_s [n] | rowp [R][kWarps] | phi_s [R] | r_s [R]
// Warps split into column chunks (32 lanes x VEC columns) x row subsets.
template <typename T>
__host__ __device__ inline int resident_row_sets(long long ld) {
  const long long nch = (ld + 32 * Vec<T>::N - 1) / (32 * Vec<T>::N);
  return nch >= kRW ? 1 : (int)(kRW / nch);
}

template <typename T>
__host__ __device__ inline size_t resident_smem_bytes(long long R, long long n, long long ld) {
  const int sets = resident_row_sets<T>(ld);
  return size_t(2 * R * ld) * sizeof(T) + size_t(n + 4) * 8 + size_t(n) * 8 +
         size_t(R) * kRW * 8 + size_t(R) * 16 + (sets > 1 ? size_t(sets) * ld * 8 : 0) + 64;
}

// TG: storage type of C / X in global memory; T: type of the shared-memory
// tiles. fp32 storage may run on fp64 tiles (when they fit): the iteration is
// then the reference's fp64 arithmetic and X is rounded to fp32 only when the
// launch writes the plan back.
template <typename T, bool CLUSTER, typename TG = T>
__global__ void __launch_bounds__(kRT, 1) resident_kernel(ResidentArgs A) {
  namespace cg = cooperative_groups;
  using V = typename Vec<T>::type;
  constexpr int VEC = Vec<T>::N;
  const int G = A.G;
  int rank, prob;
  if constexpr (CLUSTER) {
    rank = (int)cg::this_cluster().block_rank();
    prob = (int)(blockIdx.x / G);
  } else {
    rank = (int)blockIdx.x;
    prob = 0;
  }
  Ctl* ctl = A.ctl + prob;
  const Params& prm = *A.prm;
  if (ctl->done) return;  // uniform per problem
  const long long m = A.m, n = A.n, ld = A.ld;
  const int R = A.R;
  TG* Xg = static_cast<TG*>(A.X) + prob * A.mat_stride;
  const TG* Cg = static_cast<const TG*>(A.C) + prob * A.mat_stride;
  double* phi = A.phi + prob * m;
  double* av = A.a + prob * m;
  double* rv = A.r + prob * m;
  const double* pv = A.p + prob * m;
  double* psi = A.psi + prob * n;
  double* bv = A.b + prob * n;
  double* sv = A.s + prob * n;
  const double* qv = A.q + prob * n;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* Ct = reinterpret_cast<T*>(smem_raw);
  T* Xt = Ct + (size_t)R * ld;
  double* xrow = reinterpret_cast<double*>(Xt + (size_t)R * ld);  // n + 4
  double* psi_s = xrow + n + 4;                                     // n
  double* rowp = psi_s + n;                                         // R * kWarps
  double* phi_s = rowp + (size_t)R * kRW;                           // R
  double* r_s = phi_s + R;                                          // R
  double* colbuf = r_s + R;                                         // sets x ld (sets > 1)
  const int nsets = resident_row_sets<T>(ld);
  const long long nch = (ld + 32 * VEC - 1) / (32 * VEC);
  __shared__ double red[kRW];
  __shared__ double red3[kRW][3];
  __shared__ double bc[4];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long i0 = (long long)rank * R;
  long long i1 = i0 + R;
  if (i1 > m) i1 = m;
  const int nr = i1 > i0 ? (int)(i1 - i0) : 0;
  // column slice owned in the column phase
  const long long j0 = n * rank / G, j1 = n * (rank + 1) / G;

  auto xbuf = [&](int rk) -> double* {  // exchange row of CTA rk
    if constexpr (CLUSTER) return cg::this_cluster().map_shared_rank(xrow, rk);
    else return A.gscratch + (size_t)rk * (size_t)(n + 4);
  };
  auto xget = [&](int rk, long long idx) -> double {  // peer read (L2 in grid mode)
    if constexpr (CLUSTER) return xbuf(rk)[idx];
    else return __ldcg(xbuf(rk) + idx);
  };
  // fixed-order fold of one exchange slot over the G (<= 160) CTAs by one
  // warp: all peer loads are issued before any add (one L2 round trip)
  auto warp_fold = [&](long long idx) -> double {
    double v[5];
#pragma unroll
    for (int u = 0; u < 5; ++u) {
      const int h = lane + 32 * u;
      v[u] = h < G ? xget(h, idx) : 0.0;
    }
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < 5; ++u) s += v[u];
    return warp_sum(s);
  };
  auto xsync = [&]() {
    if constexpr (CLUSTER) {
      cg::this_cluster().sync();
    } else {
      grid_barrier(&ctl->bar_res);
    }
  };

  // load the tiles (once per solve)
  {
    const long long elems = (long long)nr * ld;
    if constexpr (std::is_same<T, TG>::value) {
      const V* cs = reinterpret_cast<const V*>(Cg + i0 * ld);
      const V* xs = reinterpret_cast<const V*>(Xg + i0 * ld);
      V* cd = reinterpret_cast<V*>(Ct);
      V* xd = reinterpret_cast<V*>(Xt);
      for (long long t = threadIdx.x; t < elems / VEC; t += kRT) {
        cd[t] = cs[t];
        xd[t] = xs[t];
      }
    } else {  // widen (exact)
      using VG = typename Vec<TG>::type;
      constexpr int VG_N = Vec<TG>::N;
      const VG* cs = reinterpret_cast<const VG*>(Cg + i0 * ld);
      const VG* xs = reinterpret_cast<const VG*>(Xg + i0 * ld);
      for (long long t = threadIdx.x; t < elems / VG_N; t += kRT) {
        double cw[VG_N], xw[VG_N];
        unpack(cs[t], cw);
        unpack(xs[t], xw);
#pragma unroll
        for (int e = 0; e < VG_N; ++e) {
          Ct[t * VG_N + e] = (T)cw[e];
          Xt[t * VG_N + e] = (T)xw[e];
        }
      }
    }
    for (long long j = threadIdx.x; j < n; j += kRT) psi_s[j] = psi[j];
    for (int t = threadIdx.x; t < nr; t += kRT) phi_s[t] = phi[i0 + t];
  }
  __syncthreads();

  const double rho = prm.rho, qd = prm.quad_d, qinv = prm.quad_inv;
  const bool exact = sizeof(T) == 8;
  const double dm = (double)m, dn = (double)n, mn = (double)(m + n);
  long long k = ctl->k;
  double theta = ctl->theta[k & 1];
  double best = ctl->best;
  long long last_imp = ctl->last_improvement;
  const long long k0 = ctl->k0;
  long long it = 0;

  for (;;) {
    // ---- 1. sweep own rows. Warp w: column chunk(s) of 32*VEC columns and the
    // 8-row groups g = wset, wset + nsets, ...; row sums by 8-row reduce-scatter.
    for (int t = threadIdx.x; t < nr * kRW; t += kRT) rowp[t] = 0.0;
    __syncthreads();
    const int wset = (nsets > 1) ? warp / (int)nch : 0;
    const bool wactive = (nsets > 1) ? (warp < (int)nch * nsets) : true;
    for (long long c = (nsets > 1) ? warp % nch : warp; wactive && c < nch;
         c += (nsets > 1) ? nch : kRW) {
      const long long cb = c * 32 * VEC + (long long)lane * VEC;
      const bool ok = cb < ld;
      double ps[VEC], cacc[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        ps[e] = (cb + e < n) ? psi_s[cb + e] : -INFINITY;
        cacc[e] = 0.0;
      }
      const V* xcol = reinterpret_cast<const V*>(Xt + cb);
      const V* ccol = reinterpret_cast<const V*>(Ct + cb);
      const long long ldv = ld / VEC;
      for (int t0 = wset * 8; t0 < nr; t0 += nsets * 8) {
        double rs[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int t = t0 + u;
          rs[u] = 0.0;
          if (ok && t < nr) {
            const double ph = phi_s[t];
            double x[VEC], cc[VEC], o[VEC];
            unpack(xcol[t * ldv], x);
            unpack(ccol[t * ldv], cc);
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
              const double val = exact ? __dadd_rn(__dadd_rn(__dsub_rn(x[e], __dmul_rn(rho, cc[e])), ph), ps[e])
                                       : (fma(-rho, cc[e], x[e]) + ph) + ps[e];
              double nx = clamp0(val);
              if (A.reg == REG_QUAD) nx = exact ? div_rn_by(nx, qd, qinv) : nx * qinv;
              o[e] = nx;
              cacc[e] += nx;
              rs[u] += nx;
            }
            const_cast<V*>(xcol)[t * ldv] = pack<T>(o);
          }
        }
        const double tot = reduce8_rows(rs, lane);
        const int row = t0 + row8_of(lane);
        if ((lane & 3) == 0 && row < nr) rowp[row * kRW + warp] += tot;
      }
      double* cdst = (nsets > 1) ? colbuf + (size_t)wset * ld : xrow;
#pragma unroll
      for (int e = 0; e < VEC; ++e)
        if (cb + e < ((nsets > 1) ? ld : n)) cdst[cb + e] = cacc[e];
    }
    if (nsets > 1) {  // fold the row subsets' column partials in a fixed order
      __syncthreads();
      for (long long j = threadIdx.x; j < n; j += kRT) {
        double sacc = 0.0;
        for (int w = 0; w < nsets; ++w) sacc += colbuf[(size_t)w * ld + j];
        xrow[j] = sacc;
      }
    }
    __syncthreads();
    // row sums -> r (own rows), scalar partials
    double sr = 0.0, sr2 = 0.0, sR = 0.0;
    for (int t = threadIdx.x; t < nr; t += kRT) {
      double Rr = 0.0;
#pragma unroll
      for (int w = 0; w < kRW; ++w) Rr += rowp[t * kRW + w];
      const double ri = Rr - pv[i0 + t];
      r_s[t] = ri;
      sr += ri;
      sr2 += ri * ri;
      sR += Rr;
    }
    {
      // three fixed-order block sums in one pass (one barrier pair)
      sr = warp_sum(sr);
      sr2 = warp_sum(sr2);
      sR = warp_sum(sR);
      __syncthreads();
      if (lane == 0) {
        red3[warp][0] = sr;
        red3[warp][1] = sr2;
        red3[warp][2] = sR;
      }
      __syncthreads();
      double t1 = 0.0, t2 = 0.0, t3 = 0.0;
      if (threadIdx.x == 0)
        for (int w = 0; w < kRW; ++w) {
          t1 += red3[w][0];
          t2 += red3[w][1];
          t3 += red3[w][2];
        }
      if (threadIdx.x == 0) {
        if constexpr (CLUSTER) {
          xrow[n] = t1;
          xrow[n + 1] = t2;
          xrow[n + 2] = t3;
        } else {
          double* g = xbuf(rank);
          g[n] = t1;
          g[n + 1] = t2;
          g[n + 2] = t3;
        }
      }
      if constexpr (!CLUSTER) {
        double* g = xbuf(rank);
        for (long long j = threadIdx.x; j < n; j += kRT) g[j] = xrow[j];
      }
    }
    xsync();  // ---- 2. column partials and scalar partials visible
    // the scalar folds (last two warps) and each warp's first owned column
    // fold are in flight together: one L2 round trip before the recurrence
    if (warp == kRW - 1 || warp == kRW - 2) {
      const double u = warp_fold(n + (kRW - 1 - warp));
      if (lane == 0) bc[kRW - 1 - warp] = u;
    }
    const long long jfirst = j0 + warp;
    const double Sfirst = jfirst < j1 ? warp_fold(jfirst) : 0.0;
    __syncthreads();
    const double eta = __ddiv_rn(bc[0], mn);
    const double shift = __dsub_rn(2.0 * eta, theta);
    const double rsq = bc[1];
    // ---- 3. own rows: phi, a; owned columns: s, psi, b
    for (int t = threadIdx.x; t < nr; t += kRT) {
      const double ri = r_s[t], ai = av[i0 + t];
      const double ph = __ddiv_rn(__dadd_rn(__dsub_rn(ai, 2.0 * ri), shift), dn);
      phi_s[t] = ph;
      av[i0 + t] = __dsub_rn(ai, ri);
    }
    double ssq = 0.0;  // warp per owned column: lanes fold the G partials
    for (long long j = jfirst; j < j1; j += kRW) {
      const double S = j == jfirst ? Sfirst : warp_fold(j);
      if (lane == 0) {
        const double sj = __dsub_rn(S, qv[j]);
        const double bj = bv[j];
        sv[j] = sj;
        psi[j] = __ddiv_rn(__dadd_rn(__dsub_rn(bj, 2.0 * sj), shift), dm);
        bv[j] = __dsub_rn(bj, sj);
        ssq += sj * sj;
      }
    }
    {
      const double t4 = block_sum_r(ssq, red);
      if constexpr (CLUSTER) xsync();  // peers done reading this CTA's column partials
      if (threadIdx.x == 0) {
        if constexpr (CLUSTER) xrow[n + 3] = t4;
        else xbuf(rank)[n + 3] = t4;
      }
      if constexpr (CLUSTER) {  // publish owned psi slice in smem for peers
        for (long long j = j0 + threadIdx.x; j < j1; j += kRT) xrow[j] = psi[j];
      }
    }
    xsync();  // ---- 4. psi slices and sum s^2 partials visible
    if constexpr (CLUSTER) {
      for (long long j = threadIdx.x; j < n; j += kRT) {  // owner of column j
        int h = (int)((j * G) / n);
        while (h + 1 < G && n * (h + 1) / G <= j) ++h;
        while (h > 0 && n * h / G > j) --h;
        psi_s[j] = xbuf(h)[j];
      }
    } else {
      // warp 0 folds the sum s^2 partials while the other warps gather psi
      if (warp > 0)
        for (long long j = threadIdx.x - 32; j < n; j += kRT - 32) psi_s[j] = __ldcg(psi + j);
    }
    if (warp == 0) {
      const double u4 = warp_fold(n + 3);
      if (lane == 0) bc[2] = u4;
    }
    __syncthreads();
    const double nr2 = sqrt(rsq), ns2 = sqrt(bc[2]);
    const double rp = (nr2 < ns2) ? ns2 : nr2;
    theta = __dsub_rn(theta, eta);
    ++k;
    ++it;
    const long long kk = k - k0;
    bool done = false;
    int term = TERM_MAXITER;
    if (prm.solving) {
      if (!(rp - rp == 0.0)) {
        done = true;
        term = TERM_NONFINITE;
      } else {
        if (rp < best * (1.0 - 1e-14)) {
          best = rp;
          last_imp = kk;
        }
        const bool at_check = (kk % prm.check_every) == 0;
        if (at_check && rp <= prm.tol_primal) {
          done = true;
          term = TERM_CONVERGED;
        } else if (kk - last_imp >= 10000) {
          done = true;
          term = TERM_STALLED;
        } else if (kk >= prm.max_iter) {
          done = true;
          term = TERM_MAXITER;
        }
      }
    } else if (it >= A.iters) {
      done = true;
    }
    if (done) {
      if (rank == 0 && threadIdx.x == 0) {
        ctl->k = k;
        ctl->theta[k & 1] = theta;
        ctl->eta = eta;
        ctl->r_primal = rp;
        ctl->best = best;
        ctl->last_improvement = last_imp;
        if (prm.solving) {
          ctl->done = 1;
          ctl->termination = term;
        }
      }
      break;
    }
    if constexpr (CLUSTER) {
      // peers may still read this CTA's psi slice / partials before the next
      // iteration overwrites xrow
      cg::this_cluster().sync();
    }
  }
  // primal objective <C,X> + h(X) (problem.cpp:76-85) from the resident tiles
  {
    double lin = 0.0, xsq = 0.0;
    const long long elems = (long long)nr * ld;
    for (long long t = threadIdx.x; t < elems; t += kRT) {
      const double xv = (double)Xt[t], cv = (double)Ct[t];
      lin += cv * xv;
      xsq += xv * xv;
    }
    const double t1 = block_sum_r(lin, red);
    const double t2 = block_sum_r(xsq, red);
    if (threadIdx.x == 0) {
      double* g = CLUSTER ? xrow : xbuf(rank);
      g[n] = t1;
      g[n + 1] = t2;
    }
    xsync();
    if (rank == 0 && warp == 0) {
      const double u1 = warp_fold(n), u2 = warp_fold(n + 1);
      if (lane == 0) ctl->objective = u1 + (A.reg == REG_QUAD ? 0.5 * prm.alpha * u2 : 0.0);
    }
  }
  // write back the plan, phi and r of own rows (psi, s, b, a already global)
  {
    const long long elems = (long long)nr * ld;
    if constexpr (std::is_same<T, TG>::value) {
      V* xd = reinterpret_cast<V*>(Xg + i0 * ld);
      const V* xs = reinterpret_cast<const V*>(Xt);
      for (long long t = threadIdx.x; t < elems / VEC; t += kRT) xd[t] = xs[t];
    } else {  // round to the storage type (the plan's only rounding in this launch)
      using VG = typename Vec<TG>::type;
      constexpr int VG_N = Vec<TG>::N;
      VG* xd = reinterpret_cast<VG*>(Xg + i0 * ld);
      for (long long t = threadIdx.x; t < elems / VG_N; t += kRT) {
        double o[VG_N];
#pragma unroll
        for (int e = 0; e < VG_N; ++e) o[e] = (double)Xt[t * VG_N + e];
        xd[t] = pack<TG>(o);
      }
    }
    for (int t = threadIdx.x; t < nr; t += kRT) {
      phi[i0 + t] = phi_s[t];
      rv[i0 + t] = r_s[t];
    }
  }
  if constexpr (CLUSTER) cg::this_cluster().sync();  // no CTA exits while peers read its smem
}

}  // namespace otdrk
