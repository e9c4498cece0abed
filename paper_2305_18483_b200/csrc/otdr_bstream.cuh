// otdr_bstream.cuh -- batched solve, one CTA per problem, plans streamed from
// HBM (the minibatch shape of cfg5: B = 256 problems of 512 x 512).
//
// Every CTA owns one problem for the whole solve: its vectors (phi, a, r, p,
// psi, b, s, q) live in shared memory, and every DR iteration
// (solver.cpp:95-102 + :23-38) streams the problem's C and X through
// per-thread cp.async queues (as in otdr_stream.cuh). All folds are CTA-local,
// so an iteration costs two __syncthreads and no grid or cluster barrier; the
// batch is bound by HBM bandwidth (12 B per entry per iteration) instead of
// by per-iteration exchange latency. Problems that converge retire their CTA
// and the hardware schedules the next one.
//
// Warp layout: the ld columns are cut into nch chunks of 32 x VEC columns;
// warp w streams chunk w % nch for the rows of row set w / nch (rows set,
// set + nsets, ...). Row partials rowp[row][chunk] and column partials
// colbuf[set][col] are folded in fixed order (thread per row / column).
#pragma once
#include "otdr_stream.cuh"

namespace otdrk {

constexpr int kBSTMax = 512;         // threads per CTA (template NT <= this)

struct BStreamArgs {
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
  long long m, n, ld;
  int nch, nsets;
  int reg;
};

template <typename T, int D, int NT>
__host__ __device__ inline size_t bstream_smem_bytes(long long m, long long ld, int nch, int nsets) {
  return size_t(D) * 2 * NT * 16 + size_t(4 * m + 5 * ld + m * nch + (long long)nsets * ld) * 8 +
         size_t(NT / 32 + 16) * 8;
}

// CS > 1: a thread-block cluster of CS CTAs per problem, each streaming a
// band of the rows; the column partials and the three row scalars are
// combined over distributed shared memory in cluster-rank order (identical in
// every CTA), so the problem runs CS times faster -- the batch's tail is its
// slowest problems, which otherwise run on one SM each.
template <typename T, bool EXACT, int D, int NT, int CS>
__global__ void __launch_bounds__(NT, 512 / NT) bstream_kernel(BStreamArgs A) {
  namespace cg = cooperative_groups;
  constexpr int kBST = NT;
  constexpr int kBSW = NT / 32;
  using V = typename Vec<T>::type;
  constexpr int VEC = Vec<T>::N;
  const int prob = blockIdx.x / CS;
  const int crank = CS > 1 ? (int)cg::this_cluster().block_rank() : 0;
  Ctl* ctl = A.ctl + prob;
  if (ctl->done) return;  // uniform over the cluster
  const Params& prm = *A.prm;
  const long long m = A.m, n = A.n, ld = A.ld;
  const int nch = A.nch, nsets = A.nsets;
  T* Xg = static_cast<T*>(A.X) + prob * A.mat_stride;
  const T* Cg = static_cast<const T*>(A.C) + prob * A.mat_stride;

  extern __shared__ __align__(16) unsigned char bs_smem[];
  uint4* q = reinterpret_cast<uint4*>(bs_smem);
  double* phi_s = reinterpret_cast<double*>(bs_smem + size_t(D) * 2 * kBST * 16);
  double* a_s = phi_s + m;
  double* r_s = a_s + m;
  double* p_s = r_s + m;
  double* psi_s = p_s + m;   // ld (padding: -inf)
  double* b_s = psi_s + ld;
  double* s_s = b_s + ld;
  double* q_s = s_s + ld;
  double* rowp = q_s + ld;                 // [m][nch]
  double* colbuf = rowp + m * nch;         // [nsets][ld]
  double* cpart = colbuf + (long long)nsets * ld;  // [ld] this CTA's column sums
  double* red = cpart + ld;                // [kBSW]
  double* bc = red + kBSW;                 // [8]
  double* xs = bc + 8;                     // [8] this CTA's row scalars (DSMEM-visible)
  // rows of this CTA's band
  const long long rb = m * crank / CS, re = m * (crank + 1) / CS;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (long long i = rb + threadIdx.x; i < re; i += kBST) {
    phi_s[i] = A.phi[prob * m + i];
    a_s[i] = A.a[prob * m + i];
    r_s[i] = A.r[prob * m + i];
    p_s[i] = A.p[prob * m + i];
  }
  for (long long j = threadIdx.x; j < ld; j += kBST) {
    const bool in = j < n;
    psi_s[j] = in ? A.psi[prob * n + j] : -INFINITY;
    b_s[j] = in ? A.b[prob * n + j] : 0.0;
    s_s[j] = in ? A.s[prob * n + j] : 0.0;
    q_s[j] = in ? A.q[prob * n + j] : 0.0;
  }
  __syncthreads();

  const double rho = prm.rho, qd = prm.quad_d, qinv = prm.quad_inv;
  const bool quad = A.reg == REG_QUAD;
  const double dm = (double)m, dn = (double)n, mn = (double)(m + n);
  long long k = ctl->k;
  double theta = ctl->theta[k & 1];
  double best = ctl->best;
  long long last_imp = ctl->last_improvement;
  const long long k0 = ctl->k0;

  const bool wactive = warp < nch * nsets;
  const int chunk = warp % nch, set = warp / nch;
  const long long cb = (long long)chunk * 32 * VEC + (long long)lane * VEC;
  const bool cok = wactive && cb < ld;
  auto slot = [&](int st, int kk) -> uint4* { return q + ((size_t)(st * 2 + kk) * kBST + threadIdx.x); };

  double eta = 0.0, rp = 0.0;
  for (;;) {
    // ---- sweep: this warp's chunk over rows set, set + nsets, ...
    if (wactive) {
      double ps[VEC], cacc[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        ps[e] = cok ? psi_s[cb + e] : 0.0;
        cacc[e] = 0.0;
      }
      long long iss = rb + set;
      auto issue = [&](int st) {
        if (iss < re && cok) {
          cp_async16(slot(st, 0), Xg + iss * ld + cb);
          cp_async16(slot(st, 1), Cg + iss * ld + cb);
        }
        iss += nsets;
        cp_async_commit();
      };
#pragma unroll
      for (int d = 0; d < D - 1; ++d) issue(d);
      int st = 0;
      for (long long i = rb + set; i < re; i += nsets) {
        issue(st == 0 ? D - 1 : st - 1);
        cp_async_wait<D - 1>();
        double rs = 0.0;
        if (cok) {
          const double ph = phi_s[i];
          double x[VEC], c[VEC], o[VEC];
          unpack(*reinterpret_cast<const V*>(slot(st, 0)), x);
          unpack(*reinterpret_cast<const V*>(slot(st, 1)), c);
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            const double val = EXACT ? __dadd_rn(__dadd_rn(__dsub_rn(x[e], __dmul_rn(rho, c[e])), ph), ps[e])
                                     : (fma(-rho, c[e], x[e]) + ph) + ps[e];
            double nx = clamp0(val);
            if (quad) nx = EXACT ? div_rn_by(nx, qd, qinv) : nx * qinv;
            o[e] = nx;
            cacc[e] += nx;
            rs += nx;
          }
          *reinterpret_cast<V*>(Xg + i * ld + cb) = pack<T>(o);
        }
        rs = warp_sum(rs);
        if (lane == 0) rowp[i * nch + chunk] = rs;
        st = (st + 1 == D) ? 0 : st + 1;
      }
      cp_async_wait<0>();
      if (cok) {
#pragma unroll
        for (int e = 0; e < VEC; ++e) colbuf[(long long)set * ld + cb + e] = cacc[e];
      }
    }
    __syncthreads();
    // ---- folds: rows (chunk order), this CTA's column partials (row-set order)
    double sr = 0.0, sr2 = 0.0, ssq = 0.0;
    for (long long i = rb + threadIdx.x; i < re; i += kBST) {
      double R = 0.0;
      for (int c = 0; c < nch; ++c) R += rowp[i * nch + c];
      const double ri = R - p_s[i];
      r_s[i] = ri;
      sr += ri;
      sr2 += ri * ri;
    }
    for (long long j = threadIdx.x; j < n; j += kBST) {
      double S = 0.0;
      for (int t = 0; t < nsets; ++t) S += colbuf[(long long)t * ld + j];
      cpart[j] = S;
    }
    {
      const double t1 = block_sum_n<kBSW>(sr, red);
      const double t2 = block_sum_n<kBSW>(sr2, red);
      if (threadIdx.x == 0) {
        xs[0] = t1;
        xs[1] = t2;
      }
    }
    if constexpr (CS > 1) cg::this_cluster().sync();  // peers' partials visible (DSMEM)
    else __syncthreads();
    // column sums and scalars folded in cluster-rank order (same in every CTA)
    for (long long j = threadIdx.x; j < n; j += kBST) {
      double S = 0.0;
#pragma unroll
      for (int r = 0; r < CS; ++r) {
        const double* pc = CS > 1 ? cg::this_cluster().map_shared_rank(cpart, r) : cpart;
        S += pc[j];
      }
      const double sj = __dsub_rn(S, q_s[j]);
      s_s[j] = sj;
      ssq += sj * sj;
    }
    {
      const double t4 = block_sum_n<kBSW>(ssq, red);
      if (threadIdx.x == 0) {
        double u0 = 0.0, u1 = 0.0;
#pragma unroll
        for (int r = 0; r < CS; ++r) {
          const double* px = CS > 1 ? cg::this_cluster().map_shared_rank(xs, r) : xs;
          u0 += px[0];
          u1 += px[1];
        }
        bc[0] = u0;
        bc[1] = u1;
        bc[3] = t4;
      }
    }
    __syncthreads();
    eta = __ddiv_rn(bc[0], mn);
    const double shift = __dsub_rn(2.0 * eta, theta);
    for (long long i = rb + threadIdx.x; i < re; i += kBST) {
      const double ri = r_s[i], ai = a_s[i];
      phi_s[i] = __ddiv_rn(__dadd_rn(__dsub_rn(ai, 2.0 * ri), shift), dn);
      a_s[i] = __dsub_rn(ai, ri);
    }
    for (long long j = threadIdx.x; j < n; j += kBST) {
      const double sj = s_s[j], bj = b_s[j];
      psi_s[j] = __ddiv_rn(__dadd_rn(__dsub_rn(bj, 2.0 * sj), shift), dm);
      b_s[j] = __dsub_rn(bj, sj);
    }
    const double nr2 = sqrt(bc[1]), ns2 = sqrt(bc[3]);
    rp = (nr2 < ns2) ? ns2 : nr2;  // std::max semantics (solver.cpp:179)
    theta = __dsub_rn(theta, eta);
    ++k;
    const long long kk = k - k0;
    bool done = false;
    int term = TERM_MAXITER;
    if (!(rp - rp == 0.0)) {  // solver.cpp:181-185
      done = true;
      term = TERM_NONFINITE;
    } else {
      if (rp < best * (1.0 - 1e-14)) {  // solver.cpp:200-203
        best = rp;
        last_imp = kk;
      }
      const bool at_check = (kk % prm.check_every) == 0;
      if (at_check && rp <= prm.tol_primal) {
        done = true;
        term = TERM_CONVERGED;
      } else if (kk - last_imp >= 10000) {  // solver.cpp:17, :232-235
        done = true;
        term = TERM_STALLED;
      } else if (kk >= prm.max_iter) {
        done = true;
        term = TERM_MAXITER;
      }
    }
    // phi / psi complete before the next sweep; peers done reading cpart / xs
    if constexpr (CS > 1) cg::this_cluster().sync();
    else __syncthreads();
    if (done) {
      if (threadIdx.x == 0 && crank == 0) {
        ctl->k = k;
        ctl->theta[k & 1] = theta;
        ctl->eta = eta;
        ctl->r_primal = rp;
        ctl->best = best;
        ctl->last_improvement = last_imp;
        ctl->done = 1;
        ctl->termination = term;
      }
      break;
    }
  }
  // primal objective <C,X> + h(X) (problem.cpp:76-85, regularizers.cpp:49-51)
  {
    double lin = 0.0, xsq = 0.0;
    for (long long t = threadIdx.x; t < (re - rb) * (ld / VEC); t += kBST) {
      const long long i = rb + t / (ld / VEC), cv = t % (ld / VEC);
      double x[VEC], c[VEC];
      unpack(reinterpret_cast<const V*>(Xg + i * ld)[cv], x);
      unpack(reinterpret_cast<const V*>(Cg + i * ld)[cv], c);
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        lin += c[e] * x[e];
        xsq += x[e] * x[e];
      }
    }
    const double t1 = block_sum_n<kBSW>(lin, red);
    const double t2 = block_sum_n<kBSW>(xsq, red);
    if (threadIdx.x == 0) {
      xs[2] = t1;
      xs[3] = t2;
    }
    if constexpr (CS > 1) cg::this_cluster().sync();
    else __syncthreads();
    if (threadIdx.x == 0 && crank == 0) {
      double u1 = 0.0, u2 = 0.0;
#pragma unroll
      for (int r = 0; r < CS; ++r) {
        const double* px = CS > 1 ? cg::this_cluster().map_shared_rank(xs, r) : xs;
        u1 += px[2];
        u2 += px[3];
      }
      ctl->objective = u1 + (quad ? 0.5 * prm.alpha * u2 : 0.0);
    }
  }
  for (long long i = rb + threadIdx.x; i < re; i += kBST) {
    A.phi[prob * m + i] = phi_s[i];
    A.a[prob * m + i] = a_s[i];
    A.r[prob * m + i] = r_s[i];
  }
  if (crank == 0) {
    for (long long j = threadIdx.x; j < n; j += kBST) {
      A.psi[prob * n + j] = psi_s[j];
      A.b[prob * n + j] = b_s[j];
      A.s[prob * n + j] = s_s[j];
    }
  }
  if constexpr (CS > 1) cg::this_cluster().sync();  // no CTA exits while peers read its smem
}

}  // namespace otdrk
