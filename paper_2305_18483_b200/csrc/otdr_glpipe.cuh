// otdr_glpipe.cuh -- single-pass group-lasso sweep with a software pipeline
// across column stripes (regularizers.cpp:85-99 fused into the DR sweep).
//
// After the class-sort permutation every group (column j, class c) of
// column_class_blocks (groups.cpp:37-60) is the contiguous row segment of
// class c in column j. The block soft-threshold needs the norm of the whole
// segment column before any entry can be written, so v = [((X - rho C) + phi)
// + psi]_+ of one segment x 128-byte stripe is staged in shared memory (vbuf,
// 125 KB for a 1000-row class in fp32).
//
// One persistent CTA per SM (512 threads) claims work items -- (segment,
// position = run of up to 10 consecutive stripes) -- from an atomic counter,
// position-major, so the short positions at the end of the stripe range
// (2 stripes) are the last claims and CTA finish times stay close. Inside an item
// the stripes are pipelined row by row through the SAME staging buffer:
//   step j: for every row r of the segment
//             phase 2 of stripe j-1: read v[r], scale by sigma_{j-1}, store X,
//                                    row / column sums
//             phase 1 of stripe j:   v[r] from the cp.async queue (X, C),
//                                    stage it in the slot just freed, sum v^2
//           then one CTA barrier: norms of stripe j -> sigma_j, column sums
//           of stripe j-1 -> colpart
// so HBM sees the loads of stripe j and the stores of stripe j-1 at the
// same time and no CTA ever idles on a whole-tile load. Every thread streams
// its own 16-byte chunks of X and C through a private D-deep cp.async queue
// (as in otdr_stream.cuh). Row sums accumulate in shared memory over the
// item's stripes and are flushed to rowpart[row][item group]; column sums go
// to colpart[segment][col] -- the reduce kernel's layout.
//
// Staging precision is T: fp64 storage stages fp64 v (element-wise identical
// to the reference); fp32 storage stages fp32 v (<= 1 ulp(fp32) from v*scale).
#pragma once
#include "otdr_stream.cuh"

namespace otdrk {

constexpr int kGLPThreads = 512;
constexpr int kGLPWarps = kGLPThreads / 32;
constexpr int kGLPMaxG = 16;

struct GLPipeArgs {
  void* X;
  const void* C;
  const double* phi;
  const double* psi;
  double* rowpart;        // [m][ngroups]
  double* colpart;        // [nseg][ld]
  const Segment* seg;
  const int2* pos;        // [ngroups] stripe positions {first stripe, stripes}, shared by all segments
  const Params* prm;
  Ctl* ctl;
  long long m, ld;
  int nseg, nstr, ngroups, Lmax;
};

template <typename T, int D>
__host__ __device__ constexpr size_t glpipe_queue_bytes() {
  return size_t(D) * 2 * kGLPThreads * 16;
}
template <typename T, int D, int WB>
__host__ __device__ inline size_t glpipe_smem_bytes(int Lmax) {
  constexpr int W = WB / (int)sizeof(T);
  return glpipe_queue_bytes<T, D>() + size_t(Lmax) * WB /* vbuf */ + size_t(Lmax) * 16 /* phi, rowacc */ +
         size_t(kGLPMaxG) * W * 8 /* psi */ + 2 * size_t(kGLPWarps) * W * 8 /* red */ + 2 * W * 8 /* sig */;
}

// Sweeps work items claimed from *claim until none is left (all threads of the
// CTA return together). Shared by the per-iteration gl_pipe_kernel and the
// persistent gl_stream_kernel.
template <typename T, bool EXACT, int D, int WB>
__device__ __forceinline__ void gl_pipe_items(const GLPipeArgs& A, unsigned* claim) {
  using V = typename Vec<T>::type;
  constexpr int VEC = Vec<T>::N;
  constexpr int W = WB / (int)sizeof(T);   // stripe width: WB (128 or 64) bytes per row
  constexpr int LPR = W / VEC;             // lanes per row (8 for 128-B stripes)
  constexpr int RPW = 32 / LPR;            // rows per warp instruction
  constexpr int RSTEP = kGLPWarps * RPW;   // rows per step
  const Params& prm = *A.prm;
  const double rho = prm.rho, thr = prm.gl_thr;
  T* X = static_cast<T*>(A.X);
  const T* C = static_cast<const T*>(A.C);

  extern __shared__ __align__(16) unsigned char glp_smem[];
  uint4* q = reinterpret_cast<uint4*>(glp_smem);
  T* vbuf = reinterpret_cast<T*>(glp_smem + glpipe_queue_bytes<T, D>());
  double* phi_s = reinterpret_cast<double*>(glp_smem + glpipe_queue_bytes<T, D>() + size_t(A.Lmax) * WB);
  double* rowacc = phi_s + A.Lmax;
  double* psi_s = rowacc + A.Lmax;          // [G][W]
  double* redq = psi_s + kGLPMaxG * W;      // [warps][W]
  double* redc = redq + kGLPWarps * W;      // [warps][W]
  double* sig = redc + kGLPWarps * W;       // [2][W]
  __shared__ unsigned s_item;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane % LPR, rsub = lane / LPR;
  const int rbase = warp * RPW + rsub;
  const int nitems = A.nseg * A.ngroups;

  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(claim, 1u);
    __syncthreads();
    const int item = (int)s_item;
    if (item >= nitems) break;
    // position-major numbering: the short tail positions are claimed last
    const int gi = item / A.nseg, si = item % A.nseg;
    const Segment sg = A.seg[si];
    const int L = (int)(sg.end - sg.begin);
    const int2 ps2 = A.pos[gi];
    const int s0 = ps2.x, Gi = ps2.y;
    const int nk = (L + RSTEP - 1) / RSTEP;
    for (int t = threadIdx.x; t < L; t += kGLPThreads) {
      phi_s[t] = __ldcg(A.phi + sg.begin + t);
      rowacc[t] = 0.0;
    }
    for (int t = threadIdx.x; t < Gi * W; t += kGLPThreads) {
      const long long col = (long long)(s0 + t / W) * W + t % W;
      psi_s[t] = col < A.ld ? __ldcg(A.psi + col) : 0.0;
    }
    __syncthreads();

    auto slot = [&](int st, int k) -> uint4* { return q + ((size_t)(st * 2 + k) * kGLPThreads + threadIdx.x); };
    // phase-1 issue cursor (stripe ij, step ik), D-1 row steps ahead of use
    int ij = 0, ik = 0;
    auto issue_next = [&](int st) {
      if (ij < Gi) {
        const int r = rbase + ik * RSTEP;
        const long long col = (long long)(s0 + ij) * W + sub * VEC;
        if (r < L && col < A.ld) {
          const long long off = (sg.begin + r) * A.ld + col;
          cp_async16(slot(st, 0), X + off);
          cp_async16(slot(st, 1), C + off);
        }
        if (++ik == nk) {
          ik = 0;
          ++ij;
        }
      }
      cp_async_commit();
    };
#pragma unroll
    for (int d = 0; d < D - 1; ++d) issue_next(d);
    int st = 0;

    double cs[VEC];
    for (int j = 0; j <= Gi; ++j) {
      const bool ph1 = j < Gi, ph2 = j > 0;
      const long long col1 = (long long)(s0 + j) * W + sub * VEC;      // phase-1 columns
      const long long col2 = col1 - W;                                   // phase-2 columns
      const bool ok1 = ph1 && col1 < A.ld, ok2 = ph2 && col2 < A.ld;
      double ps[VEC], sc[VEC], sq[VEC];
      float sc32[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        ps[e] = ph1 ? psi_s[j * W + sub * VEC + e] : 0.0;
        sc[e] = ph2 ? sig[((j - 1) & 1) * W + sub * VEC + e] : 0.0;
        sc32[e] = (float)sc[e];
        sq[e] = 0.0;
        cs[e] = 0.0;
      }
      for (int k = 0; k < nk; ++k) {
        const int r = rbase + k * RSTEP;
        const bool valid = r < L;
        T* vrow = vbuf + (size_t)r * W + sub * VEC;
        if (ph2) {  // stripe j-1: X = v * sigma, sums
          double rs = 0.0;
          if (valid && ok2) {
            if constexpr (EXACT) {
              double v[VEC], o[VEC];
              unpack(*reinterpret_cast<const V*>(vrow), v);
#pragma unroll
              for (int e = 0; e < VEC; ++e) {
                const double nx = sg.grouped ? __dmul_rn(v[e], sc[e]) : v[e];
                o[e] = nx;
                cs[e] += nx;
                rs += nx;
              }
              *reinterpret_cast<V*>(X + (sg.begin + r) * A.ld + col2) = pack<T>(o);
            } else {
              // fp32 storage: the staged v is fp32 already, scale in fp32 (<= 1
              // ulp from rounding v * sigma in fp64) and widen once for the sums
              V vv = *reinterpret_cast<const V*>(vrow);
              float* vf = reinterpret_cast<float*>(&vv);
#pragma unroll
              for (int e = 0; e < VEC; ++e) {
                if (sg.grouped) vf[e] = __fmul_rn(vf[e], sc32[e]);
                const double nx = vf[e];
                cs[e] += nx;
                rs += nx;
              }
              *reinterpret_cast<V*>(X + (sg.begin + r) * A.ld + col2) = vv;
            }
          }
#pragma unroll
          for (int o = 1; o < LPR; o <<= 1) rs += __shfl_xor_sync(0xffffffffu, rs, o);
          if (sub == 0 && valid) rowacc[r] += rs;
        }
        if (ph1) {  // stripe j: v = [((X - rho C) + phi) + psi]_+ staged in the slot just freed
          issue_next(st == 0 ? D - 1 : st - 1);
          cp_async_wait<D - 1>();
          if (valid && ok1) {
            const double ph = phi_s[r];
            double x[VEC], c[VEC], o[VEC];
            unpack(*reinterpret_cast<const V*>(slot(st, 0)), x);
            unpack(*reinterpret_cast<const V*>(slot(st, 1)), c);
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
              const double val = EXACT ? __dadd_rn(__dadd_rn(__dsub_rn(x[e], __dmul_rn(rho, c[e])), ph), ps[e])
                                       : (fma(-rho, c[e], x[e]) + ph) + ps[e];
              const double v = clamp0(val);
              o[e] = v;
              sq[e] += v * v;
            }
            *reinterpret_cast<V*>(vrow) = pack<T>(o);
          }
          st = (st + 1 == D) ? 0 : st + 1;
        }
      }
      // fold: ||v||^2 of stripe j (-> sigma_j) and the column sums of stripe j-1
#pragma unroll
      for (int e = 0; e < VEC; ++e)
#pragma unroll
        for (int o = LPR; o < 32; o <<= 1) {
          sq[e] += __shfl_xor_sync(0xffffffffu, sq[e], o);
          cs[e] += __shfl_xor_sync(0xffffffffu, cs[e], o);
        }
      if (rsub == 0) {
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          redq[warp * W + sub * VEC + e] = sq[e];
          redc[warp * W + sub * VEC + e] = cs[e];
        }
      }
      __syncthreads();
      if (threadIdx.x < W) {
        const int w = threadIdx.x;
        if (ph1) {
          double s = 0.0;
#pragma unroll
          for (int u = 0; u < kGLPWarps; ++u) s += redq[u * W + w];
          const double nrm = sqrt(s);  // regularizers.cpp:90-96
          sig[(j & 1) * W + w] = !sg.grouped ? 1.0
                                 : (nrm <= thr) ? 0.0
                                                : (EXACT ? __dsub_rn(1.0, __ddiv_rn(thr, nrm)) : 1.0 - thr / nrm);
        }
        if (ph2) {
          const long long col = (long long)(s0 + j - 1) * W + w;
          if (col < A.ld) {
            double s = 0.0;
#pragma unroll
            for (int u = 0; u < kGLPWarps; ++u) s += redc[u * W + w];
            st_hint(A.colpart + (long long)si * A.ld + col, s, policy_evict_last());
          }
        }
      }
      __syncthreads();
    }
    cp_async_wait<0>();
    for (int t = threadIdx.x; t < L; t += kGLPThreads)
      st_hint(A.rowpart + (sg.begin + t) * (long long)A.ngroups + gi, rowacc[t], policy_evict_last());
    __syncthreads();  // rowacc / phi_s / s_item reused by the next item
  }
}

template <typename T, bool EXACT, int D, int WB>
__global__ void __launch_bounds__(kGLPThreads, 1) gl_pipe_kernel(GLPipeArgs A) {
  Ctl* ctl = A.ctl;
  if (ctl->done) return;  // grid-uniform
  gl_pipe_items<T, EXACT, D, WB>(A, &ctl->gl_ctr);
  // the last CTA out resets the claim counter for the next launch
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&ctl->gl_done, 1u) == gridDim.x - 1) {
      ctl->gl_ctr = 0;
      ctl->gl_done = 0;
      __threadfence();
    }
  }
}

}  // namespace otdrk

namespace otdrk {

// ---------------------------------------------------------------------------
// Persistent group-lasso solve: the whole solve (or a step(k) run) in ONE
// cooperative launch of one 512-thread CTA per SM, like stream_kernel
// (otdr_stream.cuh) but with the pipelined GL sweep as phase A:
//   A  gl_pipe_items: rowpart[row][position], colpart[segment][col]
//   -- grid barrier --
//   B  row folds (warp per row, position order) -> r, (sum r, sum r^2, sum R)
//      column folds (thread per column, segment order) -> S_j; single GPU:
//      s = S - q and sum s^2; row-sharded: S_j stored to every rank (NVLink)
//   -- grid barrier --
//   C  scalar folds in a fixed order (every CTA, identical), the peer exchange
//      when sharded, the recurrence and the stopping logic (solver.cpp:179-235)
struct GLStreamArgs {
  GLPipeArgs g;
  double* phi;
  double* psi;
  double* a;
  double* b;
  double* r;
  double* s;
  const double* p;
  const double* q;
  double* part;           // [P][4]
  long long m_glob, n;
  double* const* peers;   // nullptr: single GPU
  double* rbuf;
  unsigned long long* xep;
  int rank, nranks;
  long long iters;        // raw mode (prm.solving == 0)
};

template <typename T, bool EXACT, int D, int WB>
__global__ void __launch_bounds__(kGLPThreads, 1) gl_stream_kernel(GLStreamArgs A) {
  constexpr int NT = kGLPThreads, NW = kGLPWarps;
  Ctl* ctl = A.g.ctl;
  if (ctl->done) return;  // grid-uniform
  const Params& prm = *A.g.prm;
  __shared__ double sred[NW];
  __shared__ double bc[4];
  const int c = (int)blockIdx.x, P = (int)gridDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long m = A.g.m, n = A.n;
  const long long gwarp = (long long)c * NW + warp, nwarps = (long long)P * NW;
  const long long gtid = (long long)c * NT + threadIdx.x, nthr = (long long)P * NT;
  const double dm = (double)A.m_glob, dn = (double)n, mn = (double)(A.m_glob + n);
  const bool peer = A.peers != nullptr;
  const int G = A.g.ngroups;
  long long k = ctl->k;
  double theta = ctl->theta[k & 1];
  double best = ctl->best;
  long long last_imp = ctl->last_improvement;
  const long long k0 = ctl->k0;
  long long it = 0;
  const unsigned long long ebase = peer ? *A.xep : 0ull;
  unsigned long long epoch = ebase + 1;

  auto bsum = [&](double v) -> double {  // fixed-order block sum, valid in thread 0
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) sred[warp] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
      for (int i = 0; i < NW; ++i) t += sred[i];
    return t;
  };

  for (;;) {
    // ---- A. pipelined group-lasso sweep
    gl_pipe_items<T, EXACT, D, WB>(A.g, &ctl->gl_ctr);
    grid_barrier(&ctl->bar_gls);

    // ---- B. row folds and column folds
    double sr = 0.0, sr2 = 0.0, sR = 0.0, ssq = 0.0;
    for (long long i0 = gwarp * 4; i0 < m; i0 += nwarps * 4) {
      double R[4] = {0.0, 0.0, 0.0, 0.0};
      for (int t = lane; t < G; t += 32) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i0 + u < m) R[u] += __ldcg(A.g.rowpart + (i0 + u) * G + t);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        R[u] = warp_sum(R[u]);
        if (lane == 0 && i0 + u < m) {
          const double ri = R[u] - A.p[i0 + u];
          A.r[i0 + u] = ri;
          sr += ri;
          sr2 += ri * ri;
          sR += R[u];
        }
      }
    }
    const int par = int(epoch & 1);
    for (long long j = gtid; j < n; j += nthr) {
      double S = 0.0;
      for (int sg = 0; sg < A.g.nseg; ++sg) S += __ldcg(A.g.colpart + (long long)sg * A.g.ld + j);
      if (peer) {
        for (int rr = 0; rr < A.nranks; ++rr) xslot(A.peers[rr], par, A.rank, A.nranks, n)[j] = S;
      } else {
        const double sj = __dsub_rn(S, A.q[j]);
        A.s[j] = sj;
        ssq += sj * sj;
      }
    }
    {
      const double t1 = bsum(sr), t2 = bsum(sr2), t3 = bsum(sR), t4 = bsum(ssq);
      if (threadIdx.x == 0) {
        if (peer) __threadfence_system();  // this CTA's peer stores (cumulative through bar.sync)
        A.part[c * 4 + 0] = t1;
        A.part[c * 4 + 1] = t2;
        A.part[c * 4 + 2] = t3;
        A.part[c * 4 + 3] = t4;
      }
    }
    grid_barrier(&ctl->bar_gls);

    // ---- C. scalar folds, exchange, recurrence, stopping
    if (c == 0 && threadIdx.x == 0) ctl->gl_ctr = 0;  // every CTA is past its last claim
    if (peer) {
      if (c == 0 && warp < 3) {
        const double u = warp_fold_strided(A.part + warp, P, 4);
        if (lane == 0)
          for (int rr = 0; rr < A.nranks; ++rr) xslot(A.peers[rr], par, A.rank, A.nranks, n)[n + warp] = u;
      }
      if (c == 0) {
        __syncthreads();
        if (threadIdx.x == 0) xpublish(A.peers, A.rank, A.nranks, n, epoch);
      }
      if (threadIdx.x == 0) xwait(A.rbuf, A.nranks, n, epoch);
      __syncthreads();
      if (warp < 3 && lane == 0) {
        double u = 0.0;
        for (int rr = 0; rr < A.nranks; ++rr) u += __ldcg(xslot(A.rbuf, par, rr, A.nranks, n) + n + warp);
        bc[warp] = u;
      }
      __syncthreads();
      const double eta_p = __ddiv_rn(bc[0], mn);
      const double shift_p = __dsub_rn(2.0 * eta_p, theta);
      double ss = 0.0;
      for (long long j = gtid; j < n; j += nthr) {
        double S = 0.0;
        for (int rr = 0; rr < A.nranks; ++rr) S += __ldcg(xslot(A.rbuf, par, rr, A.nranks, n) + j);
        const double sj = __dsub_rn(S, A.q[j]), bj = A.b[j];
        A.s[j] = sj;
        ss += sj * sj;
        A.psi[j] = __ddiv_rn(__dadd_rn(__dsub_rn(bj, 2.0 * sj), shift_p), dm);
        A.b[j] = __dsub_rn(bj, sj);
      }
      for (long long i = gtid; i < m; i += nthr) {
        const double ri = __ldcg(A.r + i), ai = A.a[i];
        A.phi[i] = __ddiv_rn(__dadd_rn(__dsub_rn(ai, 2.0 * ri), shift_p), dn);
        A.a[i] = __dsub_rn(ai, ri);
      }
      const double t4 = bsum(ss);
      if (threadIdx.x == 0) A.part[c * 4 + 3] = t4;
      grid_barrier(&ctl->bar_gls);  // phi / psi / s complete, ssq partials visible
      if (warp == 0) {
        const double u = warp_fold_strided(A.part + 3, P, 4);
        if (lane == 0) bc[3] = u;
      }
      __syncthreads();
    } else {
      if (warp < 4) {
        const double u = warp_fold_strided(A.part + warp, P, 4);
        if (lane == 0) bc[warp] = u;
      }
      __syncthreads();
      const double eta_l = __ddiv_rn(bc[0], mn);
      const double shift_l = __dsub_rn(2.0 * eta_l, theta);
      for (long long i = gtid; i < m; i += nthr) {
        const double ri = __ldcg(A.r + i), ai = A.a[i];
        A.phi[i] = __ddiv_rn(__dadd_rn(__dsub_rn(ai, 2.0 * ri), shift_l), dn);
        A.a[i] = __dsub_rn(ai, ri);
      }
      for (long long j = gtid; j < n; j += nthr) {
        const double sj = __ldcg(A.s + j), bj = A.b[j];
        A.psi[j] = __ddiv_rn(__dadd_rn(__dsub_rn(bj, 2.0 * sj), shift_l), dm);
        A.b[j] = __dsub_rn(bj, sj);
      }
    }
    const double eta = __ddiv_rn(bc[0], mn);
    const double nr2 = sqrt(bc[1]), ns2 = sqrt(bc[3]);
    const double rp = (nr2 < ns2) ? ns2 : nr2;  // std::max semantics (solver.cpp:179)
    theta = __dsub_rn(theta, eta);
    ++k;
    ++it;
    ++epoch;
    const long long kk = k - k0;
    bool done = false, want_cert = false;
    int term = TERM_MAXITER;
    if (prm.solving) {
      if (!(rp - rp == 0.0)) {  // solver.cpp:181-185
        done = true;
        term = TERM_NONFINITE;
      } else {
        if (rp < best * (1.0 - 1e-14)) {  // solver.cpp:200-203
          best = rp;
          last_imp = kk;
        }
        const bool at_check = (kk % prm.check_every) == 0;
        if (at_check && rp <= prm.tol_primal && prm.has_tol_gap) {
          // tol_gap: the launch ends here; the host runs the certificate
          // kernels, whose finisher applies converged / stalled / max_iter
          want_cert = true;
        } else if (at_check && rp <= prm.tol_primal) {
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
    } else if (it >= A.iters) {
      done = true;
    }
    if (done || want_cert) {
      if (c == 0 && threadIdx.x == 0) {
        ctl->k = k;
        ctl->theta[k & 1] = theta;
        ctl->eta = eta;
        ctl->r_primal = rp;
        ctl->best = best;
        ctl->last_improvement = last_imp;
        ctl->want_cert = want_cert ? 1 : 0;
        if (prm.solving && done) {
          ctl->done = 1;
          ctl->termination = term;
        }
        if (peer) *A.xep = epoch - 1;
      }
      break;
    }
    if (!peer) grid_barrier(&ctl->bar_gls);  // phi / psi complete before the next sweep
  }
}

}  // namespace otdrk
