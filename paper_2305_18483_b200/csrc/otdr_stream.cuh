// otdr_stream.cuh -- persistent streaming solve loop for plans that live in
// HBM (zero / quadratic regularizer; single GPU or row-sharded).
//
// One cooperative launch runs many DR iterations (solver.cpp:95-102 + :23-38):
// P = SMs x 2 co-resident CTAs sweep the plan every iteration, so there are
// no per-iteration launches and no separate reduce / update kernels.
//
// Work split. The plan is cut into tiles of rows x 256 columns, numbered
// stripe-major (all row ranges of stripe 0, then stripe 1, ...); the last
// stripes use short tiles so the sweep ends with a fine-grained tail. CTAs
// claim tiles from a per-iteration atomic counter: a static equal split was
// measured to leave a 350 us spread of CTA finish times per sweep on B200 at
// 20000^2, dynamic claiming lets fast CTAs take more tiles.
//
// One iteration:
//   A  sweep the claimed tiles: X <- prox([((X - rho C) + phi_i) + psi_j]_+)
//      with every thread streaming its own 16-byte chunks of X, C and phi
//      through a private cp.async queue; row partials rowpart[row][stripe]
//      (warp butterfly), per-tile column partials (registers -> fixed-order
//      cross-warp smem sum -> colpart[tile]: one slot per tile, so the fold
//      order does not depend on which CTA swept it). The CTA completing a
//      stripe's last tile folds its column partials (tile order): single GPU
//      s = S - q and the stripe's sum of s^2; row-sharded: S stored into every
//      rank's receive buffer (NVLink) while the sweep goes on
//   -- grid barrier --
//   B  row folds (warp per row, stripe order): r = R - p, partial sums of r,
//      r^2, R; one (sr, sr2, sR) record per CTA
//   -- grid barrier --
//   C  every CTA folds the P records in the same fixed order -> identical eta,
//      shift, r_primal and stopping decision everywhere (row-sharded: after
//      the epoch-flag exchange, folding the ranks' contributions in rank
//      order); phi/a (thread per row), psi/b (thread per column); the solve
//      loop's stopping logic (solver.cpp:179-235)
//   -- grid barrier (only when continuing) --
// Cross-CTA data (phi, psi, r, partials) is read with ld.global.cg (L2), so
// no stale L1 line survives a barrier; X and C tiles are owned by one CTA.
#pragma once
#include "otdr_kernels.cuh"

namespace otdrk {

struct StreamArgs {
  void* X;
  const void* C;
  double* phi;
  double* a;
  double* r;
  const double* p;
  double* psi;
  double* b;
  double* s;
  const double* q;
  double* rowpart;        // [m][stripes]
  double* colpart;        // [ntiles][TN] one slot per tile
  const int* sfirst;      // [stripes + 1] first tile of each stripe (tiles: see `tiles`)
  unsigned* scnt;         // [stripes] tiles completed this sweep (zero between sweeps)
  double* sspart;         // [stripes] sum of s_j^2 over the stripe's columns
  double* part;           // [P][4]
  Ctl* ctl;
  const Params* prm;
  long long m, n, ld;
  int stripes, ntiles;
  long long iters;        // raw mode (prm.solving == 0): iterations to run
  unsigned long long* tstamp;  // optional phase timestamps [kTraceIters][P + 12] (debug)
  // Row-sharded runs: the exchange goes over peer memory (NVLink P2P) inside
  // this kernel. peers[r] = rank r's receive buffer (mapped here), layout
  // [2 parities][nranks][n + 4] doubles then [2][nranks] u64 flags.
  long long m_glob;
  double* const* peers;   // nullptr: single GPU
  double* rbuf;           // this rank's receive buffer (== peers[rank])
  unsigned long long* xep;  // exchange epoch (monotonic, identical on every rank)
  int rank, nranks;
  // tile table {stripe, r0, r1, 0}, stripe-major; stripes >= fin_first are the
  // final wave of short tiles, folded in phase B (one stripe per CTA)
  const int4* tiles;
  int fin_first;
};

// Stripe-completion counter: gpu-scope acq_rel atomic by one thread after a
// CTA barrier. The release half is cumulative over the CTA's stores that
// bar.sync ordered before it (the colpart partials of the tile), the acquire
// half over every other CTA's released partials -- so no per-thread
// __threadfence (a full fence plus an L1 invalidate) is needed on either
// side; the folding CTA reads the partials with ld.global.cg (L2).
__device__ __forceinline__ unsigned atomic_add_acq_rel_gpu(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// ---- peer-memory exchange helpers (system scope)
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double* xslot(double* buf, int par, int src, int nranks, long long n) {
  return buf + ((long long)par * nranks + src) * (n + 4);
}
__device__ __forceinline__ unsigned long long* xflag(double* buf, int par, int src, int nranks,
                                                     long long n) {
  return reinterpret_cast<unsigned long long*>(buf + 2LL * nranks * (n + 4)) + par * nranks + src;
}
// publish this rank's contribution of epoch e: caller has fenced its data
// stores at system scope; one thread per CTA-group calls this.
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void xpublish(double* const* peers, int rank, int nranks, long long n,
                                         unsigned long long e) {
  // one system-scope fence (cumulative over the CTA's and, through the grid
  // barriers, the grid's prior peer stores), then relaxed flag stores
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  for (int r = 0; r < nranks; ++r) st_relaxed_sys(xflag(peers[r], int(e & 1), rank, nranks, n), e);
}
// Fixed-order fold of count values (stride apart) by one warp: every load is
// issued before any add (one L2 round trip for count <= 32 * 16).
__device__ __forceinline__ double warp_fold_strided(const double* p, int count, int stride) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int base = 0; base < count; base += 32 * 16) {
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int i = base + u * 32 + lane;
      v[u] = i < count ? __ldcg(p + (long long)i * stride) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) s += v[u];
  }
  return warp_sum(s);
}
__device__ __forceinline__ void xwait(double* rbuf, int nranks, long long n, unsigned long long e) {
  for (int r = 0; r < nranks; ++r) {
    const unsigned long long* f = xflag(rbuf, int(e & 1), r, nranks, n);
    while (ld_acquire_sys(f) < e) {
    }
  }
}
constexpr int kTraceIters = 4;

constexpr int kStreamTN = 256;

template <typename T, int REG, bool EXACT, int NV, int U>
__device__ __forceinline__ void stream_segment(const StreamArgs& A, int tile, long long stripe,
                                               long long r0, long long r1, double rho, double qd,
                                               double qinv, double (*red)[kStreamTN]) {
  using V = typename Vec<T>::type;
  constexpr int VEC = Vec<T>::N;
  static_assert(32 * VEC * NV == kStreamTN, "stripe width");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T* X = static_cast<T*>(A.X);
  const T* C = static_cast<const T*>(A.C);
  const long long col0 = stripe * kStreamTN;
  long long cols[NV];
  bool cok[NV];
  double psi_r[NV][VEC], cacc[NV][VEC];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    cols[v] = col0 + v * 32 * VEC + lane * VEC;
    cok[v] = cols[v] < A.ld;
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      psi_r[v][e] = cok[v] ? __ldcg(A.psi + cols[v] + e) : 0.0;
      cacc[v][e] = 0.0;
    }
  }
  for (long long i0 = r0 + warp; i0 < r1; i0 += (long long)kWarps * U) {
    V xv[U][NV], cv[U][NV];
    double phv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = i0 + (long long)u * kWarps;
      if (i < r1) {
        phv[u] = __ldcg(A.phi + i);
        const V* xrow = reinterpret_cast<const V*>(X + i * A.ld);
        const V* crow = reinterpret_cast<const V*>(C + i * A.ld);
#pragma unroll
        for (int v = 0; v < NV; ++v)
          if (cok[v]) {
            xv[u][v] = ld_rw(xrow + cols[v] / VEC);
            cv[u][v] = ld_ro(crow + cols[v] / VEC);
          }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = i0 + (long long)u * kWarps;
      if (i >= r1) break;  // warp-uniform
      double rs = 0.0;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        if (!cok[v]) continue;
        double x[VEC], cc[VEC], o[VEC];
        unpack(xv[u][v], x);
        unpack(cv[u][v], cc);
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          // ((X - rho C) + phi) + psi, clamp (solver.cpp:97-99), prox
          const double val = EXACT ? __dadd_rn(__dadd_rn(__dsub_rn(x[e], __dmul_rn(rho, cc[e])), phv[u]),
                                               psi_r[v][e])
                                   : (fma(-rho, cc[e], x[e]) + phv[u]) + psi_r[v][e];
          double nx = clamp0(val);
          if (REG == REG_QUAD) nx = EXACT ? div_rn_by(nx, qd, qinv) : nx * qinv;  // regularizers.cpp:54
          o[e] = nx;
          cacc[v][e] += nx;
          rs += nx;
        }
        reinterpret_cast<V*>(X + i * A.ld)[cols[v] / VEC] = pack<T>(o);
      }
      rs = warp_sum(rs);
      if (lane == 0) A.rowpart[i * (long long)A.stripes + stripe] = rs;
    }
  }
  // column partial of this segment: fixed-order cross-warp sum
  __syncthreads();  // red reused across segments
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int e = 0; e < VEC; ++e) red[warp][v * 32 * VEC + lane * VEC + e] = cacc[v][e];
  __syncthreads();
  double* dst = A.colpart + (long long)tile * kStreamTN;
  for (int t = threadIdx.x; t < kStreamTN; t += kThreads) {
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) sum += red[w][t];
    dst[t] = sum;
  }
}

// cp.async (LDGSTS) variant: every thread keeps a private D-deep queue of its
// own 16-byte chunks (X, C of one row, plus the row's phi) in shared memory,
// so D rows per warp are always in flight without holding them in registers.
// Each thread reads back only what it copied itself: no barriers, only
// cp.async.wait_group. .cg copies bypass L1 (phi changes every iteration).
// L2 policies: the plan streams (C, X) use the default policy -- marking them
// evict_first measured 1.4-6 % slower once X lives in compressible memory
// (profiles/r01g_stream_policy.txt); the row / column partials are re-read
// after the sweep (evict_last), so they survive the 4.8 GB that streams past.
__device__ __forceinline__ unsigned long long policy_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_hint(double* ptr, double v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(ptr), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint(float4* ptr, float4 v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(ptr), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_hint(double2* ptr, double2 v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(ptr), "d"(v.x), "d"(v.y),
               "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, unsigned long long pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(smem))),
               "l"(gmem), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <typename T, int NV, int D>
__host__ __device__ constexpr size_t stream_async_smem() {
  return size_t(D) * size_t(2 * NV + 1) * kThreads * 16;
}

template <typename T, int REG, bool EXACT, int NV, int D, int mode = MODE_NORMAL>
__device__ __forceinline__ void stream_segment_async(const StreamArgs& A, int tile, long long stripe,
                                                     long long r0, long long r1, double rho,
                                                     double qd, double qinv,
                                                     double (*red)[kStreamTN], uint4* q) {
  using V = typename Vec<T>::type;
  constexpr int VEC = Vec<T>::N;
  constexpr int NS = 2 * NV + 1;  // 16-byte slots per row: X[NV], C[NV], phi
  static_assert(32 * VEC * NV == kStreamTN, "stripe width");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T* X = static_cast<T*>(A.X);
  const T* C = static_cast<const T*>(A.C);
  const long long col0 = stripe * kStreamTN;
  long long cols[NV];
  bool cok[NV];
  double psi_r[NV][VEC], cacc[NV][VEC];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    cols[v] = col0 + v * 32 * VEC + lane * VEC;
    cok[v] = cols[v] < A.ld;
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      psi_r[v][e] = cok[v] ? __ldcg(A.psi + cols[v] + e) : 0.0;
      cacc[v][e] = 0.0;
    }
  }
  const unsigned long long plast = policy_evict_last();
  auto slot = [&](int st, int k) -> uint4* { return q + ((size_t)(st * NS + k) * kThreads + threadIdx.x); };
  auto issue = [&](long long i, int st) {
    if (i < r1) {
      const T* xrow = X + i * A.ld;
      const T* crow = C + i * A.ld;
#pragma unroll
      for (int v = 0; v < NV; ++v)
        if (cok[v]) {
          // default L2 policy (evict_first on these streams measured 1.4-6 %
          // slower: profiles/r01g_stream_policy.txt)
          cp_async16(slot(st, v), xrow + cols[v]);
          if (mode != MODE_ODD) cp_async16(slot(st, NV + v), crow + cols[v]);  // odd: B only
        }
      cp_async16(slot(st, 2 * NV), A.phi + (i & ~1LL));
    }
    cp_async_commit();
  };
  const long long step = kWarps;
  long long i = r0 + warp;
#pragma unroll
  for (int d = 0; d < D - 1; ++d) issue(i + d * step, d);
  int st = 0;
  for (; i < r1; i += step) {
    issue(i + (D - 1) * step, (st + D - 1) % D);
    cp_async_wait<D - 1>();
    const double2 ph2 = *reinterpret_cast<const double2*>(slot(st, 2 * NV));
    const double ph = (i & 1) ? ph2.y : ph2.x;
    double rs = 0.0;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if (!cok[v]) continue;
      double x[VEC], cc[VEC], o[VEC];
      unpack(*reinterpret_cast<const V*>(slot(st, v)), x);
      if (mode != MODE_ODD) unpack(*reinterpret_cast<const V*>(slot(st, NV + v)), cc);
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        double val;
        if (mode == MODE_ODD)  // B + phi + psi (solver.cpp:170-172): the buffer holds B = X - rho C
          val = EXACT ? __dadd_rn(__dadd_rn(x[e], ph), psi_r[v][e]) : (x[e] + ph) + psi_r[v][e];
        else
          val = EXACT ? __dadd_rn(__dadd_rn(__dsub_rn(x[e], __dmul_rn(rho, cc[e])), ph), psi_r[v][e])
                      : (fma(-rho, cc[e], x[e]) + ph) + psi_r[v][e];
        double nx = clamp0(val);
        if (REG == REG_QUAD) nx = EXACT ? div_rn_by(nx, qd, qinv) : nx * qinv;
        // even step of the fused path stores B = (-rho C) + X_{k+1} (solver.cpp:162,167)
        o[e] = mode == MODE_EVEN ? (EXACT ? __dadd_rn(-__dmul_rn(rho, cc[e]), nx) : nx - rho * cc[e]) : nx;
        cacc[v][e] += nx;
        rs += nx;
      }
      reinterpret_cast<V*>(X + i * A.ld)[cols[v] / VEC] = pack<T>(o);
    }
    rs = warp_sum(rs);
    if (lane == 0) st_hint(A.rowpart + i * (long long)A.stripes + stripe, rs, plast);
    st = (st + 1 == D) ? 0 : st + 1;
  }
  cp_async_wait<0>();  // drain the (empty) tail groups before the queue is reused
  __syncthreads();
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int e = 0; e < VEC; ++e) red[warp][v * 32 * VEC + lane * VEC + e] = cacc[v][e];
  __syncthreads();
  double* dst = A.colpart + (long long)tile * kStreamTN;
  for (int t = threadIdx.x; t < kStreamTN; t += kThreads) {
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) sum += red[w][t];
    st_hint(dst + t, sum, plast);
  }
}

// The CTA that completes the last tile of a stripe folds the stripe's column
// partials in tile order: S_j -> s_j = S_j - q_j, and the stripe's sum of
// s_j^2 (column folds leave the critical path except for the last stripes).
__device__ __forceinline__ void stream_stripe_done(const StreamArgs& A, long long stripe,
                                                   double* sred, bool* s_last, int par) {
  if (stripe >= A.fin_first) {  // final-wave stripe: folded in phase B
    __syncthreads();            // (the partial staging is reused by the next tile)
    return;
  }
  __syncthreads();  // the CTA's colpart stores before thread 0's release
  if (threadIdx.x == 0) {
    const unsigned need = (unsigned)(A.sfirst[stripe + 1] - A.sfirst[stripe]);
    *s_last = atomic_add_acq_rel_gpu(A.scnt + stripe, 1u) == need - 1;
  }
  __syncthreads();  // thread 0's acquire before every thread's ld.cg of the partials
  if (!*s_last) return;
  const long long j = stripe * kStreamTN + threadIdx.x;
  double ss = 0.0;
  if (threadIdx.x < kStreamTN && j < A.n) {
    const double* src = A.colpart + threadIdx.x;
    const int t0 = A.sfirst[stripe], t1 = A.sfirst[stripe + 1];
    double S = 0.0;
#pragma unroll 16
    for (int t = t0; t < t1; ++t) S += __ldcg(src + (long long)t * kStreamTN);
    if (A.peers) {  // local column sums to every rank's receive slot (NVLink stores)
      for (int r = 0; r < A.nranks; ++r) xslot(A.peers[r], par, A.rank, A.nranks, A.n)[j] = S;
    } else {
      const double sj = __dsub_rn(S, A.q[j]);
      A.s[j] = sj;
      ss = sj * sj;
    }
  }
  if (A.peers) {
    // one system-scope fence per completed stripe, after the CTA's stores
    // (bar.sync orders them before thread 0's fence; the flag publish after
    // the grid barriers is a release at system scope)
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      A.scnt[stripe] = 0;
    }
    return;
  }
  const double tot = block_sum(ss, sred);
  if (threadIdx.x == 0) {
    A.sspart[stripe] = tot;
    A.scnt[stripe] = 0;  // every tile of this stripe is done for this iteration
  }
}


// Phase-B fold of one final-wave stripe by a whole CTA (NT >= 256 threads):
// the same fold as stream_stripe_done (tile order), after the grid barrier
// made every tile's column partials visible.
template <int NT>
__device__ __forceinline__ void stream_fin_fold(const StreamArgs& A, long long stripe, double* sred,
                                                int par, double* scratch) {
  // warp w sums tiles w, w + NW, ... of every column (independent loads in
  // flight), then the NW partials are added in warp order: a fixed order.
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t0 = A.sfirst[stripe], t1 = A.sfirst[stripe + 1];
  double acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.0;
  for (int t = t0 + warp; t < t1; t += NW) {
    const double* src = A.colpart + (long long)t * kStreamTN + lane;
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] += __ldcg(src + 32 * e);
  }
  __syncthreads();  // scratch (NW x 256 doubles) free
#pragma unroll
  for (int e = 0; e < 8; ++e) scratch[warp * kStreamTN + 32 * e + lane] = acc[e];
  __syncthreads();
  const long long j = stripe * kStreamTN + threadIdx.x;
  double ss = 0.0;
  if (threadIdx.x < kStreamTN && j < A.n) {
    double Ssum = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) Ssum += scratch[w * kStreamTN + threadIdx.x];
    // scratch may be a TMA ring: order these generic accesses before the
    // next iteration's async-proxy (TMA) writes into it
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (A.peers) {
      for (int r = 0; r < A.nranks; ++r) xslot(A.peers[r], par, A.rank, A.nranks, A.n)[j] = Ssum;
    } else {
      const double sj = __dsub_rn(Ssum, A.q[j]);
      A.s[j] = sj;
      ss = sj * sj;
    }
  }
  if (A.peers) {
    __syncthreads();
    if (threadIdx.x == 0) __threadfence_system();
    return;
  }
  const double tot = block_sum_n<NT / 32>(ss, sred);
  if (threadIdx.x == 0) A.sspart[stripe] = tot;
}

// Loop state of a persistent streaming solve (identical in every CTA).
struct StreamLoop {
  long long k, last_imp, k0, it;
  double theta, best;
  unsigned long long epoch;
  int shifted;
};

// Phases B and C of one DR iteration of the persistent streaming kernels,
// after the sweep (phase A) of every CTA: grid barrier, row folds, scalar
// folds (fixed order: every CTA derives the same eta, shift, r_primal and
// stopping decision), the recurrence (solver.cpp:23-38) and the solve loop's
// stopping logic (solver.cpp:179-235). NT threads per CTA, all of which call
// this. Returns true when the launch ends (state written to ctl).
template <int NT, typename Stamp>
__device__ __forceinline__ bool stream_finish_iteration(const StreamArgs& A, const Params& prm,
                                                        StreamLoop& L, double* sred, double* bc,
                                                        unsigned long long* bar, Stamp&& stamp,
                                                        double* scratch) {
  Ctl* ctl = A.ctl;
  const int c = (int)blockIdx.x, P = (int)gridDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long m = A.m, n = A.n;
  const long long gwarp = (long long)c * (NT / 32) + warp, nwarps = (long long)P * (NT / 32);
  const long long gtid = (long long)c * NT + threadIdx.x, nthr = (long long)P * NT;
  const double dm = (double)A.m_glob, dn = (double)n, mn = (double)(A.m_glob + n);
  const long long k0 = L.k0;
  const bool peer = A.peers != nullptr;
    grid_barrier(bar);
    if (c < A.stripes - A.fin_first)  // final-wave stripes, one per CTA
      stream_fin_fold<NT>(A, A.fin_first + c, sred, int(L.epoch & 1), scratch);
    stamp(P + 1);

    // ---- B. row folds (warp per row, stripe order) and column folds (CTA order)
    double sr = 0.0, sr2 = 0.0, sR = 0.0;
    for (long long i0 = gwarp * 4; i0 < m; i0 += nwarps * 4) {  // 4 rows per warp trip
      double R[4] = {0.0, 0.0, 0.0, 0.0};
      for (int t = lane; t < A.stripes; t += 32) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i0 + u < m) R[u] += __ldcg(A.rowpart + (i0 + u) * A.stripes + t);
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
    stamp(P + 5);
    stamp(P + 6);
    {
      const double t1 = block_sum_n<NT / 32>(sr, sred);
      const double t2 = block_sum_n<NT / 32>(sr2, sred);
      const double t3 = block_sum_n<NT / 32>(sR, sred);
      if (threadIdx.x == 0) {
        A.part[c * 4 + 0] = t1;
        A.part[c * 4 + 1] = t2;
        A.part[c * 4 + 2] = t3;
      }
    }
    stamp(P + 2);
    grid_barrier(bar);
    stamp(P + 3);

    // ---- C. scalar folds (same order in every CTA), recurrence, stopping
    double pre_r = 0.0, pre_a = 0.0, pre_s = 0.0, pre_b = 0.0;
    if (peer) {
      if (gtid < m) {  // row operands in flight during the exchange
        pre_r = __ldcg(A.r + gtid);
        pre_a = A.a[gtid];
      }
      // exchange: CTA 0 sends this rank's (sum r, sum r^2, sum R) and the
      // L.epoch flags; every CTA waits for all ranks, then folds in rank order
      if (c == 0 && warp < 3) {
        const double u = warp_fold_strided(A.part + warp, P, 4);
        if (lane == 0)
          for (int r = 0; r < A.nranks; ++r)
            xslot(A.peers[r], int(L.epoch & 1), A.rank, A.nranks, n)[n + warp] = u;
      }
      if (c == 0) {
        __syncthreads();
        if (threadIdx.x == 0) xpublish(A.peers, A.rank, A.nranks, n, L.epoch);
      }
      stamp(P + 8);
      if (threadIdx.x == 0) xwait(A.rbuf, A.nranks, n, L.epoch);
      __syncthreads();
      stamp(P + 9);
      if (warp < 3) {
        double u = 0.0;
        if (lane == 0)
          for (int r = 0; r < A.nranks; ++r)
            u += __ldcg(xslot(A.rbuf, int(L.epoch & 1), r, A.nranks, n) + n + warp);
        if (lane == 0) bc[warp] = u;
      }
      __syncthreads();
      if (c == 0 && threadIdx.x == 0) ctl->tile_ctr = 0;
      const double eta_p = __ddiv_rn(bc[0], mn);
      const double shift_p = __dsub_rn(2.0 * eta_p, L.theta);
      double ssq = 0.0;
      for (long long j = gtid; j < n; j += nthr) {
        double S = 0.0;
        for (int r = 0; r < A.nranks; ++r) S += __ldcg(xslot(A.rbuf, int(L.epoch & 1), r, A.nranks, n) + j);
        const double sj = __dsub_rn(S, A.q[j]), bj = A.b[j];
        A.s[j] = sj;
        ssq += sj * sj;
        A.psi[j] = __ddiv_rn(__dadd_rn(__dsub_rn(bj, 2.0 * sj), shift_p), dm);
        A.b[j] = __dsub_rn(bj, sj);
      }
      for (long long i = gtid; i < m; i += nthr) {
        const double ri = i == gtid ? pre_r : __ldcg(A.r + i), ai = i == gtid ? pre_a : A.a[i];
        A.phi[i] = __ddiv_rn(__dadd_rn(__dsub_rn(ai, 2.0 * ri), shift_p), dn);
        A.a[i] = __dsub_rn(ai, ri);
      }
      const double t4 = block_sum_n<NT / 32>(ssq, sred);
      if (threadIdx.x == 0) A.part[c * 4 + 3] = t4;
      stamp(P + 10);
      grid_barrier(bar);  // phi / psi / s complete, ssq partials visible
      stamp(P + 11);
      if (warp == 0) {
        const double u = warp_fold_strided(A.part + 3, P, 4);
        if (lane == 0) bc[3] = u;
      }
      __syncthreads();
    } else {
      // this thread's first row / column operands are loaded while the
      // scalar folds are in flight (one L2 round trip for both)
      if (gtid < m) {
        pre_r = __ldcg(A.r + gtid);
        pre_a = A.a[gtid];
      }
      if (gtid < n) {
        pre_s = __ldcg(A.s + gtid);
        pre_b = A.b[gtid];
      }
      if (warp < 3) {
        const double u = warp_fold_strided(A.part + warp, P, 4);
        if (lane == 0) bc[warp] = u;
      } else if (warp == 3) {  // sum s^2: stripe partials in stripe order
        const double u = warp_fold_strided(A.sspart, A.stripes, 1);
        if (lane == 0) bc[3] = u;
      }
    }
    if (!peer) {
      __syncthreads();
      if (c == 0 && threadIdx.x == 0) ctl->tile_ctr = 0;  // every CTA is past its last claim
      const double eta_l = __ddiv_rn(bc[0], mn);
      const double shift_l = __dsub_rn(2.0 * eta_l, L.theta);
      for (long long i = gtid; i < m; i += nthr) {
        const double ri = i == gtid ? pre_r : __ldcg(A.r + i), ai = i == gtid ? pre_a : A.a[i];
        A.phi[i] = __ddiv_rn(__dadd_rn(__dsub_rn(ai, 2.0 * ri), shift_l), dn);
        A.a[i] = __dsub_rn(ai, ri);
      }
      for (long long j = gtid; j < n; j += nthr) {
        const double sj = j == gtid ? pre_s : __ldcg(A.s + j), bj = j == gtid ? pre_b : A.b[j];
        A.psi[j] = __ddiv_rn(__dadd_rn(__dsub_rn(bj, 2.0 * sj), shift_l), dm);
        A.b[j] = __dsub_rn(bj, sj);
      }
    }
    const double eta = __ddiv_rn(bc[0], mn);
    stamp(P + 4);
    const double nr2 = sqrt(bc[1]), ns2 = sqrt(bc[3]);
    const double rp = (nr2 < ns2) ? ns2 : nr2;  // std::max semantics (solver.cpp:179)
    L.theta = __dsub_rn(L.theta, eta);
    ++L.k;
    ++L.it;
    ++L.epoch;
    if (prm.fused) L.shifted ^= 1;
    const long long kk = L.k - k0;
    bool done = false, want_cert = false;
    int term = TERM_MAXITER;
    if (prm.solving) {
      if (!(rp - rp == 0.0)) {  // solver.cpp:181-185
        done = true;
        term = TERM_NONFINITE;
      } else {
        if (rp < L.best * (1.0 - 1e-14)) {  // solver.cpp:200-203
          L.best = rp;
          L.last_imp = kk;
        }
        const bool at_check = (kk % prm.check_every) == 0;
        if (at_check && rp <= prm.tol_primal && prm.has_tol_gap) {
          // tol_gap: the launch ends here; the host runs the certificate
          // kernels, whose finisher applies converged / stalled / max_iter
          want_cert = true;
        } else if (at_check && rp <= prm.tol_primal) {
          done = true;
          term = TERM_CONVERGED;
        } else if (kk - L.last_imp >= 10000) {  // solver.cpp:17, :232-235
          done = true;
          term = TERM_STALLED;
        } else if (kk >= prm.max_iter) {
          done = true;
          term = TERM_MAXITER;
        }
      }
    } else if (L.it >= A.iters) {
      done = true;
    }
    if (done || want_cert) {
      if (c == 0 && threadIdx.x == 0) {
        ctl->k = L.k;
        ctl->theta[L.k & 1] = L.theta;
        ctl->eta = eta;
        ctl->r_primal = rp;
        ctl->best = L.best;
        ctl->last_improvement = L.last_imp;
        ctl->want_cert = want_cert ? 1 : 0;
        if (prm.solving && done) {
          ctl->done = 1;
          ctl->termination = term;
        }
        ctl->fused_shifted = L.shifted;
        if (peer) *A.xep = L.epoch - 1;  // every CTA read the base at entry
      }
      return true;
    }
    if (!peer) grid_barrier(bar);  // phi / psi complete before the next sweep
  return false;
}

template <typename T, int REG, bool EXACT, int NV, int U, int D>
__global__ void __launch_bounds__(kThreads, 2) stream_kernel(StreamArgs A) {
  Ctl* ctl = A.ctl;
  if (ctl->done) return;  // grid-uniform
  const Params& prm = *A.prm;
  // column-partial staging: aliases the (drained) cp.async queue when there is one
  extern __shared__ __align__(16) uint4 squeue[];
  __shared__ double red_static[D > 0 ? 1 : kWarps][kStreamTN];
  double(*red)[kStreamTN] = D > 0 ? reinterpret_cast<double(*)[kStreamTN]>(squeue) : red_static;
  __shared__ double sred[kWarps];
  __shared__ double bc[4];
  const int c = (int)blockIdx.x, P = (int)gridDim.x;
  __shared__ unsigned s_tile;
  __shared__ bool s_last;

  const double rho = prm.rho, qd = prm.quad_d, qinv = prm.quad_inv;
  StreamLoop L;
  L.k = ctl->k;
  L.theta = ctl->theta[L.k & 1];
  L.best = ctl->best;
  L.last_imp = ctl->last_improvement;
  L.k0 = ctl->k0;
  L.it = 0;
  L.epoch = (A.peers != nullptr ? *A.xep : 0ull) + 1;
  // fused even/odd path (solver.cpp:127-177): the X buffer alternates
  // between X (even iterations read C) and B = X - rho C (odd ones do not)
  L.shifted = prm.fused ? ctl->fused_shifted : 0;

  auto stamp = [&](int slot) {
    if (A.tstamp && L.it < kTraceIters && threadIdx.x == 0 && (slot < P ? true : c == 0))
      A.tstamp[L.it * (P + 12) + slot] = globaltimer_ns();
  };
  for (;;) {
    stamp(P + 0);
    const int fmode = prm.fused ? (L.shifted ? MODE_ODD : MODE_EVEN) : MODE_NORMAL;
    // ---- A. sweep tiles claimed from the iteration's tile counter
    for (;;) {
      if (threadIdx.x == 0) s_tile = atomicAdd(&ctl->tile_ctr, 1u);
      __syncthreads();
      const int tile = (int)s_tile;  // the tile sweep ends with __syncthreads
      if (tile >= A.ntiles) break;
      int4 tl = A.tiles[tile];  // {stripe, r0, r1}
      if constexpr (D > 0) {
        if (fmode == MODE_EVEN)
          stream_segment_async<T, REG, EXACT, NV, D, MODE_EVEN>(A, tile, tl.x, tl.y, tl.z, rho, qd, qinv, red, squeue);
        else if (fmode == MODE_ODD)
          stream_segment_async<T, REG, EXACT, NV, D, MODE_ODD>(A, tile, tl.x, tl.y, tl.z, rho, qd, qinv, red, squeue);
        else
          stream_segment_async<T, REG, EXACT, NV, D>(A, tile, tl.x, tl.y, tl.z, rho, qd, qinv, red, squeue);
      } else {
        stream_segment<T, REG, EXACT, NV, U>(A, tile, tl.x, tl.y, tl.z, rho, qd, qinv, red);
      }
      stream_stripe_done(A, tl.x, sred, &s_last, int(L.epoch & 1));
    }
    stamp(c);
    // scratch for the final-wave folds: the (drained) cp.async queue / staging
    if (stream_finish_iteration<kThreads>(A, prm, L, sred, bc, &ctl->bar_str, stamp, &red[0][0])) break;
  }
}

// Small all-reduce (sum, or max when op_max) of `count` <= n + 4 doubles over peer memory, for the
// non-hot exchanges of row-sharded runs (make_state sums, certificate / objective
// partials, the group-lasso graph path): one CTA writes the vector into every
// rank's receive slot, publishes the epoch flag, waits for every rank and sums
// in rank order -- identical results on every rank.
__global__ void __launch_bounds__(512) p2p_allreduce_kernel(double* buf, long long count,
                                                             double* const* peers, double* rbuf,
                                                             unsigned long long* xep, int rank,
                                                             int nranks, long long n, int op_max) {
  const unsigned long long e = *xep + 1;
  const int par = int(e & 1);
  for (long long t = threadIdx.x; t < count; t += blockDim.x) {
    const double v = buf[t];
    for (int r = 0; r < nranks; ++r) xslot(peers[r], par, rank, nranks, n)[t] = v;
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    xpublish(peers, rank, nranks, n, e);
    xwait(rbuf, nranks, n, e);
  }
  __syncthreads();
  for (long long t = threadIdx.x; t < count; t += blockDim.x) {
    double s = op_max ? __ldcg(xslot(rbuf, par, 0, nranks, n) + t) : 0.0;
    for (int r = op_max ? 1 : 0; r < nranks; ++r) {
      const double v = __ldcg(xslot(rbuf, par, r, nranks, n) + t);
      s = op_max ? (v > s ? v : s) : s + v;
    }
    buf[t] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) *xep = e;
}

}  // namespace otdrk
