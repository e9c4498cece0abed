// otdr_tstream.cuh -- the persistent streaming solve loop with a TMA
// producer warp (zero / quadratic regularizer; single GPU or row-sharded).
//
// Same iteration, work split and fold order as stream_kernel
// (otdr_stream.cuh); only phase A (the sweep) is organised differently:
//
//   * one producer warp per CTA claims tiles (rows x 256 columns, the same
//     stripe-major tile numbering and per-iteration atomic counter) and
//     streams each tile as blocks of RB rows through an S-stage shared-memory
//     ring: a 2-D TMA box of X (RB x 256), one of C, a 1-D bulk copy of the
//     block's phi and -- on a tile's first block -- of the stripe's psi, all
//     completing on the stage's `full` mbarrier (complete_tx);
//   * NCW consumer warps take the stages in order: every warp owns RB / NCW
//     rows of the block, reads X and C from shared memory (conflict-free
//     16-byte lanes), computes clamp + prox in fp64 (solver.cpp:97-100,
//     regularizers.cpp:53-55), stores X_{k+1} with coalesced 16-byte stores,
//     reduces its row sums by warp butterfly (rowpart[row][stripe]) and keeps
//     its 8 columns' partial sums in registers, then releases the stage on its
//     `empty` mbarrier. On a tile's last block the consumers fold their column
//     partials (fixed warp order) into colpart[tile] and the CTA completing a
//     stripe folds the stripe (tile order), exactly as stream_stripe_done.
//
// The consumers issue no global loads and no address arithmetic for the
// stream; the copy engine keeps S blocks (S x RB x 2 KB) in flight per SM.
// Phases B and C (row folds, scalar folds, recurrence, stopping logic, the
// peer exchange of row-sharded runs) are stream_finish_iteration, shared with
// stream_kernel, so both loops produce identical iterates.
#pragma once
#include "otdr_stream.cuh"

namespace otdrk {

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
// 1-D bulk copy global -> shared completing on an mbarrier (bytes % 16 == 0)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes,
                                          unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

struct TSMeta {
  int tile;    // -1: end of this iteration's sweep
  int stripe;
  int row0;
  int nrows;   // rows of the block inside the tile (<= RB)
  int flags;   // kTSFirst | kTSLast
  int pad_[3];
};
constexpr int kTSFirst = 1, kTSLast = 2;

template <typename T, int NCW, int RB, int S>
struct TSLayout {
  static constexpr size_t kTile = size_t(RB) * kStreamTN * sizeof(T);  // one X or C box
  static constexpr size_t kStage = 2 * kTile;
  static constexpr size_t oTiles = 0;
  static constexpr size_t oPsi = oTiles + S * kStage;                   // S x 256 doubles
  static constexpr size_t oPhi = oPsi + size_t(S) * kStreamTN * 8;      // S x RB doubles
  static constexpr size_t oMeta = oPhi + size_t(S) * RB * 8;
  static constexpr size_t oBar = oMeta + size_t(S) * sizeof(TSMeta);   // full[S], empty[S]
  static constexpr size_t oRed = (oBar + 2 * S * 8 + 127) / 128 * 128;  // NCW x 256 doubles
  static constexpr size_t kBytes = oRed + size_t(NCW) * kStreamTN * 8;
};

// Column partial of a finished tile (fixed warp order) and the stripe fold of
// the CTA completing the stripe -- stream_stripe_done for the NCW consumer
// warps only (named barrier 1; the producer warp is elsewhere).
template <int NCW, int NV, int VEC>
__device__ __forceinline__ void ts_flush(const StreamArgs& A, int tile, long long stripe,
                                         double (*cacc)[VEC], double* red, double* sred,
                                         int* s_last, int par, unsigned long long plast) {
  constexpr int NC = NCW * 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int e = 0; e < VEC; ++e) red[warp * kStreamTN + v * 32 * VEC + lane * VEC + e] = cacc[v][e];
  named_bar_sync(1, NC);
  for (int col = threadIdx.x; col < kStreamTN; col += NC) {
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < NCW; ++w) sum += red[w * kStreamTN + col];
    st_hint(A.colpart + (long long)tile * kStreamTN + col, sum, plast);
  }
  if (stripe >= A.fin_first) {  // final-wave stripe: folded in phase B
    named_bar_sync(1, NC);       // red is reused by the next tile
    return;
  }
  named_bar_sync(1, NC);  // the consumers' colpart stores before thread 0's release
  if (threadIdx.x == 0) {
    const unsigned need = (unsigned)(A.sfirst[stripe + 1] - A.sfirst[stripe]);
    *s_last = atomic_add_acq_rel_gpu(A.scnt + stripe, 1u) == need - 1;  // otdr_stream.cuh
  }
  named_bar_sync(1, NC);  // thread 0's acquire before the ld.cg of the partials
  if (!*s_last) return;
  double ss = 0.0;
  for (int col = threadIdx.x; col < kStreamTN; col += NC) {  // NC may be < kStreamTN
    const long long j = stripe * kStreamTN + col;
    if (j >= A.n) break;
    const double* src = A.colpart + col;
    const int t0 = A.sfirst[stripe], t1 = A.sfirst[stripe + 1];
    double Ssum = 0.0;
#pragma unroll 16
    for (int t = t0; t < t1; ++t) Ssum += __ldcg(src + (long long)t * kStreamTN);
    if (A.peers) {  // local column sums to every rank's receive slot (NVLink stores)
      for (int r = 0; r < A.nranks; ++r) xslot(A.peers[r], par, A.rank, A.nranks, A.n)[j] = Ssum;
    } else {
      const double sj = __dsub_rn(Ssum, A.q[j]);
      A.s[j] = sj;
      ss += sj * sj;
    }
  }
  if (A.peers) {
    named_bar_sync(1, NC);
    if (threadIdx.x == 0) {
      __threadfence_system();
      A.scnt[stripe] = 0;
    }
    return;
  }
  ss = warp_sum(ss);
  if (lane == 0) sred[warp] = ss;
  named_bar_sync(1, NC);
  if (threadIdx.x == 0) {
    double tot = 0.0;
#pragma unroll
    for (int w = 0; w < NCW; ++w) tot += sred[w];
    A.sspart[stripe] = tot;
    A.scnt[stripe] = 0;  // every tile of this stripe is done for this iteration
  }
  named_bar_sync(1, NC);  // sred free again
}

// One sweep (phase A) of the consumer warps: stages in ring order until the
// producer's end-of-sweep marker. MODE is the fused even/odd mode.
template <typename T, int REG, bool EXACT, int NCW, int RB, int S, int MODE>
__device__ __forceinline__ void ts_consume(const StreamArgs& A, unsigned char* smem, int& ring,
                                           unsigned& round, double* sred, int* s_last, int par,
                                           double rho, double qd, double qinv) {
  using V = typename Vec<T>::type;
  using LY = TSLayout<T, NCW, RB, S>;
  constexpr int VEC = Vec<T>::N;
  constexpr int NV = kStreamTN / (32 * VEC);
  constexpr int RPW = RB / NCW;
  T* tiles = reinterpret_cast<T*>(smem + LY::oTiles);
  const double* psis = reinterpret_cast<const double*>(smem + LY::oPsi);
  const double* phis = reinterpret_cast<const double*>(smem + LY::oPhi);
  const TSMeta* meta = reinterpret_cast<const TSMeta*>(smem + LY::oMeta);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + LY::oBar);
  unsigned long long* empty = full + S;
  double* red = reinterpret_cast<double*>(smem + LY::oRed);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned long long plast = policy_evict_last();
  T* X = static_cast<T*>(A.X);
  double psi_r[NV][VEC], cacc[NV][VEC];
  bool cok[NV];
  T* xrow_base = X;  // X + stripe column offset of the current tile
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    cok[v] = false;
#pragma unroll
    for (int e = 0; e < VEC; ++e) cacc[v][e] = psi_r[v][e] = 0.0;
  }
  for (;;) {
    mbar_wait(&full[ring], round);
    const TSMeta md = meta[ring];
    if (md.tile < 0) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[ring]);
      if (++ring == S) {
        ring = 0;
        round ^= 1u;
      }
      return;
    }
    const long long stripe = md.stripe;
    if (md.flags & kTSFirst) {
      // padded columns beyond ld read psi = -inf (allocation fill) and X = C = 0
      // (TMA out-of-bounds fill), so they clamp to exactly 0: no masks below
      const double* ps = psis + (size_t)ring * kStreamTN;
      xrow_base = X + stripe * kStreamTN;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        cok[v] = stripe * kStreamTN + v * 32 * VEC + lane * VEC < A.ld;
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          psi_r[v][e] = ps[v * 32 * VEC + lane * VEC + e];
          cacc[v][e] = 0.0;
        }
      }
    }
    const T* xt = tiles + (size_t)ring * 2 * RB * kStreamTN;
    const T* ct = xt + RB * kStreamTN;
    const double* ph_s = phis + (size_t)ring * RB;
    double rs[RPW];
#pragma unroll
    for (int u = 0; u < RPW; ++u) {
      const int t = warp + u * NCW;
      rs[u] = 0.0;
      if (t < md.nrows) {  // warp-uniform
        const long long i = md.row0 + t;
        const double ph = ph_s[t];
        V* xg = reinterpret_cast<V*>(xrow_base + i * A.ld);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          double x[VEC], cc[VEC], o[VEC];
          unpack(reinterpret_cast<const V*>(xt + (size_t)t * kStreamTN)[v * 32 + lane], x);
          if (MODE != MODE_ODD) unpack(reinterpret_cast<const V*>(ct + (size_t)t * kStreamTN)[v * 32 + lane], cc);
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            double val;
            if (MODE == MODE_ODD)  // B + phi + psi (solver.cpp:170-172)
              val = EXACT ? __dadd_rn(__dadd_rn(x[e], ph), psi_r[v][e]) : (x[e] + ph) + psi_r[v][e];
            else  // ((X - rho C) + phi) + psi (solver.cpp:97-99)
              val = EXACT ? __dadd_rn(__dadd_rn(__dsub_rn(x[e], __dmul_rn(rho, cc[e])), ph), psi_r[v][e])
                          : (fma(-rho, cc[e], x[e]) + ph) + psi_r[v][e];
            double nx = clamp0(val);
            if (REG == REG_QUAD) nx = EXACT ? div_rn_by(nx, qd, qinv) : nx * qinv;  // regularizers.cpp:54
            // even step of the fused path stores B = (-rho C) + X_{k+1} (solver.cpp:162,167)
            o[e] = MODE == MODE_EVEN ? (EXACT ? __dadd_rn(-__dmul_rn(rho, cc[e]), nx) : nx - rho * cc[e]) : nx;
            cacc[v][e] += nx;
            rs[u] += nx;
          }
          if (cok[v]) xg[v * 32 + lane] = pack<T>(o);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[ring]);  // the stage's shared memory is free
    if (++ring == S) {
      ring = 0;
      round ^= 1u;
    }
    if constexpr (RPW == 2) {
      // both rows at once: one exchange halves the pair (lanes 0-15 keep row
      // u = 0, lanes 16-31 row u = 1), then a 16-lane butterfly
      const bool hi = lane & 16;
      double tot = (hi ? rs[1] : rs[0]) + __shfl_xor_sync(0xffffffffu, hi ? rs[0] : rs[1], 16);
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
      const int t = warp + (hi ? NCW : 0);
      if ((lane & 15) == 0 && t < md.nrows)
        st_hint(A.rowpart + (long long)(md.row0 + t) * A.stripes + stripe, tot, plast);
    } else {
#pragma unroll
      for (int u = 0; u < RPW; ++u) {
        const int t = warp + u * NCW;
        if (t < md.nrows) {
          const double tot = warp_sum(rs[u]);
          if (lane == 0) st_hint(A.rowpart + (long long)(md.row0 + t) * A.stripes + stripe, tot, plast);
        }
      }
    }
    if (md.flags & kTSLast) ts_flush<NCW, NV, VEC>(A, md.tile, stripe, cacc, red, sred, s_last, par, plast);
  }
}

// FUSED: the even/odd path (solver.cpp:127-177) -- a separate instantiation,
// so the plain loop carries no mode branches (fp32 storage runs `fused` on the
// plain loop: otdr_dev_solve)
template <typename T, int REG, bool EXACT, int NCW, int RB, int S, int MINB, bool FUSED = false>
__global__ void __launch_bounds__((NCW + 1) * 32, MINB)
    tstream_kernel(StreamArgs A, const __grid_constant__ CUtensorMap mapX,
                   const __grid_constant__ CUtensorMap mapC) {
  using LY = TSLayout<T, NCW, RB, S>;
  constexpr int NT = (NCW + 1) * 32;
  static_assert(RB % NCW == 0 && RB % 2 == 0, "consumer geometry");
  Ctl* ctl = A.ctl;
  if (ctl->done) return;  // grid-uniform
  const Params& prm = *A.prm;
  extern __shared__ __align__(128) unsigned char ts_smem[];
  T* tiles = reinterpret_cast<T*>(ts_smem + LY::oTiles);
  double* psis = reinterpret_cast<double*>(ts_smem + LY::oPsi);
  double* phis = reinterpret_cast<double*>(ts_smem + LY::oPhi);
  TSMeta* meta = reinterpret_cast<TSMeta*>(ts_smem + LY::oMeta);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(ts_smem + LY::oBar);
  unsigned long long* empty = full + S;
  __shared__ double sred[NT / 32];
  __shared__ double bc[4];
  __shared__ int s_last;
  const int c = (int)blockIdx.x, P = (int)gridDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
  }
  __syncthreads();

  const double rho = prm.rho, qd = prm.quad_d, qinv = prm.quad_inv;
  StreamLoop L;
  L.k = ctl->k;
  L.theta = ctl->theta[L.k & 1];
  L.best = ctl->best;
  L.last_imp = ctl->last_improvement;
  L.k0 = ctl->k0;
  L.it = 0;
  L.epoch = (A.peers != nullptr ? *A.xep : 0ull) + 1;
  L.shifted = prm.fused ? ctl->fused_shifted : 0;
  // ring position: the same sequence in the producer and the consumers
  int ring = 0;
  unsigned round = 0;
  auto stamp = [&](int slot) {
    if (A.tstamp && L.it < kTraceIters && threadIdx.x == 0 && (slot < P ? true : c == 0))
      A.tstamp[L.it * (P + 12) + slot] = globaltimer_ns();
  };

  for (;;) {
    stamp(P + 0);
    const int fmode = prm.fused ? (L.shifted ? MODE_ODD : MODE_EVEN) : MODE_NORMAL;
    if (warp == NCW) {
      // ------------------------------------------------ producer warp
      if (lane == 0) {
        // X, phi and psi were written through the generic proxy (previous
        // iteration, any CTA; ordered by the grid barrier): make them visible
        // to this thread's async-proxy (TMA / bulk) reads
        fence_proxy_async_global();
        const unsigned blk = (unsigned)LY::kTile;
        for (;;) {
          const int tile = (int)atomicAdd(&ctl->tile_ctr, 1u);
          if (tile >= A.ntiles) {
            mbar_wait(&empty[ring], round ^ 1u);
            meta[ring].tile = -1;
            mbar_arrive(&full[ring]);
            if (++ring == S) {
              ring = 0;
              round ^= 1u;
            }
            break;
          }
          const int4 tl = A.tiles[tile];  // {stripe, r0, r1}
          const int st_ = tl.x;
          const long long r0 = tl.y, r1 = tl.z;
          const int col0 = st_ * kStreamTN;
          for (long long rb = r0; rb < r1; rb += RB) {
            mbar_wait(&empty[ring], round ^ 1u);
            TSMeta& md = meta[ring];
            const bool first = rb == r0, last = rb + RB >= r1;
            md.tile = tile;
            md.stripe = st_;
            md.row0 = (int)rb;
            md.nrows = (int)((r1 - rb) < RB ? (r1 - rb) : RB);
            md.flags = (first ? kTSFirst : 0) | (last ? kTSLast : 0);
            const unsigned bytes = blk * (fmode == MODE_ODD ? 1u : 2u) + RB * 8u +
                                   (first ? unsigned(kStreamTN * 8) : 0u);
            mbar_expect_tx(&full[ring], bytes);
            T* xt = tiles + (size_t)ring * 2 * RB * kStreamTN;
            tma_load_2d(xt, &mapX, col0, (int)rb, &full[ring]);
            if (fmode != MODE_ODD) tma_load_2d(xt + RB * kStreamTN, &mapC, col0, (int)rb, &full[ring]);
            bulk_load(phis + (size_t)ring * RB, A.phi + rb, RB * 8u, &full[ring]);
            if (first) bulk_load(psis + (size_t)ring * kStreamTN, A.psi + col0, kStreamTN * 8u, &full[ring]);
            if (++ring == S) {
              ring = 0;
              round ^= 1u;
            }
          }
        }
      }
      __syncwarp();
    } else {
      // ------------------------------------------------ consumer warps
      const int par = int(L.epoch & 1);
      if constexpr (FUSED) {
        if (fmode == MODE_EVEN)
          ts_consume<T, REG, EXACT, NCW, RB, S, MODE_EVEN>(A, ts_smem, ring, round, sred, &s_last, par, rho, qd, qinv);
        else
          ts_consume<T, REG, EXACT, NCW, RB, S, MODE_ODD>(A, ts_smem, ring, round, sred, &s_last, par, rho, qd, qinv);
      } else {
        ts_consume<T, REG, EXACT, NCW, RB, S, MODE_NORMAL>(A, ts_smem, ring, round, sred, &s_last, par, rho, qd, qinv);
      }
      // this sweep's X stores are read by the next iteration's TMA (async proxy)
      fence_proxy_async_global();
    }
    stamp(c);
    // scratch for the final-wave folds: the ring (idle between sweeps)
    if (stream_finish_iteration<NT>(A, prm, L, sred, bc, &ctl->bar_tst, stamp,
                                    reinterpret_cast<double*>(ts_smem + LY::oTiles)))
      break;
  }
}

}  // namespace otdrk
