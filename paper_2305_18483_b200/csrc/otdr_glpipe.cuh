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
// position = run of up to 8 consecutive stripes) -- from an atomic counter,
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

template <typename T, bool EXACT, int D, int WB>
__global__ void __launch_bounds__(kGLPThreads, 1) gl_pipe_kernel(GLPipeArgs A) {
  using V = typename Vec<T>::type;
  constexpr int VEC = Vec<T>::N;
  constexpr int W = WB / (int)sizeof(T);   // stripe width: WB (128 or 64) bytes per row
  constexpr int LPR = W / VEC;             // lanes per row (8 for 128-B stripes)
  constexpr int RPW = 32 / LPR;            // rows per warp instruction
  constexpr int RSTEP = kGLPWarps * RPW;   // rows per step
  Ctl* ctl = A.ctl;
  if (ctl->done) return;  // grid-uniform
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
    if (threadIdx.x == 0) s_item = atomicAdd(&ctl->gl_ctr, 1u);
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
            A.colpart[(long long)si * A.ld + col] = s;
          }
        }
      }
      __syncthreads();
    }
    cp_async_wait<0>();
    for (int t = threadIdx.x; t < L; t += kGLPThreads)
      A.rowpart[(sg.begin + t) * (long long)A.ngroups + gi] = rowacc[t];
    __syncthreads();  // rowacc / phi_s / s_item reused by the next item
  }
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
