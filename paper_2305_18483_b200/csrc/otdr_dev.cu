// otdr_dev.cu -- C-ABI (include/otdr_dev.h) over the sm_100a RDROT kernels.
//
// Host side of the drop-in boundary: owns device memory, the stream, CUDA
// graphs and (row-sharded runs) the NCCL communicator. The solve loop of
// solver.cpp:104-241 runs entirely on device: one CUDA graph whose WHILE
// conditional node repeats a body of `unroll` DR iterations until the update
// kernel clears the condition (converged / stalled / max_iter / non-finite).
// Multi-rank contexts (NCCL inside the body) use host-polled chunk graphs.
#include "otdr_dev.h"
#include "otdr_kernels.cuh"
#include "otdr_resident.cuh"
#include "otdr_stream.cuh"
#include "otdr_glpipe.cuh"
#include "otdr_bstream.cuh"
#include "otdr_tstream.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <fcntl.h>
#include <unistd.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <numeric>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

using otdrk::Ctl;
using otdrk::Params;
using otdrk::Segment;

namespace {

constexpr int kNumSMs = 148;
constexpr int kSweepTN = 256;  // plain sweep stripe width (both storages)
constexpr size_t kStageDoubles = size_t(1) << 25;  // 256 MB fp64 staging
constexpr size_t kPinBytes = size_t(64) << 20;      // pinned host chunk (x2, double-buffered)

// Host threads for the fp64 <-> storage conversions of uploads / downloads
// (OTDR_HOST_THREADS overrides; the reference API hands us pageable fp64
// rows, which the DMA engines cannot read directly).
int host_threads() {
  static const int t = [] {
    if (const char* e = std::getenv("OTDR_HOST_THREADS")) return std::max(1, std::atoi(e));
    const unsigned hc = std::thread::hardware_concurrency();
    return int(std::min(16u, std::max(1u, hc)));
  }();
  return t;
}

// f(lo, hi) over [0, count) split across the host threads.
template <typename F>
void host_parallel(long long count, F&& f) {
  const int th = host_threads();
  if (th <= 1 || count < (1LL << 18)) {
    f(0LL, count);
    return;
  }
  const long long per = (count + th - 1) / th;
  std::vector<std::thread> pool;
  pool.reserve(size_t(th));
  for (int t = 1; t < th; ++t) {
    const long long lo = t * per, hi = std::min(count, lo + per);
    if (lo < hi) pool.emplace_back([&f, lo, hi] { f(lo, hi); });
  }
  f(0LL, std::min(count, per));
  for (auto& x : pool) x.join();
}

struct Error {
  otdr_status code;
  std::string msg;
};

#define CK(expr)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (expr);                                                          \
    if (e_ != cudaSuccess)                                                            \
      throw Error{OTDR_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)};   \
  } while (0)
// NCCL is bound at run time (dlopen) so the process uses whichever libnccl is
// already loaded (e.g. the one PyTorch bundles); only row-sharded contexts
// need it.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(h, "ncclAllReduce"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.GetUniqueId && a.CommInitRank && a.AllReduce && a.CommDestroy && a.GetErrorString;
    return a;
  }();
  return api;
}

#define NK(expr)                                                                      \
  do {                                                                                \
    if (!nccl().ok) throw Error{OTDR_E_NCCL, "libnccl.so.2 could not be loaded"};     \
    ncclResult_t r_ = (expr);                                                         \
    if (r_ != ncclSuccess)                                                            \
      throw Error{OTDR_E_NCCL, std::string(#expr) + ": " + nccl().GetErrorString(r_)}; \
  } while (0)

template <typename T>
T* dalloc(size_t count) {
  void* p = nullptr;
  if (count == 0) count = 1;
  CK(cudaMalloc(&p, count * sizeof(T)));
  return static_cast<T*>(p);
}

// Driver virtual-memory allocation with generic (L2 <-> HBM) compression:
// lines that compress (all-zero, repeated values) travel between L2 and HBM
// in fewer sectors. The driver functions are looked up at run time so the
// library still links against cudart only.
struct CompAlloc {
  PFN_cuMemGetAllocationGranularity gran = nullptr;
  PFN_cuMemCreate create = nullptr;
  PFN_cuMemAddressReserve reserve = nullptr;
  PFN_cuMemMap map = nullptr;
  PFN_cuMemSetAccess access = nullptr;
  PFN_cuMemUnmap unmap = nullptr;
  PFN_cuMemAddressFree afree = nullptr;
  PFN_cuMemRelease release = nullptr;
  PFN_cuMemRetainAllocationHandle retain = nullptr;
  PFN_cuMemGetAllocationPropertiesFromHandle props = nullptr;
  bool ok = false;
  CompAlloc() {
    auto get = [](const char* name) -> void* {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess)
        return nullptr;
      return fn;
    };
    gran = (PFN_cuMemGetAllocationGranularity)get("cuMemGetAllocationGranularity");
    create = (PFN_cuMemCreate)get("cuMemCreate");
    reserve = (PFN_cuMemAddressReserve)get("cuMemAddressReserve");
    map = (PFN_cuMemMap)get("cuMemMap");
    access = (PFN_cuMemSetAccess)get("cuMemSetAccess");
    unmap = (PFN_cuMemUnmap)get("cuMemUnmap");
    afree = (PFN_cuMemAddressFree)get("cuMemAddressFree");
    release = (PFN_cuMemRelease)get("cuMemRelease");
    retain = (PFN_cuMemRetainAllocationHandle)get("cuMemRetainAllocationHandle");
    props = (PFN_cuMemGetAllocationPropertiesFromHandle)get("cuMemGetAllocationPropertiesFromHandle");
    ok = gran && create && reserve && map && access && unmap && afree && release;
  }
};

inline CompAlloc& comp_alloc() {
  static CompAlloc c;
  return c;
}

// One contiguous virtual range over two physical allocations: the first
// comp_bytes (rounded to the granularity) with generic compression, the rest
// without. Returns nullptr (and leaves nothing allocated) when the driver
// cannot provide it; *size_out = mapped size, *compressed = whether the
// driver really granted compression to the first part.
inline void* comp_malloc(int device, size_t bytes, size_t comp_bytes, size_t* size_out, bool* compressed) {
  CompAlloc& d = comp_alloc();
  *compressed = false;
  if (!d.ok) return nullptr;
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  prop.allocFlags.compressionType = CU_MEM_ALLOCATION_COMP_GENERIC;
  size_t g = 0, g2 = 0;
  if (d.gran(&g, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || !g) return nullptr;
  CUmemAllocationProp plain = prop;
  plain.allocFlags.compressionType = 0;
  if (d.gran(&g2, &plain, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || !g2) return nullptr;
  g = std::max(g, g2);
  const size_t size = (bytes + g - 1) / g * g;
  const size_t csize = std::min(size, (comp_bytes + g - 1) / g * g);
  if (csize == 0) return nullptr;
  CUdeviceptr va = 0;
  if (d.reserve(&va, size, g, 0, 0) != CUDA_SUCCESS) return nullptr;
  size_t mapped = 0;
  bool fail = false;
  for (int part = 0; part < 2 && !fail; ++part) {
    const size_t len = part == 0 ? csize : size - csize;
    if (!len) continue;
    CUmemGenericAllocationHandle h;
    if (d.create(&h, len, part == 0 ? &prop : &plain, 0) != CUDA_SUCCESS) {
      fail = true;
      break;
    }
    if (d.map(va + mapped, len, 0, h, 0) != CUDA_SUCCESS) fail = true;
    else mapped += len;
    d.release(h);  // the mapping keeps the physical memory alive
  }  CUmemAccessDesc acc{};
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if (fail || d.access(va, size, &acc, 1) != CUDA_SUCCESS) {
    if (mapped) d.unmap(va, mapped);
    d.afree(va, size);
    return nullptr;
  }
  // the driver may silently grant an uncompressed allocation
  if (d.props && d.retain) {
    CUmemGenericAllocationHandle h2;
    if (d.retain(&h2, (void*)va) == CUDA_SUCCESS) {
      CUmemAllocationProp got{};
      if (d.props(&got, h2) == CUDA_SUCCESS)
        *compressed = got.allocFlags.compressionType == CU_MEM_ALLOCATION_COMP_GENERIC;
      d.release(h2);
    }
  }
  *size_out = size;
  return (void*)va;
}

inline void comp_free(void* p, size_t size) {
  if (!p) return;
  CompAlloc& d = comp_alloc();
  d.unmap((CUdeviceptr)p, size);
  d.afree((CUdeviceptr)p, size);
}

}  // namespace

struct otdr_dev {
  otdr_dev_config cfg{};
  int storage = OTDR_STORE_F32;
  size_t esz = 4;
  long long m_glob = 0, n = 0, m_loc = 0, row0 = 0, ld = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  ncclComm_t comm = nullptr;
  std::string err;

  void* C = nullptr;
  void* X = nullptr;
  size_t x_vmm = 0, c_vmm = 0;  // mapped sizes when X / C are compressible VMM allocations
  bool x_comp = false, c_comp = false;
  double *p = nullptr, *q = nullptr, *phi = nullptr, *psi = nullptr, *a = nullptr, *b = nullptr,
         *r = nullptr, *s = nullptr;
  double *rowpart = nullptr, *colpart = nullptr, *exch = nullptr, *bpart = nullptr,
         *cpart = nullptr, *csum = nullptr, *stage = nullptr;
  int num_sms = 148;
  // on-chip resident solve (plans that fit the GPU's aggregate shared memory)
  bool allow_resident = true;
  bool sharded = false;  // NCCL exchange path (row shards, or a 1-rank communicator)
  int res_G = 0, res_R = 0;
  size_t res_smem = 0;
  // fp32 storage on fp64 shared-memory tiles when they fit (OTDR_RESIDENT_TILES=f32: storage type)
  bool res_wide = false, res_allow_wide = true;
  double* gscratch = nullptr;
  // peer-memory exchange of row-sharded runs (CUDA IPC over NVLink)
  bool p2p = false;
  double* rbuf = nullptr;            // this rank's receive buffer
  double** d_peers = nullptr;        // [nranks] receive buffers of every rank
  unsigned long long* d_xep = nullptr;
  std::vector<void*> ipc_opened;
  // persistent streaming solve (single GPU, zero / quadratic, HBM-resident plan)
  bool allow_stream = true;
  int str_P = 0, str_ntiles = 0, str_tpc = 0, str_tail = 4;
  size_t str_part_cap = 0;
  double *str_part = nullptr, *str_colpart = nullptr;
  int str_big = 1, str_small = 1;  // streaming tile rows (long / tail tiles)
  int4* d_tiles = nullptr;     // streaming tiles {stripe, r0, r1, 0}, stripe-major
  int str_fin_first = 1 << 30;  // first stripe of the final wave (folded in phase B)
  bool str_fin = false;         // OTDR_STREAM_FIN=1: final wave (measured slower)
  // streaming kernel: 1 = TMA producer warp + consumer warps (tstream_kernel,
  // the fp32-storage default), 0 = per-thread cp.async queues (stream_kernel;
  // fp64 storage, and fp32 with OTDR_STREAM_KERNEL=async); ts_cfg picks the
  // tstream consumer geometry
  int str_kind = 1, ts_cfg = 0;
  std::string kname;  // otdr_dev_kernel_name
  CUtensorMap ts_mapX{}, ts_mapC{};
  bool ts_maps = false;
  int* d_sfirst = nullptr;
  unsigned* d_scnt = nullptr;
  double* str_sspart = nullptr;
  long long* d_dev_row = nullptr;
  Segment *d_seg = nullptr, *d_cert_seg = nullptr;
  Params* d_prm = nullptr;
  Ctl* d_ctl = nullptr;
  Ctl* h_ctl = nullptr;  // pinned
  otdrk::TraceRow* d_trace = nullptr;
  long long trace_cap = 0;
  unsigned long long* d_mx = nullptr;

  // host mirrors
  Params prm{};
  std::vector<long long> dev_row;  // host (local) row -> device row
  std::vector<double> h_p, h_q;
  std::vector<int32_t> labels;
  int reg_kind = OTDR_REG_NONE;
  double reg_param = 0.0;
  bool has_problem = false, has_state = false;

  // geometry
  int stripes = 1, rowgroups = 1, rows_per_cta = 1;
  int gl_stripes = 1, num_segs = 0, cert_stripes = 1, num_cert_segs = 0;
  // pipelined single-pass GL sweep: persistent CTAs over (segment, G stripes)
  int glp_G = 0, glp_nstr = 0, glp_groups = 0, glp_lmax = 0, glp_d = 0, glp_wb = 128;
  int2* d_glp_pos = nullptr;
  size_t glp_smem = 0;
  int RB = 1, CB = 1;
  size_t rowpart_cap = 0, colpart_cap = 0, cpart_cap = 0;
  std::vector<Segment> segs, cert_segs;

  // graphs keyed by (kind, unroll/chunk, track, cert, fused)
  std::map<std::tuple<int, int, int, int, int>, cudaGraphExec_t> graphs;

  bool f64() const { return storage == OTDR_STORE_F64; }
  int tn_seg() const { return f64() ? 64 : 128; }  // GL / certificate stripe width

  // ---------------------------------------------------------------- launches
  static constexpr int kGLThreads = 512;


  // 2-D tensor map over a row-major (m_loc x ld) matrix, box TN x R.
  void encode_map(CUtensorMap* map, void* base, int tn, int rows) {
    static PFN_cuTensorMapEncodeTiled encode = [] {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
              cudaSuccess ||
          q != cudaDriverEntryPointSuccess)
        fn = nullptr;
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
    }();
    if (!encode) throw Error{OTDR_E_CUDA, "cuTensorMapEncodeTiled unavailable"};
    const cuuint64_t dims[2] = {cuuint64_t(ld), cuuint64_t(std::max<long long>(m_loc, 1))};
    const cuuint64_t strides[1] = {cuuint64_t(ld) * esz};
    const cuuint32_t box[2] = {cuuint32_t(tn), cuuint32_t(rows)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode(map, f64() ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                              2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error{OTDR_E_CUDA, "cuTensorMapEncodeTiled failed"};
  }

  // The pipelined kernel covers the plain (non-fused, untracked) iteration;
  // the even/odd and support-tracking variants use the two-phase kernel.
  bool gl_pipe_active(bool track) const { return glp_G > 0 && !track && !prm.fused; }

  template <typename T, int D, int WB>
  void launch_gl_pipe_t() {
    auto kern = otdrk::gl_pipe_kernel<T, sizeof(T) == 8, D, WB>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(glp_smem)));
    otdrk::GLPipeArgs ga{X, C, phi, psi, rowpart, colpart, d_seg, d_glp_pos, d_prm, d_ctl, m_loc, ld,
                         num_segs, glp_nstr, glp_groups, glp_lmax};
    // OTDR_GL_PIPE_GRID caps the persistent grid (several ranks sharing one GPU in tests)
    const int cap = std::getenv("OTDR_GL_PIPE_GRID") ? std::atoi(std::getenv("OTDR_GL_PIPE_GRID")) : 0;
    const int grid = cap > 0 ? std::min(cap, num_sms) : num_sms;
    kern<<<grid, otdrk::kGLPThreads, glp_smem, stream>>>(ga);
  }
  template <typename T>
  void launch_gl_pipe_d() {
    if (glp_wb == 64) {
      if (glp_d == 8) launch_gl_pipe_t<T, 8, 64>();
      else if (glp_d == 6) launch_gl_pipe_t<T, 6, 64>();
      else launch_gl_pipe_t<T, 4, 64>();
    } else {
      if (glp_d == 4) launch_gl_pipe_t<T, 4, 128>();
      else if (glp_d == 3) launch_gl_pipe_t<T, 3, 128>();
      else launch_gl_pipe_t<T, 2, 128>();
    }
  }
  void launch_gl_pipe() {
    if (f64()) launch_gl_pipe_d<double>();
    else launch_gl_pipe_d<float>();
  }

  // Persistent group-lasso solve (one cooperative launch; OTDR_GL_STREAM=off
  // keeps the CUDA-graph loop of gl_pipe + reduce + update).
  bool allow_gl_stream = true;
  bool gl_stream_active(bool track, bool cert) const {
    return allow_gl_stream && reg_kind == OTDR_REG_GROUP_LASSO && gl_pipe_active(track) && !cert &&
           (!sharded || p2p) && gls_grid > 0;
  }
  int gls_grid = 0;
  template <typename T, int D, int WB>
  void launch_gl_stream_t(long long iters) {
    auto kern = otdrk::gl_stream_kernel<T, sizeof(T) == 8, D, WB>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(glp_smem)));
    otdrk::GLStreamArgs ga{
        otdrk::GLPipeArgs{X, C, phi, psi, rowpart, colpart, d_seg, d_glp_pos, d_prm, d_ctl, m_loc, ld,
                          num_segs, glp_nstr, glp_groups, glp_lmax},
        phi, psi, a, b, r, s, p, q, str_part, m_glob, n, sharded ? d_peers : nullptr, rbuf, d_xep,
        cfg.rank, cfg.nranks, iters};
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(unsigned(gls_grid), 1, 1);
    lc.blockDim = dim3(otdrk::kGLPThreads, 1, 1);
    lc.dynamicSmemBytes = glp_smem;
    lc.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    CK(cudaLaunchKernelEx(&lc, kern, ga));
  }
  template <typename T>
  void launch_gl_stream_d(long long iters) {
    if (glp_wb == 64) {
      if (glp_d == 8) launch_gl_stream_t<T, 8, 64>(iters);
      else if (glp_d == 6) launch_gl_stream_t<T, 6, 64>(iters);
      else launch_gl_stream_t<T, 4, 64>(iters);
    } else {
      if (glp_d == 4) launch_gl_stream_t<T, 4, 128>(iters);
      else if (glp_d == 3) launch_gl_stream_t<T, 3, 128>(iters);
      else launch_gl_stream_t<T, 2, 128>(iters);
    }
  }
  void launch_gl_stream(long long iters) {
    if (f64()) launch_gl_stream_d<double>(iters);
    else launch_gl_stream_d<float>(iters);
  }

  static size_t glpipe_smem(bool f64s, int d, int wb, int lmax) {
    const size_t q = size_t(d) * 2 * otdrk::kGLPThreads * 16;
    const size_t base = f64s ? (wb == 64 ? otdrk::glpipe_smem_bytes<double, 2, 64>(lmax)
                                         : otdrk::glpipe_smem_bytes<double, 2, 128>(lmax))
                             : (wb == 64 ? otdrk::glpipe_smem_bytes<float, 2, 64>(lmax)
                                         : otdrk::glpipe_smem_bytes<float, 2, 128>(lmax));
    return base - otdrk::glpipe_queue_bytes<float, 2>() + q;
  }

  void launch_sweep(bool track, bool sums_only) {
    if (reg_kind == OTDR_REG_GROUP_LASSO && !sums_only && gl_pipe_active(track)) {
      launch_gl_pipe();
      return;
    }
    if (reg_kind == OTDR_REG_GROUP_LASSO && !sums_only) {
      dim3 grid((unsigned)((ld + tn_seg() - 1) / tn_seg()), num_segs);
      if (f64()) {
        otdrk::GLArgs<double> ga{(double*)X, (const double*)C, phi, psi, rowpart, colpart,
                                 d_seg, d_prm, d_ctl, m_loc, ld};
        if (track) otdrk::gl_sweep_kernel<double, true, true, 1><<<grid, otdrk::kThreads, 0, stream>>>(ga);
        else otdrk::gl_sweep_kernel<double, true, false, 1><<<grid, otdrk::kThreads, 0, stream>>>(ga);
      } else {
        otdrk::GLArgs<float> ga{(float*)X, (const float*)C, phi, psi, rowpart, colpart,
                                d_seg, d_prm, d_ctl, m_loc, ld};
        if (track) otdrk::gl_sweep_kernel<float, false, true, 1><<<grid, otdrk::kThreads, 0, stream>>>(ga);
        else otdrk::gl_sweep_kernel<float, false, false, 1><<<grid, otdrk::kThreads, 0, stream>>>(ga);
      }
      return;
    }
    dim3 grid(stripes, rowgroups);
    const int so = sums_only ? 1 : 0;
    if (f64()) {
      otdrk::SweepArgs<double> sa{(double*)X, (const double*)C, phi, psi, rowpart, colpart,
                                  d_prm, d_ctl, m_loc, ld, rows_per_cta, so};
      if (reg_kind == OTDR_REG_QUAD) {
        if (track) otdrk::sweep_kernel<double, otdrk::REG_QUAD, true, true, 4, 1><<<grid, otdrk::kThreads, 0, stream>>>(sa);
        else otdrk::sweep_kernel<double, otdrk::REG_QUAD, true, false, 4, 1><<<grid, otdrk::kThreads, 0, stream>>>(sa);
      } else {
        if (track) otdrk::sweep_kernel<double, otdrk::REG_NONE, true, true, 4, 1><<<grid, otdrk::kThreads, 0, stream>>>(sa);
        else otdrk::sweep_kernel<double, otdrk::REG_NONE, true, false, 4, 1><<<grid, otdrk::kThreads, 0, stream>>>(sa);
      }
    } else {
      otdrk::SweepArgs<float> sa{(float*)X, (const float*)C, phi, psi, rowpart, colpart,
                                 d_prm, d_ctl, m_loc, ld, rows_per_cta, so};
      if (reg_kind == OTDR_REG_QUAD) {
        if (track) otdrk::sweep_kernel<float, otdrk::REG_QUAD, false, true, 2, 2><<<grid, otdrk::kThreads, 0, stream>>>(sa);
        else otdrk::sweep_kernel<float, otdrk::REG_QUAD, false, false, 2, 2><<<grid, otdrk::kThreads, 0, stream>>>(sa);
      } else {
        if (track) otdrk::sweep_kernel<float, otdrk::REG_NONE, false, true, 2, 2><<<grid, otdrk::kThreads, 0, stream>>>(sa);
        else otdrk::sweep_kernel<float, otdrk::REG_NONE, false, false, 2, 2><<<grid, otdrk::kThreads, 0, stream>>>(sa);
      }
    }
  }

  bool gl_active(bool sums_only) const { return reg_kind == OTDR_REG_GROUP_LASSO && !sums_only; }

  // (stripes of the row partials, row groups of the column partials) written
  // by the sweep variant that runs in this configuration.
  std::pair<int, int> partial_shape(bool sums_only, bool track) const {
    if (gl_active(sums_only)) {
      if (gl_pipe_active(track)) return {glp_groups, num_segs};
      return {int((ld + tn_seg() - 1) / tn_seg()), num_segs};
    }
    return {stripes, rowgroups};
  }

  void launch_reduce(bool sums_only, bool track) {
    const auto [nstripes, ngroups] = partial_shape(sums_only, track);
    otdrk::ReduceArgs ra{rowpart, colpart, p, r, exch, bpart, d_ctl, m_loc, n, ld,
                         nstripes, ngroups, RB};
    otdrk::reduce_kernel<<<RB + CB, otdrk::kThreads, 0, stream>>>(ra);
  }

  void launch_exchange(double* buf, size_t count, bool op_max = false) {
    if (comm) {
      NK(nccl().AllReduce(buf, buf, count, ncclDouble, op_max ? ncclMax : ncclSum, comm, stream));
    } else if (p2p) {
      otdrk::p2p_allreduce_kernel<<<1, 512, 0, stream>>>(buf, (long long)count, d_peers, rbuf, d_xep,
                                                          cfg.rank, cfg.nranks, n, op_max ? 1 : 0);
    } else if (cfg.nranks > 1) {
      throw Error{OTDR_E_STATE, "row-sharded context has no exchange: pass an NCCL id or link peers"};
    }
  }

  size_t rbuf_bytes() const {
    return size_t(2 * cfg.nranks) * size_t(n + 4) * 8 + size_t(2 * cfg.nranks) * 8;
  }
  void alloc_rbuf() {
    if (rbuf) return;
    CK(cudaMalloc(&rbuf, rbuf_bytes()));
    CK(cudaMemset(rbuf, 0, rbuf_bytes()));
    d_xep = dalloc<unsigned long long>(1);
    CK(cudaMemset(d_xep, 0, 8));
  }
  // Under lazy module loading (CUDA 12 default) the first launch of a kernel
  // waits for the device to idle. Ranks that share ONE GPU (the multi-context
  // tests) would deadlock: a rank's exchange kernel spins until the other rank
  // launches, and that launch waits for the spinning kernel. Load every kernel
  // a sharded context can launch before the first exchange.
  template <typename K>
  static void touch(K k) {
    cudaFuncAttributes at;
    CK(cudaFuncGetAttributes(&at, reinterpret_cast<const void*>(k)));
  }
  template <typename T, int REG>
  static void touch_stream() {
    constexpr bool E = sizeof(T) == 8;
    constexpr int NV = E ? 4 : 2, U = E ? 1 : 2;
    touch(otdrk::stream_kernel<T, REG, E, NV, U, 0>);
    touch(otdrk::stream_kernel<T, REG, E, NV, U, 2>);
    touch(otdrk::stream_kernel<T, REG, E, NV, U, 3>);
    touch(otdrk::stream_kernel<T, REG, E, NV, U, 4>);
    touch(otdrk::stream_kernel<T, REG, E, NV, U, 5>);
  }
  static void preload_kernels() {
    static bool done = false;
    if (done) return;
    touch(otdrk::p2p_allreduce_kernel);
    touch_stream<float, otdrk::REG_NONE>();
    touch_stream<float, otdrk::REG_QUAD>();
    touch_stream<double, otdrk::REG_NONE>();
    touch_stream<double, otdrk::REG_QUAD>();
    touch(otdrk::sweep_kernel<double, otdrk::REG_NONE, true, false, 4, 1>);
    touch(otdrk::sweep_kernel<double, otdrk::REG_NONE, true, true, 4, 1>);
    touch(otdrk::sweep_kernel<double, otdrk::REG_QUAD, true, false, 4, 1>);
    touch(otdrk::sweep_kernel<double, otdrk::REG_QUAD, true, true, 4, 1>);
    touch(otdrk::sweep_kernel<float, otdrk::REG_NONE, false, false, 2, 2>);
    touch(otdrk::sweep_kernel<float, otdrk::REG_NONE, false, true, 2, 2>);
    touch(otdrk::sweep_kernel<float, otdrk::REG_QUAD, false, false, 2, 2>);
    touch(otdrk::sweep_kernel<float, otdrk::REG_QUAD, false, true, 2, 2>);
    touch(otdrk::gl_pipe_kernel<float, false, 2, 128>);
    touch(otdrk::gl_pipe_kernel<float, false, 3, 128>);
    touch(otdrk::gl_pipe_kernel<float, false, 4, 128>);
    touch(otdrk::gl_pipe_kernel<double, true, 2, 128>);
    touch(otdrk::gl_pipe_kernel<double, true, 3, 128>);
    touch(otdrk::gl_pipe_kernel<double, true, 4, 128>);
    touch(otdrk::gl_pipe_kernel<float, false, 4, 64>);
    touch(otdrk::gl_pipe_kernel<float, false, 6, 64>);
    touch(otdrk::gl_pipe_kernel<float, false, 8, 64>);
    touch(otdrk::gl_pipe_kernel<double, true, 4, 64>);
    touch(otdrk::gl_pipe_kernel<double, true, 6, 64>);
    touch(otdrk::gl_pipe_kernel<double, true, 8, 64>);
    touch(otdrk::gl_stream_kernel<float, false, 2, 128>);
    touch(otdrk::gl_stream_kernel<float, false, 3, 128>);
    touch(otdrk::gl_stream_kernel<float, false, 4, 128>);
    touch(otdrk::gl_stream_kernel<double, true, 2, 128>);
    touch(otdrk::gl_stream_kernel<double, true, 3, 128>);
    touch(otdrk::gl_stream_kernel<double, true, 4, 128>);
    touch(otdrk::gl_sweep_kernel<double, true, false, 1>);
    touch(otdrk::gl_sweep_kernel<double, true, true, 1>);
    touch(otdrk::gl_sweep_kernel<float, false, false, 1>);
    touch(otdrk::gl_sweep_kernel<float, false, true, 1>);
    touch(otdrk::reduce_kernel);
    touch(otdrk::update_kernel);
    touch(otdrk::seed_state_kernel);
    touch(otdrk::stamp_t0_kernel);
    touch(otdrk::cert_partial_kernel<double, 1>);
    touch(otdrk::cert_partial_kernel<float, 1>);
    touch(otdrk::cert_final_kernel);
    touch(otdrk::unshift_kernel<double>);
    touch(otdrk::unshift_kernel<float>);
    touch(otdrk::scatter_rows_kernel<double>);
    touch(otdrk::scatter_rows_kernel<float>);
    touch(otdrk::gather_rows_kernel<double>);
    touch(otdrk::gather_rows_kernel<float>);
    touch(otdrk::move_rows_kernel);
    touch(otdrk::sqdist_kernel<double>);
    touch(otdrk::sqdist_kernel<float>);
    done = true;
  }

  void set_peers(const std::vector<double*>& peers) {
    preload_kernels();
    if (!d_peers) d_peers = dalloc<double*>(size_t(cfg.nranks));
    CK(cudaMemcpy(d_peers, peers.data(), size_t(cfg.nranks) * sizeof(double*), cudaMemcpyHostToDevice));
    p2p = true;
    sharded = true;  // a linked 1-rank context runs the sharded (peer-exchange) loop
    res_G = 0;
    invalidate_graphs();
    plan_stream();
  }

  void launch_update(cudaGraphConditionalHandle cond, int use_cond, int cert_follows) {
    otdrk::UpdateArgs ua{exch, q, r, s, phi, psi, a, b, bpart, d_prm, d_ctl, d_trace,
                         m_loc, m_glob, n, RB, CB, cond, use_cond, cert_follows};
    otdrk::update_kernel<<<RB + CB, otdrk::kThreads, 0, stream>>>(ua);
  }

  void launch_cert(int objective_only, cudaGraphConditionalHandle cond, int use_cond) {
    const int regk = reg_kind == OTDR_REG_GROUP_LASSO ? otdrk::REG_GL
                     : reg_kind == OTDR_REG_QUAD      ? otdrk::REG_QUAD
                                                      : otdrk::REG_NONE;
    dim3 grid(cert_stripes, num_cert_segs);
    if (f64()) {
      otdrk::CertArgs<double> ca{(const double*)X, (const double*)C, phi, psi, p, d_cert_seg,
                                 cpart, csum, d_prm, d_ctl, m_loc, ld, regk, objective_only};
      otdrk::cert_partial_kernel<double, 1><<<grid, otdrk::kThreads, 0, stream>>>(ca);
    } else {
      otdrk::CertArgs<float> ca{(const float*)X, (const float*)C, phi, psi, p, d_cert_seg,
                                cpart, csum, d_prm, d_ctl, m_loc, ld, regk, objective_only};
      otdrk::cert_partial_kernel<float, 1><<<grid, otdrk::kThreads, 0, stream>>>(ca);
    }
    launch_exchange(csum, otdrk::kCertVals);
    otdrk::CertFinalArgs fa{csum, q, psi, d_prm, d_ctl, d_trace, n, regk, objective_only,
                            cond, use_cond};
    otdrk::cert_final_kernel<<<1, otdrk::kThreads, 0, stream>>>(fa);
  }


  // One DR iteration on the graph path: sweep, reduce, (row shards) all-reduce
  // of the exchange vector, update; [certificate].
  void launch_iteration(bool track, bool cert, cudaGraphConditionalHandle cond, int use_cond) {
    launch_sweep(track, false);
    launch_reduce(false, track);
    launch_exchange(exch, size_t(n) + 3);
    launch_update(cond, use_cond, cert ? 1 : 0);
    if (cert) launch_cert(0, cond, use_cond);
  }

  void check_launch() { CK(cudaGetLastError()); }


  // ---------------------------------------------------------------- geometry
  void plan_geometry() {
    stripes = int((ld + kSweepTN - 1) / kSweepTN);
    const long long target = 8LL * 2 * kNumSMs;  // ~8 waves at 2 CTAs/SM
    long long rg = std::max<long long>(1, target / stripes);
    rg = std::min<long long>(rg, std::max<long long>(1, (m_loc + 15) / 16));
    rows_per_cta = int((m_loc + rg - 1) / rg);
    rowgroups = int((m_loc + rows_per_cta - 1) / rows_per_cta);
    gl_stripes = int((ld + tn_seg() - 1) / tn_seg());
    cert_stripes = int((ld + tn_seg() - 1) / tn_seg());
    RB = int((m_loc + otdrk::kThreads - 1) / otdrk::kThreads);
    CB = int((n + otdrk::kThreads - 1) / otdrk::kThreads);
  }

  // Segments for the group-lasso sweep (class runs in device order) and the
  // certificate (class runs for GL; uniform row chunks otherwise).
  void build_segments() {
    segs.clear();
    cert_segs.clear();
    if (reg_kind == OTDR_REG_GROUP_LASSO) {
      std::vector<int32_t> dev_lab(static_cast<size_t>(m_loc));
      for (long long h = 0; h < m_loc; ++h) dev_lab[size_t(dev_row[h])] = labels[size_t(h)];
      long long i = 0;
      while (i < m_loc) {
        long long j = i;
        while (j < m_loc && dev_lab[size_t(j)] == dev_lab[size_t(i)]) ++j;
        const int grouped = dev_lab[size_t(i)] >= 0 ? 1 : 0;
        if (grouped) {
          segs.push_back(Segment{i, j, 1, 0});
          cert_segs.push_back(Segment{i, j, 1, 0});
        } else {
          for (long long t = i; t < j; t += 256) {
            segs.push_back(Segment{t, std::min(j, t + 256), 0, 0});
            cert_segs.push_back(Segment{t, std::min(j, t + 256), 0, 0});
          }
        }
        i = j;
      }
    } else {
      const long long chunk = std::max<long long>(64, (m_loc + 63) / 64);
      for (long long t = 0; t < m_loc; t += chunk)
        cert_segs.push_back(Segment{t, std::min(m_loc, t + chunk), 0, 0});
    }
    if (segs.empty()) segs.push_back(Segment{0, 0, 0, 0});
    if (cert_segs.empty()) cert_segs.push_back(Segment{0, 0, 0, 0});
    num_segs = int(segs.size());
    num_cert_segs = int(cert_segs.size());
    plan_gl();
    plan_resident();
    plan_stream();
    if (d_seg) cudaFree(d_seg);
    if (d_cert_seg) cudaFree(d_cert_seg);
    d_seg = dalloc<Segment>(segs.size());
    d_cert_seg = dalloc<Segment>(cert_segs.size());
    CK(cudaMemcpy(d_seg, segs.data(), segs.size() * sizeof(Segment), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_cert_seg, cert_segs.data(), cert_segs.size() * sizeof(Segment),
                  cudaMemcpyHostToDevice));
    ensure_partials();
  }

  // Resident plan: one CTA per SM owning R = ceil(m / G) rows of C and X in
  // shared memory for the whole solve (single rank, zero/quadratic).
  void plan_resident() {
    res_G = 0;
    res_R = 0;
    res_smem = 0;
    if (!allow_resident || sharded || m_loc < 1 || reg_kind == OTDR_REG_GROUP_LASSO) return;
    int max_smem = 0;
    CK(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, cfg.device));
    const long long G = std::min<long long>(num_sms, m_loc);
    const long long R = (m_loc + G - 1) / G;
    res_wide = false;
    size_t bytes = f64() ? otdrk::resident_smem_bytes<double>(R, n, ld)
                         : otdrk::resident_smem_bytes<float>(R, n, ld);
    if (!f64() && res_allow_wide) {
      const size_t wide = otdrk::resident_smem_bytes<double>(R, n, ld);
      if (wide + 2048 <= size_t(max_smem)) {
        bytes = wide;
        res_wide = true;
      }
    }
    if (bytes + 2048 > size_t(max_smem)) return;
    res_G = int((m_loc + R - 1) / R);
    res_R = int(R);
    res_smem = bytes;
    if (!gscratch) gscratch = dalloc<double>(size_t(num_sms) * size_t(n + 4));
  }

  // Streaming plan: P co-resident CTAs claiming (row group, stripe) tiles of
  // the plain sweep's geometry (rows_per_cta x 256 columns).
  void plan_stream() {
    str_P = 0;
    if (!allow_stream || (sharded && !p2p) || m_loc < 1 || reg_kind == OTDR_REG_GROUP_LASSO) return;
    int occ = 0;
    if (str_d < 0) str_d = default_stream_d();
    cudaLaunchConfig_t lc{};
    if (use_tstream()) tstream_dispatch(lc, otdrk::StreamArgs{}, &occ);
    else stream_dispatch(lc, otdrk::StreamArgs{}, &occ);
    if (occ < 1) return;
    long long P = (long long)num_sms * occ;
    // OTDR_STREAM_GRID caps the persistent grid (several ranks' kernels
    // sharing one GPU in the multi-context tests must all be co-resident)
    if (const char* sg = std::getenv("OTDR_STREAM_GRID")) P = std::max(1LL, std::min(P, std::atoll(sg)));
    const long long S = (ld + otdrk::kStreamTN - 1) / otdrk::kStreamTN;
    // long tiles (the plain sweep's rows_per_cta), short ones for the last
    // stripes, about two rounds of long tiles' worth of rows
    // about str_tpc long tiles per CTA (OTDR_STREAM_TILES)
    // (>= 128 rows: shorter tiles cost more in pipeline fill and partial
    // folds than they gain in balance -- measured at 4000^2)
    const long long min_rows = std::getenv("OTDR_STREAM_MINROWS") ? std::atoll(std::getenv("OTDR_STREAM_MINROWS")) : 128;
    // str_tpc = 0 (default): 6 long tiles per CTA below 1M tile-rows (cfg2
    // 10000^2, 5000-row bands: 3.5 % / 2 % faster), 8 above (20000^2 and up;
    // profiles/r01g_stream_policy.txt)
    const long long tpc = str_tpc > 0 ? str_tpc : (m_loc * S < 1000000 ? 6 : 8);
    const long long big = std::min<long long>(
        std::max<long long>(1, m_loc), std::max<long long>(min_rows, (m_loc * S + tpc * P - 1) / (tpc * P)));
    // short tail tiles: a quarter of a long tile, but >= 96 rows (smaller tiles
    // cost more in per-tile pipeline fill than they save in tail; measured at
    // 10000^2 and 20000^2)
    const long long small = std::min(big, std::max<long long>(std::min<long long>(96, min_rows), big / std::max(1, str_tail)));
    const long long tail_stripes =
        str_tail > 1 ? std::min<long long>(S, (P * big + m_loc - 1) / m_loc) : 0;
    // TMA kernel: tiles are whole blocks of ts_rb() rows (a block never
    // straddles two tiles, and phi block copies stay 16-byte aligned)
    const long long rb = use_tstream() ? ts_rb() : 1;
    auto rnd = [&](long long v) { return (v + rb - 1) / rb * rb; };
    str_big = int(rnd(big));
    str_small = int(rnd(small));
    // Final wave: the last fin stripes are cut into short tiles (about one
    // tile per CTA in all), so the sweep ends on ~fin-row tiles instead of a
    // 96..128-row one (the one-tile finish spread of the sweep); their column
    // folds move from the completing CTA to phase B, one stripe per CTA in
    // parallel (a stripe of many short tiles would otherwise put a long fold
    // on the critical path). Off by default: at the 2500-row band the fold
    // costs more than the narrower tail saves (OTDR_STREAM_FIN=1 enables it).
    long long fin_rows = std::max<long long>(32, rnd((m_loc + P - 1) / P));
    long long fin = 0;
    if (str_fin && S > 1) {
      const long long per = (m_loc + fin_rows - 1) / fin_rows;
      fin = std::min<long long>({(P + per - 1) / per, S - 1, P});
    }
    fin_rows = rnd(fin_rows);
    std::vector<int> first;
    std::vector<int4> tiles;
    for (long long st = 0; st < S; ++st) {
      first.push_back(int(tiles.size()));
      const long long R = st >= S - fin ? fin_rows : st >= S - tail_stripes ? str_small : str_big;
      for (long long r0 = 0; r0 < m_loc; r0 += R)
        tiles.push_back(int4{int(st), int(r0), int(std::min(m_loc, r0 + R)), 0});
    }
    first.push_back(int(tiles.size()));
    const long long ntiles = (long long)tiles.size();
    str_fin_first = int(S - fin);
    if (d_tiles) cudaFree(d_tiles);
    d_tiles = dalloc<int4>(tiles.size());
    CK(cudaMemcpy(d_tiles, tiles.data(), tiles.size() * sizeof(int4), cudaMemcpyHostToDevice));
    for (void* ptr : {(void*)str_part, (void*)str_colpart, (void*)d_sfirst,
                      (void*)d_scnt, (void*)str_sspart})
      if (ptr) cudaFree(ptr);
    d_scnt = dalloc<unsigned>(size_t(S));
    CK(cudaMemset(d_scnt, 0, size_t(S) * sizeof(unsigned)));
    str_sspart = dalloc<double>(size_t(S));
    str_part = dalloc<double>(size_t(std::max<long long>(P, num_sms)) * 4);
    str_part_cap = size_t(std::max<long long>(P, num_sms)) * 4;
    str_colpart = dalloc<double>(size_t(ntiles) * otdrk::kStreamTN);
    d_sfirst = dalloc<int>(first.size());
    CK(cudaMemcpy(d_sfirst, first.data(), first.size() * sizeof(int), cudaMemcpyHostToDevice));
    str_ntiles = int(ntiles);
    str_P = int(P);
  }

  // cp.async queue depth (rows in flight per warp, OTDR_STREAM_D); 0 = register-staged sweep
  int str_d = -1;
  // measured (profiles/r01g_stream_knobs_20000.txt): fp32 3 beats 4 by 0.3 % at
  // 10000^2..40000^2 and 1.2 % on 2500-row bands; fp64 2 beats 3 by 1.5 %
  int default_stream_d() const { return f64() ? 2 : 3; }
  template <typename T, int REG, int D>
  static constexpr size_t stream_smem_of() {
    return D > 0 ? otdrk::stream_async_smem<T, sizeof(T) == 8 ? 4 : 2, D>() : 0;
  }
  template <typename T, int REG, int D>
  void stream_call(cudaLaunchConfig_t& lc, const otdrk::StreamArgs& sa, int* occ) {
    constexpr bool E = sizeof(T) == 8;
    constexpr int NV = E ? 4 : 2, U = E ? 1 : 2;
    stream_launch(otdrk::stream_kernel<T, REG, E, NV, U, D>, stream_smem_of<T, REG, D>(), lc, sa, occ);
  }
  template <typename K>
  void stream_launch(K kern, size_t smem, cudaLaunchConfig_t& lc, const otdrk::StreamArgs& sa, int* occ) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    if (occ) {
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, kern, otdrk::kThreads, smem));
      return;
    }
    lc.dynamicSmemBytes = smem;
    CK(cudaLaunchKernelEx(&lc, kern, sa));
  }
  template <typename T, int REG>
  void stream_dispatch_d(cudaLaunchConfig_t& lc, const otdrk::StreamArgs& sa, int* occ) {
    switch (str_d) {
      case 0: stream_call<T, REG, 0>(lc, sa, occ); break;
      case 2: stream_call<T, REG, 2>(lc, sa, occ); break;
      case 3: stream_call<T, REG, 3>(lc, sa, occ); break;
      case 4: stream_call<T, REG, 4>(lc, sa, occ); break;
      default: stream_call<T, REG, 5>(lc, sa, occ); break;
    }
  }
  void stream_dispatch(cudaLaunchConfig_t& lc, const otdrk::StreamArgs& sa, int* occ) {
    const bool quad = reg_kind == OTDR_REG_QUAD;
    if (f64()) {
      if (quad) stream_dispatch_d<double, otdrk::REG_QUAD>(lc, sa, occ);
      else stream_dispatch_d<double, otdrk::REG_NONE>(lc, sa, occ);
    } else {
      if (quad) stream_dispatch_d<float, otdrk::REG_QUAD>(lc, sa, occ);
      else stream_dispatch_d<float, otdrk::REG_NONE>(lc, sa, occ);
    }
  }

  // ---- TMA-producer streaming kernel (otdr_tstream.cuh)
  // geometry (consumer warps, rows per block, ring stages, CTAs per SM):
  // 4/8/3/3 by default; OTDR_TS_CFG=1: 8/8/5/2, 2: 16/16/5/1
  int ts_rb() const { return ts_cfg == 2 ? 16 : 8; }
  template <typename T, int REG, int NCW, int RB, int S, int MINB>
  void tstream_call(cudaLaunchConfig_t& lc, const otdrk::StreamArgs& sa, int* occ) {
    constexpr bool E = sizeof(T) == 8;
    auto kern = otdrk::tstream_kernel<T, REG, E, NCW, RB, S, MINB>;
    constexpr size_t smem = otdrk::TSLayout<T, NCW, RB, S>::kBytes;
    constexpr int nt = (NCW + 1) * 32;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    if (occ) {
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, kern, nt, smem));
      return;
    }
    if (!ts_maps) {
      encode_map(&ts_mapX, X, otdrk::kStreamTN, RB);
      encode_map(&ts_mapC, C, otdrk::kStreamTN, RB);
      ts_maps = true;
    }
    lc.blockDim = dim3(unsigned(nt), 1, 1);
    lc.dynamicSmemBytes = smem;
    CK(cudaLaunchKernelEx(&lc, kern, sa, ts_mapX, ts_mapC));
  }
  template <typename T, int REG>
  void tstream_dispatch_t(cudaLaunchConfig_t& lc, const otdrk::StreamArgs& sa, int* occ) {
    // fp32: three CTAs per SM of 4 consumer warps (two rows per warp per
    // block) + a producer warp, 3-stage ring of 8-row blocks (~63 KB per CTA);
    // OTDR_TS_CFG=1: the round-2 geometry (two CTAs of 8 consumer warps, one
    // row each, 5 stages), 2: one CTA of 16 consumer warps, 16-row blocks
    //
    if (ts_cfg == 1) tstream_call<T, REG, 8, 8, 5, 2>(lc, sa, occ);
    else if (ts_cfg == 2) tstream_call<T, REG, 16, 16, 5, 1>(lc, sa, occ);
    else tstream_call<T, REG, 4, 8, 3, 3>(lc, sa, occ);
  }
  void tstream_dispatch(cudaLaunchConfig_t& lc, const otdrk::StreamArgs& sa, int* occ) {
    const bool quad = reg_kind == OTDR_REG_QUAD;
    if (quad) tstream_dispatch_t<float, otdrk::REG_QUAD>(lc, sa, occ);
    else tstream_dispatch_t<float, otdrk::REG_NONE>(lc, sa, occ);
  }
  // the bulk-copy kernels cover fp32 storage; fp64 rows (2 KB per 256
  // columns) keep the per-thread cp.async kernel
  bool use_tstream() const { return str_kind == 1 && !f64(); }

  bool stream_active(bool track, bool cert) const {
    return str_P > 0 && res_G == 0 && !track && !cert && (!prm.fused || str_d > 0);
  }

  void launch_stream(long long iters) {
    const long long S = (ld + otdrk::kStreamTN - 1) / otdrk::kStreamTN;
    otdrk::StreamArgs sa{X, C, phi, a, r, p, psi, b, s, q, rowpart, str_colpart,
                         d_sfirst, d_scnt, str_sspart, str_part, d_ctl, d_prm, m_loc, n, ld, int(S), str_ntiles,
                         iters, nullptr, m_glob, sharded ? d_peers : nullptr, rbuf, d_xep,
                         cfg.rank, cfg.nranks};
    sa.tiles = d_tiles;
    sa.fin_first = str_fin_first;
    static const bool trace = std::getenv("OTDR_STREAM_TRACE") != nullptr;
    unsigned long long* ts = nullptr;
    const size_t tsn = size_t(otdrk::kTraceIters) * size_t(str_P + 12);
    if (trace) {
      ts = dalloc<unsigned long long>(tsn);
      CK(cudaMemset(ts, 0, tsn * 8));
      sa.tstamp = ts;
    }
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(unsigned(str_P), 1, 1);
    lc.blockDim = dim3(otdrk::kThreads, 1, 1);
    lc.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    if (use_tstream()) tstream_dispatch(lc, sa, nullptr);
    else stream_dispatch(lc, sa, nullptr);
    if (trace) {  // debug: per-iteration phase times of the first iterations
      std::vector<unsigned long long> h(tsn);
      CK(cudaStreamSynchronize(stream));
      CK(cudaMemcpy(h.data(), ts, tsn * 8, cudaMemcpyDeviceToHost));
      cudaFree(ts);
      for (int it = 0; it < otdrk::kTraceIters; ++it) {
        const unsigned long long* row = h.data() + size_t(it) * size_t(str_P + 12);
        const unsigned long long t0 = row[str_P];
        if (!t0) break;
        unsigned long long mn = ~0ull, mx = 0;
        for (int c = 0; c < str_P; ++c) {
          mn = std::min(mn, row[c]);
          mx = std::max(mx, row[c]);
        }
        std::fprintf(stderr,
                     "stream it %d: sweep first %.1f last %.1f us | bar1 %.1f | rows %.1f cols %.1f | B %.1f | bar2 %.1f | C %.1f\n",
                     it, (mn - t0) * 1e-3, (mx - t0) * 1e-3, (row[str_P + 1] - t0) * 1e-3,
                     (row[str_P + 5] - t0) * 1e-3, (row[str_P + 6] - t0) * 1e-3,
                     (row[str_P + 2] - t0) * 1e-3, (row[str_P + 3] - t0) * 1e-3,
                     (row[str_P + 4] - t0) * 1e-3);
        if (row[str_P + 8])
          std::fprintf(stderr, "   peer: published %.1f waited %.1f cols+rows %.1f bar %.1f\n",
                       (row[str_P + 8] - t0) * 1e-3, (row[str_P + 9] - t0) * 1e-3,
                       (row[str_P + 10] - t0) * 1e-3, (row[str_P + 11] - t0) * 1e-3);
        if (it == 1) {
          std::vector<double> dv(static_cast<size_t>(str_P));
          for (int c = 0; c < str_P; ++c) dv[size_t(c)] = (row[c] - t0) * 1e-3;
          std::fprintf(stderr, "  per-CTA sweep end (us):");
          for (int c = 0; c < str_P; ++c) std::fprintf(stderr, " %.0f", dv[size_t(c)]);
          std::fprintf(stderr, "\n");
        }
      }
    }
  }

  bool resident_active(bool track, bool cert) const {
    return res_G > 0 && !track && !cert && !prm.fused;
  }

  void launch_resident(long long iters) {
    otdrk::ResidentArgs ra{X, C, 0, phi, a, r, p, psi, b, s, q, d_ctl, d_prm, gscratch,
                           m_loc, n, ld, res_R, res_G,
                           reg_kind == OTDR_REG_QUAD ? otdrk::REG_QUAD : otdrk::REG_NONE, iters};
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(unsigned(res_G), 1, 1);
    lc.blockDim = dim3(otdrk::kRT, 1, 1);
    lc.dynamicSmemBytes = res_smem;
    lc.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    if (f64()) {
      auto kern = otdrk::resident_kernel<double, false>;
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(res_smem)));
      CK(cudaLaunchKernelEx(&lc, kern, ra));
    } else if (res_wide) {
      auto kern = otdrk::resident_kernel<double, false, float>;
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(res_smem)));
      CK(cudaLaunchKernelEx(&lc, kern, ra));
    } else {
      auto kern = otdrk::resident_kernel<float, false>;
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(res_smem)));
      CK(cudaLaunchKernelEx(&lc, kern, ra));
    }
  }

  // TMA tile plan: column stripes of 256 B (else 512 B) per box row, R <= 256
  // rows per CTA (TMA box limit), a cluster of K <= 8 CTAs per class
  // segment, <= ~72 KB of tiles per CTA so three CTAs share an SM.
  // Group-lasso sweep plan: the pipelined single-pass kernel when a class
  // segment's staging fits shared memory (OTDR_GL_KERNEL=twopass forces the
  // two-phase gl_sweep_kernel, which also serves fused / traced iterations).
  void plan_gl() {
    gl_stripes = int((ld + tn_seg() - 1) / tn_seg());
    glp_G = 0;
    glp_groups = 0;
    glp_smem = 0;
    if (reg_kind != OTDR_REG_GROUP_LASSO || m_loc == 0) return;
    long long lmax = 0;
    for (const Segment& sg : segs) lmax = std::max(lmax, sg.end - sg.begin);
    if (lmax == 0) return;
    {  // pipelined kernel (default): deepest cp.async queue whose staging fits
      const char* gk0 = std::getenv("OTDR_GL_KERNEL");
      if (!gk0 || std::strcmp(gk0, "pipe") == 0) {
        int max_smem = 0;
        CK(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, cfg.device));
        glp_wb = 128;
        if (const char* gw = std::getenv("OTDR_GL_PIPE_W")) glp_wb = std::atoi(gw) == 64 ? 64 : 128;
        int dmax = glp_wb == 64 ? 8 : 4;
        if (const char* gd = std::getenv("OTDR_GL_PIPE_D")) dmax = std::max(2, std::min(dmax, std::atoi(gd)));
        const std::vector<int> ds = glp_wb == 64 ? std::vector<int>{8, 6, 4} : std::vector<int>{4, 3, 2};
        for (int d : ds) {
          if (d > dmax) continue;
          const size_t need = glpipe_smem(f64(), d, glp_wb, int(lmax));
          if (need + 1024 <= size_t(max_smem)) {
            glp_d = d;
            glp_smem = need;
            break;
          }
        }
        if (glp_smem) {
          const long long W = glp_wb / (long long)esz;
          glp_nstr = int((ld + W - 1) / W);
          glp_G = 10;
          if (const char* ge = std::getenv("OTDR_GL_PIPE_G"))
            glp_G = std::max(1, std::min(otdrk::kGLPMaxG, std::atoi(ge)));
          // stripe positions: runs of glp_G stripes, then runs of 2 for the
          // last ~2 items per CTA (claimed last, position-major)
          const long long tail_items = 2LL * num_sms;
          long long tail_str = std::min<long long>(glp_nstr, 2 * ((tail_items + num_segs - 1) / num_segs));
          std::vector<int2> pos;
          const long long head = glp_nstr - tail_str;
          for (long long s0 = 0; s0 < head; s0 += glp_G)
            pos.push_back(int2{int(s0), int(std::min<long long>(glp_G, head - s0))});
          for (long long s0 = head; s0 < glp_nstr; s0 += 2)
            pos.push_back(int2{int(s0), int(std::min<long long>(2, glp_nstr - s0))});
          glp_groups = int(pos.size());
          // persistent GL solve: one CTA per SM must be co-resident (cooperative)
          gls_grid = 0;
          {
            int occ = 0;
            const void* kern = f64() ? (glp_wb == 64 ? (const void*)otdrk::gl_stream_kernel<double, true, 4, 64>
                                                     : (const void*)otdrk::gl_stream_kernel<double, true, 4, 128>)
                                     : (glp_wb == 64 ? (const void*)otdrk::gl_stream_kernel<float, false, 4, 64>
                                                     : (const void*)otdrk::gl_stream_kernel<float, false, 4, 128>);
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(glp_smem)));
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, otdrk::kGLPThreads, glp_smem));
            if (occ >= 1) {
              gls_grid = num_sms;
              if (const char* gg = std::getenv("OTDR_GL_PIPE_GRID")) gls_grid = std::max(1, std::min(gls_grid, std::atoi(gg)));
              if (!str_part || str_part_cap < size_t(gls_grid) * 4) {
                if (str_part) cudaFree(str_part);
                str_part = dalloc<double>(size_t(std::max(gls_grid, 2 * num_sms)) * 4);
                str_part_cap = size_t(std::max(gls_grid, 2 * num_sms)) * 4;
              }
            }
          }
          if (d_glp_pos) cudaFree(d_glp_pos);
          d_glp_pos = dalloc<int2>(pos.size());
          CK(cudaMemcpy(d_glp_pos, pos.data(), pos.size() * sizeof(int2), cudaMemcpyHostToDevice));
          glp_lmax = int(lmax);
        }
      }
    }
  }

  void ensure_partials() {
    const int seg_stripes = int((ld + tn_seg() - 1) / tn_seg());
    const size_t need_row = size_t(std::max(std::max(stripes, gl_stripes), std::max(seg_stripes, glp_groups))) *
                            size_t(std::max<long long>(m_loc, 1));
    const size_t need_col = size_t(std::max(rowgroups, num_segs)) * size_t(ld);
    const size_t need_c = size_t(cert_stripes) * size_t(num_cert_segs) * otdrk::kCertVals;
    if (need_row > rowpart_cap) {
      if (rowpart) cudaFree(rowpart);
      rowpart = dalloc<double>(need_row);
      rowpart_cap = need_row;
    }
    if (need_col > colpart_cap) {
      if (colpart) cudaFree(colpart);
      colpart = dalloc<double>(need_col);
      colpart_cap = need_col;
    }
    if (need_c > cpart_cap) {
      if (cpart) cudaFree(cpart);
      cpart = dalloc<double>(need_c);
      cpart_cap = need_c;
    }
  }

  void invalidate_graphs() {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    graphs.clear();
  }

  // ---------------------------------------------------------------- ctl I/O
  void pull_ctl() {
    CK(cudaMemcpyAsync(h_ctl, d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
  }
  void push_ctl() {
    CK(cudaMemcpyAsync(d_ctl, h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, stream));
  }
  void push_prm() {
    CK(cudaMemcpyAsync(d_prm, &prm, sizeof(Params), cudaMemcpyHostToDevice, stream));
    CK(cudaStreamSynchronize(stream));  // prm is a host member reused by later calls
  }

  void set_rho_params(double rho) {
    prm.rho = rho;
    prm.alpha = reg_kind == OTDR_REG_QUAD ? reg_param : 0.0;
    prm.lambda = reg_kind == OTDR_REG_GROUP_LASSO ? reg_param : 0.0;
    prm.quad_d = 1.0 + rho * prm.alpha;
    prm.quad_inv = 1.0 / prm.quad_d;
    prm.gl_thr = rho * prm.lambda;
  }

  // ---------------------------------------------------------------- graphs
  // kind 0: plain chunk of `count` iterations; kind 1: WHILE loop whose body
  // is `count` iterations.
  cudaGraphExec_t get_graph(int kind, int count, bool track, bool cert) {
    auto key = std::make_tuple(kind, count, track ? 1 : 0, cert ? 1 : 0, prm.fused ? 1 : 0);
    auto it = graphs.find(key);
    if (it != graphs.end()) return it->second;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ex = nullptr;
    if (kind == 0) {
      CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
      for (int t = 0; t < count; ++t) launch_iteration(track, cert, 0, 0);
      CK(cudaStreamEndCapture(stream, &g));
    } else {
      CK(cudaGraphCreate(&g, 0));
      cudaGraphConditionalHandle h;
      CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
      cudaGraphNodeParams np{};
      np.type = cudaGraphNodeTypeConditional;
      np.conditional.handle = h;
      np.conditional.type = cudaGraphCondTypeWhile;
      np.conditional.size = 1;
      cudaGraphNode_t node;
      CK(cudaGraphAddNode(&node, g, nullptr, 0, &np));
      cudaGraph_t body = np.conditional.phGraph_out[0];
      CK(cudaStreamBeginCaptureToGraph(stream, body, nullptr, nullptr, 0,
                                       cudaStreamCaptureModeThreadLocal));
      for (int t = 0; t < count; ++t) launch_iteration(track, cert, h, 1);
      CK(cudaStreamEndCapture(stream, &body));
    }
    CK(cudaGraphInstantiate(&ex, g, 0));
    CK(cudaGraphDestroy(g));
    graphs[key] = ex;
    return ex;
  }

  // Raw iterations (step): graph chunks plus a directly launched remainder.
  void run_raw(long long iters) {
    if (iters > 0 && resident_active(false, false)) {
      launch_resident(iters);
      check_launch();
      return;
    }
    if (iters > 0 && stream_active(false, false)) {
      launch_stream(iters);
      check_launch();
      return;
    }
    if (iters > 0 && gl_stream_active(false, false)) {
      launch_gl_stream(iters);
      check_launch();
      return;
    }
    const int chunk = 16;
    if (iters >= chunk) {
      cudaGraphExec_t ex = get_graph(0, chunk, false, false);
      for (long long t = 0; t + chunk <= iters; t += chunk) CK(cudaGraphLaunch(ex, stream));
    }
    for (long long t = 0; t < iters % chunk; ++t) launch_iteration(false, false, 0, 0);
    check_launch();
  }

  // ---------------------------------------------------------------- upload
  // Host rows move through two pinned chunks: host threads convert chunk c
  // (fp64 -> storage type, so fp32 storage crosses PCIe at 4 B/entry) while
  // the copy engine moves chunk c-1 and a kernel scatters it into the padded,
  // device-ordered rows. Works the same for pageable and pinned sources.
  void* hpin[2] = {nullptr, nullptr};
  cudaEvent_t ev_pin[2] = {nullptr, nullptr};
  size_t stage_bytes = 0;

  void ensure_pinned() {
    for (int b = 0; b < 2; ++b) {
      if (!hpin[b]) CK(cudaHostAlloc(&hpin[b], kPinBytes, cudaHostAllocDefault));
      if (!ev_pin[b]) {
        CK(cudaEventCreateWithFlags(&ev_pin[b], cudaEventDisableTiming));
        CK(cudaEventRecord(ev_pin[b], stream));
      }
    }
  }
  template <typename T>
  long long chunk_rows() const {
    const size_t cap = std::min(kPinBytes, stage_bytes / 2);
    return std::max<long long>(1, (long long)(cap / (size_t(n) * sizeof(T))));
  }

  template <typename T>
  void upload_rows(T* dst, const double* src_rows) {
    if (m_loc == 0) return;
    ensure_pinned();
    const long long rows_per = chunk_rows<T>();
    int c = 0;
    for (long long r0 = 0; r0 < m_loc; r0 += rows_per, ++c) {
      const int b = c & 1;
      const long long rows = std::min(rows_per, m_loc - r0), cnt = rows * n;
      CK(cudaEventSynchronize(ev_pin[b]));  // the DMA of chunk c-2 has left hpin[b]
      T* hb = static_cast<T*>(hpin[b]);
      const double* sp = src_rows + r0 * n;
      host_parallel(cnt, [hb, sp](long long lo, long long hi) {
        if (sizeof(T) == sizeof(double)) std::memcpy(hb + lo, sp + lo, size_t(hi - lo) * 8);
        else
          for (long long t = lo; t < hi; ++t) hb[t] = T(sp[t]);  // round to nearest (= device cvt.rn)
      });
      T* db = reinterpret_cast<T*>(reinterpret_cast<char*>(stage) + size_t(b) * (stage_bytes / 2));
      CK(cudaMemcpyAsync(db, hb, size_t(cnt) * sizeof(T), cudaMemcpyHostToDevice, stream));
      CK(cudaEventRecord(ev_pin[b], stream));
      otdrk::scatter_rows_kernel<T, T><<<4 * kNumSMs, 256, 0, stream>>>(dst, db, d_dev_row + r0, rows,
                                                                        n, ld);
      check_launch();
    }
    CK(cudaStreamSynchronize(stream));
  }

  template <typename T>
  void download_rows(double* dst_rows, const T* src) {
    if (m_loc == 0) return;
    ensure_pinned();
    const long long rows_per = chunk_rows<T>();
    const long long nch = (m_loc + rows_per - 1) / rows_per;
    auto enqueue = [&](long long c) {
      const int b = int(c & 1);
      const long long r0 = c * rows_per, rows = std::min(rows_per, m_loc - r0);
      T* db = reinterpret_cast<T*>(reinterpret_cast<char*>(stage) + size_t(b) * (stage_bytes / 2));
      otdrk::gather_rows_kernel<T, T><<<4 * kNumSMs, 256, 0, stream>>>(db, src, d_dev_row + r0, rows,
                                                                       n, ld);
      check_launch();
      CK(cudaMemcpyAsync(hpin[b], db, size_t(rows * n) * sizeof(T), cudaMemcpyDeviceToHost, stream));
      CK(cudaEventRecord(ev_pin[b], stream));
    };
    enqueue(0);
    for (long long c = 0; c < nch; ++c) {
      if (c + 1 < nch) enqueue(c + 1);  // hpin[(c+1)&1] was drained by the host last trip
      const int b = int(c & 1);
      CK(cudaEventSynchronize(ev_pin[b]));
      const long long r0 = c * rows_per, rows = std::min(rows_per, m_loc - r0);
      const T* hb = static_cast<const T*>(hpin[b]);
      double* dp = dst_rows + r0 * n;
      host_parallel(rows * n, [hb, dp](long long lo, long long hi) {
        if (sizeof(T) == sizeof(double)) std::memcpy(dp + lo, hb + lo, size_t(hi - lo) * 8);
        else
          for (long long t = lo; t < hi; ++t) dp[t] = double(hb[t]);
      });
    }
  }

  void upload_vec_rows(double* dst, const double* host_order) {
    std::vector<double> tmp(size_t(std::max<long long>(m_loc, 1)));
    for (long long h = 0; h < m_loc; ++h) tmp[size_t(dev_row[h])] = host_order[h];
    CK(cudaMemcpy(dst, tmp.data(), size_t(m_loc) * sizeof(double), cudaMemcpyHostToDevice));
  }
  void download_vec_rows(double* host_order, const double* src) {
    std::vector<double> tmp(size_t(std::max<long long>(m_loc, 1)));
    CK(cudaMemcpy(tmp.data(), src, size_t(m_loc) * sizeof(double), cudaMemcpyDeviceToHost));
    for (long long h = 0; h < m_loc; ++h) host_order[h] = tmp[size_t(dev_row[h])];
  }

  // Re-order device rows of C (and p) when the GL class permutation changes.
  void permute_rows(const std::vector<long long>& new_row) {
    if (new_row == dev_row) return;
    if (has_problem) {
      void* tmp = nullptr;
      const size_t bytes = size_t(m_loc) * size_t(ld) * esz;
      CK(cudaMalloc(&tmp, bytes));
      long long* d_new = dalloc<long long>(size_t(m_loc));
      CK(cudaMemcpy(d_new, new_row.data(), size_t(m_loc) * 8, cudaMemcpyHostToDevice));
      const long long units = ld * (long long)esz / 16;
      otdrk::move_rows_kernel<<<4 * kNumSMs, 256, 0, stream>>>(
          static_cast<uint4*>(tmp), static_cast<const uint4*>(C), d_new, d_dev_row, m_loc, units);
      check_launch();
      CK(cudaStreamSynchronize(stream));
      cudaFree(d_new);
      if (c_vmm) {
        comp_free(C, c_vmm);
        c_vmm = 0;
        c_comp = false;
      } else {
        CK(cudaFree(C));
      }
      C = tmp;
      invalidate_graphs();
    }
    dev_row = new_row;
    CK(cudaMemcpy(d_dev_row, dev_row.data(), size_t(m_loc) * sizeof(long long),
                  cudaMemcpyHostToDevice));
    if (has_problem) upload_vec_rows(p, h_p.data());
    has_state = false;
  }

  // make_state from the X currently in the X buffer and phi/psi buffers.
  void seed_state() {
    CK(cudaMemsetAsync(d_ctl, 0, sizeof(Ctl), stream));
    prm.solving = 0;
    prm.fused = 0;
    push_prm();
    launch_sweep(false, true);
    launch_reduce(true, false);
    launch_exchange(exch, size_t(n) + 3);
    otdrk::SeedArgs sa{exch, q, r, phi, psi, s, a, b, d_ctl, m_loc, m_glob, n};
    const long long cnt = std::max(m_loc, n);
    otdrk::seed_state_kernel<<<int((cnt + 255) / 256), 256, 0, stream>>>(sa);
    check_launch();
    CK(cudaStreamSynchronize(stream));
    has_state = true;
  }

  void release() {
    invalidate_graphs();
    if (x_vmm) {
      comp_free(X, x_vmm);
      X = nullptr;
    }
    if (c_vmm) {
      comp_free(C, c_vmm);
      C = nullptr;
    }
    if (d_tiles) cudaFree(d_tiles);
    void* ptrs[] = {C, X, p, q, phi, psi, a, b, r, s, rowpart, colpart, exch, bpart, cpart,
                    str_part, str_colpart, d_sfirst, d_scnt, str_sspart, d_glp_pos,
                    csum, stage, gscratch, d_dev_row, d_seg, d_cert_seg, d_prm, d_ctl, d_trace, d_mx};
    for (void* ptr : ptrs)
      if (ptr) cudaFree(ptr);
    if (h_ctl) cudaFreeHost(h_ctl);
    for (int b = 0; b < 2; ++b) {
      if (hpin[b]) cudaFreeHost(hpin[b]);
      if (ev_pin[b]) cudaEventDestroy(ev_pin[b]);
    }
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (stream) cudaStreamDestroy(stream);
    if (comm && nccl().ok) nccl().CommDestroy(comm);
    for (void* ptr : ipc_opened) cudaIpcCloseMemHandle(ptr);
    if (rbuf) cudaFree(rbuf);
    if (d_peers) cudaFree(d_peers);
    if (d_xep) cudaFree(d_xep);
  }
};

namespace {

otdr_status fail(otdr_dev* ctx, otdr_status code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

template <typename F>
otdr_status guarded(otdr_dev* ctx, F&& f) {
  try {
    if (ctx) CK(cudaSetDevice(ctx->cfg.device));
    return f();
  } catch (const Error& e) {
    return fail(ctx, e.code, e.msg);
  } catch (const std::exception& e) {
    return fail(ctx, OTDR_E_CUDA, e.what());
  }
}

}  // namespace

extern "C" {

int otdr_dev_nccl_unique_id(unsigned char* out128) {
  if (!nccl().ok) return OTDR_E_NCCL;
  ncclUniqueId id;
  if (nccl().GetUniqueId(&id) != ncclSuccess) return OTDR_E_NCCL;
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  std::memcpy(out128, &id, sizeof(id));
  return OTDR_OK;
}

int otdr_dev_abi_version(void) { return OTDR_DEV_ABI_VERSION; }

int otdr_dev_cuda_available(void) {
  int count = 0;
  return cudaGetDeviceCount(&count) == cudaSuccess && count > 0 ? 1 : 0;
}

const char* otdr_dev_last_error(const otdr_dev* ctx) { return ctx ? ctx->err.c_str() : ""; }

int otdr_dev_solve_path(const otdr_dev* ctx) {
  if (!ctx) return OTDR_PATH_GRAPH;
  if (ctx->resident_active(false, false)) return OTDR_PATH_RESIDENT;
  if (ctx->stream_active(false, false) || ctx->gl_stream_active(false, false)) return OTDR_PATH_STREAM;
  return OTDR_PATH_GRAPH;
}

const char* otdr_dev_kernel_name(const otdr_dev* ctx) {
  if (!ctx) return "";
  otdr_dev* c = const_cast<otdr_dev*>(ctx);
  const char* st = c->f64() ? "f64" : "f32";
  const char* rg = c->reg_kind == OTDR_REG_QUAD ? "quad" : c->reg_kind == OTDR_REG_GROUP_LASSO ? "group-lasso" : "none";
  const int path = otdr_dev_solve_path(ctx);
  if (path == OTDR_PATH_RESIDENT)
    c->kname = std::string("resident_kernel<") + st + (c->res_wide ? " storage, f64 tiles" : "") + ", " + rg + ">";
  else if (path == OTDR_PATH_STREAM && c->reg_kind == OTDR_REG_GROUP_LASSO)
    c->kname = std::string("gl_stream_kernel<") + st + ">";
  else if (path == OTDR_PATH_STREAM) {
    c->kname = std::string(c->use_tstream() ? "tstream_kernel" : "stream_kernel") + "<" + st + ", " + rg + ">";
  } else c->kname = std::string("sweep + reduce + update graph<") + st + ", " + rg + ">";
  return c->kname.c_str();
}

otdr_status otdr_dev_peer_export(otdr_dev* ctx, void* handle) {
  if (!ctx || !handle) return OTDR_E_INVALID_ARG;
  return guarded(ctx, [&] {
    ctx->alloc_rbuf();
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, ctx->rbuf));
    std::memcpy(handle, &h, sizeof(h));
    return OTDR_OK;
  });
}

otdr_status otdr_dev_peer_import(otdr_dev* ctx, const void* handles) {
  if (!ctx || !handles) return OTDR_E_INVALID_ARG;
  return guarded(ctx, [&] {
    ctx->alloc_rbuf();
    const int nr = ctx->cfg.nranks;
    std::vector<double*> peers(static_cast<size_t>(nr), nullptr);
    for (int r = 0; r < nr; ++r) {
      if (r == ctx->cfg.rank) {
        peers[size_t(r)] = ctx->rbuf;
        continue;
      }
      cudaIpcMemHandle_t h;
      std::memcpy(&h, static_cast<const unsigned char*>(handles) + size_t(r) * OTDR_PEER_HANDLE_BYTES,
                  sizeof(h));
      void* ptr = nullptr;
      CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
      ctx->ipc_opened.push_back(ptr);
      peers[size_t(r)] = static_cast<double*>(ptr);
    }
    ctx->set_peers(peers);
    return OTDR_OK;
  });
}

otdr_status otdr_dev_peer_link_local(otdr_dev** ctxs, int nranks) {
  if (!ctxs || nranks < 1) return OTDR_E_INVALID_ARG;
  for (int r = 0; r < nranks; ++r) {
    if (!ctxs[r]) return OTDR_E_INVALID_ARG;
    if (ctxs[r]->cfg.nranks != nranks || ctxs[r]->cfg.rank != r || (nranks > 1 && !ctxs[r]->sharded))
      return fail(ctxs[r], OTDR_E_STATE, "contexts must be the ranks 0..nranks-1 of one sharded run");
  }
  std::vector<double*> peers(static_cast<size_t>(nranks), nullptr);
  for (int r = 0; r < nranks; ++r) {
    const otdr_status st = guarded(ctxs[r], [&] {
      ctxs[r]->alloc_rbuf();
      peers[size_t(r)] = ctxs[r]->rbuf;
      return OTDR_OK;
    });
    if (st != OTDR_OK) return st;
  }
  for (int r = 0; r < nranks; ++r) {
    const otdr_status st = guarded(ctxs[r], [&] {
      ctxs[r]->set_peers(peers);
      return OTDR_OK;
    });
    if (st != OTDR_OK) return st;
  }
  return OTDR_OK;
}

int otdr_dev_kernels_per_iteration(const otdr_dev* ctx) {
  if (otdr_dev_solve_path(ctx) != OTDR_PATH_GRAPH) return 0;
  // sweep + reduce + update (+ the NCCL all-reduce when row-sharded)
  return 3;
}

otdr_status otdr_dev_create(const otdr_dev_config* cfg, otdr_dev** out) {
  if (!cfg || !out) return OTDR_E_INVALID_ARG;
  *out = nullptr;
  if (cfg->m < 1 || cfg->n < 1) return OTDR_E_DIMENSION;
  const int nranks = cfg->nranks < 1 ? 1 : cfg->nranks;
  if (cfg->row_begin < 0 || cfg->row_end > cfg->m || cfg->row_begin > cfg->row_end)
    return OTDR_E_DIMENSION;
  if (nranks == 1 && (cfg->row_begin != 0 || cfg->row_end != cfg->m)) return OTDR_E_DIMENSION;
  if (!otdr_dev_cuda_available()) return OTDR_E_CUDA;
  otdr_dev* ctx = new otdr_dev();
  ctx->cfg = *cfg;
  ctx->cfg.nranks = nranks;
  ctx->cfg.nccl_id = nullptr;
  try {
    CK(cudaSetDevice(cfg->device));
    ctx->storage = cfg->storage == OTDR_STORE_F64 ? OTDR_STORE_F64 : OTDR_STORE_F32;
    ctx->esz = ctx->f64() ? 8 : 4;
    ctx->m_glob = cfg->m;
    ctx->n = cfg->n;
    ctx->row0 = cfg->row_begin;
    ctx->m_loc = cfg->row_end - cfg->row_begin;
    const long long vec = ctx->f64() ? 2 : 4;
    // rows start on 256-byte boundaries for n >= 1024. Measured on B200: a
    // 40000-byte fp32 row pitch (n = 10000) left every other row's 128-byte
    // chunks straddling two L2 lines (+16 % DRAM reads in the group-lasso
    // sweep); 256-byte pitches stream faster than 128-byte ones (20000^2
    // stream kernel 5.89 -> 6.04 TB/s, 10000^2 5.24 -> 5.39 TB/s).
    long long align = vec;
    if (ctx->n >= 1024) align = 256 / (long long)ctx->esz;
    if (const char* la = std::getenv("OTDR_LD_ALIGN"))
      align = std::max<long long>(vec, std::atoll(la) / (long long)ctx->esz);
    ctx->ld = (ctx->n + align - 1) / align * align;
    CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&ctx->ev0));
    CK(cudaEventCreate(&ctx->ev1));
    const size_t mat = size_t(std::max<long long>(ctx->m_loc, 1)) * size_t(ctx->ld) * ctx->esz;
    // Generic HBM compression for the plan X: once the solve settles most of
    // the plan's 128-byte lines are all zero (measured: 57-80 % at 20000^2),
    // and those travel between L2 and HBM compressed (20000^2 fp32 stream
    // kernel 1270 -> 1550+ it/s, bit-identical iterates). The gain fades and
    // then reverses beyond about 3-4 GB of compressed footprint (40000^2:
    // 6.4 GB fully compressed 314 -> 249 it/s; first 3.2 GB compressed 347),
    // so only the first OTDR_COMPRESS_GB (default 3.2) of X is compressible.
    // OTDR_COMPRESS: "x" (default, matrices >= 16 MB) / "cx" (C too; slower
    // at 20000^2) / "off".
    {
      std::string cm = mat >= (size_t(16) << 20) ? "x" : "off";
      if (const char* e = std::getenv("OTDR_COMPRESS")) cm = e;
      double cap_gb = 3.2;
      if (const char* e = std::getenv("OTDR_COMPRESS_GB")) cap_gb = std::atof(e);
      const size_t cap = size_t(std::max(0.0, cap_gb) * 1e9);
      if (cm.find('x') != std::string::npos)
        ctx->X = comp_malloc(ctx->cfg.device, mat, std::min(mat, cap), &ctx->x_vmm, &ctx->x_comp);
      if (cm.find('c') != std::string::npos)
        ctx->C = comp_malloc(ctx->cfg.device, mat, std::min(mat, cap), &ctx->c_vmm, &ctx->c_comp);
      if (!ctx->X) ctx->x_vmm = 0;
      if (!ctx->C) ctx->c_vmm = 0;
      if (cm != "off" && std::getenv("OTDR_COMPRESS_VERBOSE"))
        std::fprintf(stderr, "otdr: X vmm=%zu compressed=%d, C vmm=%zu compressed=%d\n", ctx->x_vmm,
                     int(ctx->x_comp), ctx->c_vmm, int(ctx->c_comp));
    }
    if (!ctx->C) CK(cudaMalloc(&ctx->C, mat));
    if (!ctx->X) CK(cudaMalloc(&ctx->X, mat));
    CK(cudaMemset(ctx->C, 0, mat));
    CK(cudaMemset(ctx->X, 0, mat));
    const size_t ml = size_t(std::max<long long>(ctx->m_loc, 1));
    ctx->p = dalloc<double>(ml);
    ctx->phi = dalloc<double>(ml + 64);  // padding: 16-byte cp.async of phi pairs, block bulk copies
    ctx->a = dalloc<double>(ml);
    ctx->r = dalloc<double>(ml);
    ctx->q = dalloc<double>(size_t(ctx->ld));
    // whole 256-column stripes (bulk copies of a stripe's psi)
    const size_t psi_cap = size_t((ctx->ld + otdrk::kStreamTN - 1) / otdrk::kStreamTN * otdrk::kStreamTN);
    ctx->psi = dalloc<double>(psi_cap);
    {  // -inf everywhere: columns beyond n (and beyond ld, read by the TMA
       // kernel's stripe copies) clamp to exactly 0
      const std::vector<double> ninf(psi_cap, -std::numeric_limits<double>::infinity());
      CK(cudaMemcpy(ctx->psi, ninf.data(), psi_cap * 8, cudaMemcpyHostToDevice));
    }
    ctx->b = dalloc<double>(size_t(ctx->ld));
    ctx->s = dalloc<double>(size_t(ctx->ld));
    CK(cudaMemset(ctx->q, 0, size_t(ctx->ld) * 8));
    CK(cudaMemset(ctx->b, 0, size_t(ctx->ld) * 8));
    CK(cudaMemset(ctx->s, 0, size_t(ctx->ld) * 8));
    ctx->exch = dalloc<double>(size_t(ctx->n) + 3);
    CK(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, cfg->device));
    if (const char* re = std::getenv("OTDR_RESIDENT")) ctx->allow_resident = std::strcmp(re, "off") != 0;
    if (const char* rt = std::getenv("OTDR_RESIDENT_TILES")) ctx->res_allow_wide = std::strcmp(rt, "f32") != 0;
    if (const char* st = std::getenv("OTDR_STREAM")) ctx->allow_stream = std::strcmp(st, "off") != 0;
    if (const char* gs = std::getenv("OTDR_GL_STREAM")) ctx->allow_gl_stream = std::strcmp(gs, "off") != 0;
    ctx->str_d = -1;
    if (const char* tp = std::getenv("OTDR_STREAM_TILES")) ctx->str_tpc = std::max(1, std::atoi(tp));
    if (const char* tl = std::getenv("OTDR_STREAM_TAIL")) ctx->str_tail = std::max(1, std::atoi(tl));
    if (const char* sd = std::getenv("OTDR_STREAM_D")) ctx->str_d = std::atoi(sd);
    if (const char* sk = std::getenv("OTDR_STREAM_KERNEL")) ctx->str_kind = std::strcmp(sk, "async") == 0 ? 0 : 1;
    if (const char* tc = std::getenv("OTDR_TS_CFG")) ctx->ts_cfg = std::atoi(tc);
    if (const char* fe = std::getenv("OTDR_STREAM_FIN")) ctx->str_fin = std::strcmp(fe, "1") == 0;
    ctx->plan_geometry();
    ctx->bpart = dalloc<double>(size_t(ctx->RB + ctx->CB) * 3);
    ctx->csum = dalloc<double>(otdrk::kCertVals);
    // two halves (double-buffered transfers), each at least one fp64 row
    const size_t stage_elems = std::max<size_t>(std::min(kStageDoubles, 2 * ml * size_t(ctx->n)),
                                                2 * size_t(ctx->n));
    ctx->stage = dalloc<double>(stage_elems);
    ctx->stage_bytes = stage_elems * sizeof(double);
    ctx->d_dev_row = dalloc<long long>(ml);
    ctx->dev_row.resize(size_t(ctx->m_loc));
    std::iota(ctx->dev_row.begin(), ctx->dev_row.end(), 0LL);
    CK(cudaMemcpy(ctx->d_dev_row, ctx->dev_row.data(), size_t(ctx->m_loc) * 8,
                  cudaMemcpyHostToDevice));
    ctx->d_prm = dalloc<Params>(1);
    ctx->d_ctl = dalloc<Ctl>(1);
    ctx->d_mx = dalloc<unsigned long long>(1);
    CK(cudaMallocHost(&ctx->h_ctl, sizeof(Ctl)));
    std::memset(ctx->h_ctl, 0, sizeof(Ctl));
    CK(cudaMemset(ctx->d_ctl, 0, sizeof(Ctl)));
    ctx->prm = Params{};
    ctx->set_rho_params(2.0 / double(ctx->m_glob + ctx->n));
    ctx->push_prm();
    // psi padding: -inf keeps padded columns exactly 0 through the clamp.
    std::vector<double> pad(size_t(ctx->ld), -std::numeric_limits<double>::infinity());
    CK(cudaMemcpy(ctx->psi, pad.data(), size_t(ctx->ld) * 8, cudaMemcpyHostToDevice));
    ctx->sharded = nranks > 1 || cfg->nccl_id != nullptr;
    ctx->build_segments();
    if (ctx->sharded && cfg->nccl_id) {  // a 1-rank communicator exercises the multi-GPU path on one GPU
      ncclUniqueId id;
      std::memcpy(&id, cfg->nccl_id, sizeof(id));
      NK(nccl().CommInitRank(&ctx->comm, nranks, id, cfg->rank));
    }
  } catch (const Error& e) {
    ctx->release();
    delete ctx;
    return e.code;
  }
  *out = ctx;
  return OTDR_OK;
}

void otdr_dev_destroy(otdr_dev* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->cfg.device);
  ctx->release();
  delete ctx;
}

otdr_status otdr_dev_set_problem(otdr_dev* ctx, const double* cost_rm, const double* p,
                                 const double* q) {
  if (!ctx) return OTDR_E_INVALID_ARG;
  if (!cost_rm || !p || !q) return fail(ctx, OTDR_E_INVALID_ARG, "null problem buffer");
  return guarded(ctx, [&] {
    ctx->h_p.assign(p, p + ctx->m_loc);
    ctx->h_q.assign(q, q + ctx->n);
    if (ctx->f64()) ctx->upload_rows<double>((double*)ctx->C, cost_rm);
    else ctx->upload_rows<float>((float*)ctx->C, cost_rm);
    ctx->upload_vec_rows(ctx->p, p);
    CK(cudaMemcpy(ctx->q, q, size_t(ctx->n) * 8, cudaMemcpyHostToDevice));
    ctx->has_problem = true;
    ctx->has_state = false;
    return OTDR_OK;
  });
}

otdr_status otdr_dev_build_sqdist_cost(otdr_dev* ctx, const double* src_pts,
                                       const double* tgt_pts, int d, const double* p,
                                       const double* q, int* all_zero) {
  if (!ctx) return OTDR_E_INVALID_ARG;
  if (!src_pts || !tgt_pts || !p || !q || d < 1)
    return fail(ctx, OTDR_E_INVALID_ARG, "bad point cloud arguments");
  return guarded(ctx, [&] {
    // Source points in device row order.
    std::vector<double> src(size_t(std::max<long long>(ctx->m_loc, 1)) * d);
    for (long long h = 0; h < ctx->m_loc; ++h)
      std::memcpy(&src[size_t(ctx->dev_row[h]) * d], src_pts + h * d, sizeof(double) * d);
    double* d_src = dalloc<double>(src.size());
    double* d_tgt = dalloc<double>(size_t(ctx->n) * d);
    double* d_mxv = dalloc<double>(1);
    CK(cudaMemcpy(d_src, src.data(), src.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_tgt, tgt_pts, size_t(ctx->n) * d * 8, cudaMemcpyHostToDevice));
    CK(cudaMemsetAsync(ctx->d_mx, 0, 8, ctx->stream));
    const int grid = 8 * kNumSMs;
    if (ctx->f64())
      otdrk::sqdist_kernel<double><<<grid, 256, 0, ctx->stream>>>((double*)ctx->C, d_src, d_tgt, d, ctx->m_loc, ctx->n, ctx->ld, d_mxv, ctx->d_mx, 0);
    else
      otdrk::sqdist_kernel<float><<<grid, 256, 0, ctx->stream>>>((float*)ctx->C, d_src, d_tgt, d, ctx->m_loc, ctx->n, ctx->ld, d_mxv, ctx->d_mx, 0);
    ctx->check_launch();
    CK(cudaMemcpyAsync(d_mxv, ctx->d_mx, 8, cudaMemcpyDeviceToDevice, ctx->stream));
    if (ctx->sharded) ctx->launch_exchange(d_mxv, 1, /*op_max=*/true);  // global max (normalize_cost)
    if (ctx->f64())
      otdrk::sqdist_kernel<double><<<grid, 256, 0, ctx->stream>>>((double*)ctx->C, d_src, d_tgt, d, ctx->m_loc, ctx->n, ctx->ld, d_mxv, ctx->d_mx, 1);
    else
      otdrk::sqdist_kernel<float><<<grid, 256, 0, ctx->stream>>>((float*)ctx->C, d_src, d_tgt, d, ctx->m_loc, ctx->n, ctx->ld, d_mxv, ctx->d_mx, 1);
    ctx->check_launch();
    double mx = 0.0;
    // drain the stream (incl. the max exchange) before the pageable read-back:
    // a pageable copy queued behind a spinning exchange kernel can hold the
    // driver while the other ranks of this process still need to launch
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpy(&mx, d_mxv, 8, cudaMemcpyDeviceToHost));
    cudaFree(d_src);
    cudaFree(d_tgt);
    cudaFree(d_mxv);
    if (all_zero) *all_zero = mx > 0.0 ? 0 : 1;
    ctx->h_p.assign(p, p + ctx->m_loc);
    ctx->h_q.assign(q, q + ctx->n);
    ctx->upload_vec_rows(ctx->p, p);
    CK(cudaMemcpy(ctx->q, q, size_t(ctx->n) * 8, cudaMemcpyHostToDevice));
    ctx->has_problem = true;
    ctx->has_state = false;
    return OTDR_OK;
  });
}

namespace {

struct Fd {  // RAII file descriptor
  int fd = -1;
  ~Fd() {
    if (fd >= 0) ::close(fd);
  }
};

bool pread_all(int fd, void* buf, size_t bytes, off_t off) {
  char* p = static_cast<char*>(buf);
  while (bytes > 0) {
    const ssize_t r = ::pread(fd, p, bytes, off);
    if (r <= 0) return false;
    p += r;
    off += r;
    bytes -= size_t(r);
  }
  return true;
}

bool pwrite_all(int fd, const void* buf, size_t bytes, off_t off) {
  const char* p = static_cast<const char*>(buf);
  while (bytes > 0) {
    const ssize_t r = ::pwrite(fd, p, bytes, off);
    if (r <= 0) return false;
    p += r;
    off += r;
    bytes -= size_t(r);
  }
  return true;
}

}  // namespace

otdr_status otdr_dev_read_cost_otpb(otdr_dev* ctx, const char* path, const double* p,
                                    const double* q) {
  if (!ctx) return OTDR_E_INVALID_ARG;
  if (!path || !p || !q) return fail(ctx, OTDR_E_INVALID_ARG, "null argument");
  return guarded(ctx, [&] {
    Fd f;
    f.fd = ::open(path, O_RDONLY);
    if (f.fd < 0) return fail(ctx, OTDR_E_INVALID_ARG, std::string(path) + ": cannot open");
    unsigned char hdr[16];
    if (!pread_all(f.fd, hdr, 16, 0) || std::memcmp(hdr, "OTPB", 4) != 0)
      return fail(ctx, OTDR_E_INVALID_ARG, std::string(path) + ": not an OTPB file (bad magic)");
    uint32_t m32 = 0, n32 = 0;
    std::memcpy(&m32, hdr + 4, 4);
    std::memcpy(&n32, hdr + 8, 4);
    if ((long long)m32 != ctx->m_glob || (long long)n32 != ctx->n)
      return fail(ctx, OTDR_E_DIMENSION,
                  std::string(path) + ": OTPB is " + std::to_string(m32) + "x" +
                      std::to_string(n32) + ", context is " + std::to_string(ctx->m_glob) + "x" +
                      std::to_string(ctx->n));
    const long long n = ctx->n;
    const long long rows_per = std::max<long long>(1, (long long)(kStageDoubles / size_t(n)));
    std::vector<double> host;
    for (long long r0 = 0; r0 < ctx->m_loc; r0 += rows_per) {
      const long long rows = std::min(rows_per, ctx->m_loc - r0);
      host.resize(size_t(rows * n));
      const off_t off = 16 + off_t((ctx->row0 + r0) * n) * 8;
      if (!pread_all(f.fd, host.data(), host.size() * 8, off))
        return fail(ctx, OTDR_E_INVALID_ARG, std::string(path) + ": truncated OTPB payload");
      for (size_t t = 0; t < host.size(); ++t)
        if (!(host[t] >= 0.0) || !std::isfinite(host[t]))
          return fail(ctx, OTDR_E_NEGATIVE,
                      "cost(" + std::to_string(ctx->row0 + r0 + (long long)t / n) + "," +
                          std::to_string((long long)t % n) + ") must be finite and >= 0");
      CK(cudaMemcpy(ctx->stage, host.data(), host.size() * 8, cudaMemcpyHostToDevice));
      if (ctx->f64())
        otdrk::scatter_rows_kernel<double><<<4 * kNumSMs, 256, 0, ctx->stream>>>(
            (double*)ctx->C, ctx->stage, ctx->d_dev_row + r0, rows, n, ctx->ld);
      else
        otdrk::scatter_rows_kernel<float><<<4 * kNumSMs, 256, 0, ctx->stream>>>(
            (float*)ctx->C, ctx->stage, ctx->d_dev_row + r0, rows, n, ctx->ld);
      ctx->check_launch();
      CK(cudaStreamSynchronize(ctx->stream));
    }
    ctx->h_p.assign(p, p + ctx->m_loc);
    ctx->h_q.assign(q, q + ctx->n);
    ctx->upload_vec_rows(ctx->p, p);
    CK(cudaMemcpy(ctx->q, q, size_t(ctx->n) * 8, cudaMemcpyHostToDevice));
    ctx->has_problem = true;
    ctx->has_state = false;
    return OTDR_OK;
  });
}

otdr_status otdr_dev_write_plan_otpb(otdr_dev* ctx, const char* path) {
  if (!ctx || !path) return OTDR_E_INVALID_ARG;
  if (!ctx->has_state) return fail(ctx, OTDR_E_STATE, "write_plan before set_state");
  return guarded(ctx, [&] {
    Fd f;
    const int flags = O_WRONLY | O_CREAT | (ctx->sharded ? 0 : O_TRUNC);
    f.fd = ::open(path, flags, 0644);
    if (f.fd < 0) return fail(ctx, OTDR_E_INVALID_ARG, std::string(path) + ": cannot open for writing");
    if (ctx->row0 == 0) {
      unsigned char hdr[16] = {'O', 'T', 'P', 'B'};
      const uint32_t m32 = uint32_t(ctx->m_glob), n32 = uint32_t(ctx->n);
      std::memcpy(hdr + 4, &m32, 4);
      std::memcpy(hdr + 8, &n32, 4);
      if (!pwrite_all(f.fd, hdr, 16, 0))
        return fail(ctx, OTDR_E_INVALID_ARG, std::string(path) + ": write failed");
    }
    const long long n = ctx->n;
    const long long rows_per = std::max<long long>(1, (long long)(kStageDoubles / size_t(n)));
    std::vector<double> host;
    for (long long r0 = 0; r0 < ctx->m_loc; r0 += rows_per) {
      const long long rows = std::min(rows_per, ctx->m_loc - r0);
      if (ctx->f64())
        otdrk::gather_rows_kernel<double><<<4 * kNumSMs, 256, 0, ctx->stream>>>(
            ctx->stage, (const double*)ctx->X, ctx->d_dev_row + r0, rows, n, ctx->ld);
      else
        otdrk::gather_rows_kernel<float><<<4 * kNumSMs, 256, 0, ctx->stream>>>(
            ctx->stage, (const float*)ctx->X, ctx->d_dev_row + r0, rows, n, ctx->ld);
      ctx->check_launch();
      host.resize(size_t(rows * n));
      CK(cudaMemcpyAsync(host.data(), ctx->stage, host.size() * 8, cudaMemcpyDeviceToHost,
                         ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      const off_t off = 16 + off_t((ctx->row0 + r0) * n) * 8;
      if (!pwrite_all(f.fd, host.data(), host.size() * 8, off))
        return fail(ctx, OTDR_E_INVALID_ARG, std::string(path) + ": write failed");
    }
    return OTDR_OK;
  });
}

otdr_status otdr_dev_set_regularizer(otdr_dev* ctx, otdr_reg_kind kind, double param,
                                     const int32_t* row_labels) {
  if (!ctx) return OTDR_E_INVALID_ARG;
  if (kind == OTDR_REG_QUAD && !(param > 0.0 && std::isfinite(param)))
    return fail(ctx, OTDR_E_INVALID_ARG, "quadratic regularizer needs alpha > 0");
  if (kind == OTDR_REG_GROUP_LASSO && !(param > 0.0 && std::isfinite(param)))
    return fail(ctx, OTDR_E_INVALID_ARG, "group lasso needs lambda > 0");
  if (kind != OTDR_REG_NONE && kind != OTDR_REG_QUAD && kind != OTDR_REG_GROUP_LASSO)
    return fail(ctx, OTDR_E_UNSUPPORTED, "unsupported regularizer kind");
  if (kind == OTDR_REG_GROUP_LASSO && !row_labels && ctx->m_loc > 0)
    return fail(ctx, OTDR_E_INVALID_ARG, "group lasso needs row labels");
  return guarded(ctx, [&] {
    std::vector<long long> order(size_t(ctx->m_loc));
    std::iota(order.begin(), order.end(), 0LL);
    if (kind == OTDR_REG_GROUP_LASSO) {
      ctx->labels.assign(row_labels, row_labels + ctx->m_loc);
      for (int32_t l : ctx->labels)
        if (l < -1) return fail(ctx, OTDR_E_INVALID_ARG, "row labels must be >= -1");
      // Stable class sort: grouped classes ascending, ungrouped (-1) rows last.
      auto key = [&](long long h) {
        const int32_t l = ctx->labels[size_t(h)];
        return l < 0 ? std::numeric_limits<int64_t>::max() : int64_t(l);
      };
      std::stable_sort(order.begin(), order.end(),
                       [&](long long x, long long y) { return key(x) < key(y); });
    } else {
      ctx->labels.clear();
    }
    std::vector<long long> new_row(size_t(ctx->m_loc));
    for (long long d = 0; d < ctx->m_loc; ++d) new_row[size_t(order[size_t(d)])] = d;
    ctx->reg_kind = kind;
    ctx->reg_param = param;
    ctx->permute_rows(new_row);
    ctx->build_segments();
    ctx->invalidate_graphs();
    ctx->set_rho_params(ctx->prm.rho);
    ctx->push_prm();
    return OTDR_OK;
  });
}

otdr_status otdr_dev_set_state(otdr_dev* ctx, const double* X0, const double* phi0,
                               const double* psi0) {
  if (!ctx) return OTDR_E_INVALID_ARG;
  if (!ctx->has_problem) return fail(ctx, OTDR_E_STATE, "set_state before set_problem");
  const bool warm = X0 || phi0 || psi0;
  if (warm && !(X0 && phi0 && psi0))
    return fail(ctx, OTDR_E_DIMENSION, "warm start dimensions do not match the problem");
  return guarded(ctx, [&] {
    if (warm) {
      const size_t cnt = size_t(ctx->m_loc) * size_t(ctx->n);
      for (size_t t = 0; t < cnt; ++t)
        if (!std::isfinite(X0[t]) || X0[t] < 0.0)
          return fail(ctx, OTDR_E_NEGATIVE, "warm-start plan must be finite and >= 0");
      if (ctx->f64()) ctx->upload_rows<double>((double*)ctx->X, X0);
      else ctx->upload_rows<float>((float*)ctx->X, X0);
      ctx->upload_vec_rows(ctx->phi, phi0);
      CK(cudaMemcpy(ctx->psi, psi0, size_t(ctx->n) * 8, cudaMemcpyHostToDevice));
    } else {  // default_init (solver.cpp:59-66)
      CK(cudaMemset(ctx->X, 0, size_t(std::max<long long>(ctx->m_loc, 1)) * ctx->ld * ctx->esz));
      const double mn = double(ctx->m_glob + ctx->n);
      const double ph = (1.0 + double(ctx->m_glob) / mn) / (3.0 * mn);
      const double ps = (1.0 + double(ctx->n) / mn) / (3.0 * mn);
      std::vector<double> vphi(size_t(std::max<long long>(ctx->m_loc, 1)), ph);
      std::vector<double> vpsi(size_t(ctx->n), ps);
      CK(cudaMemcpy(ctx->phi, vphi.data(), size_t(ctx->m_loc) * 8, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(ctx->psi, vpsi.data(), size_t(ctx->n) * 8, cudaMemcpyHostToDevice));
    }
    ctx->seed_state();
    return OTDR_OK;
  });
}

otdr_status otdr_dev_load_state(otdr_dev* ctx, const double* X, const double* phi,
                                const double* psi, const double* a, const double* b,
                                const double* r, const double* s, double theta, double eta,
                                int64_t k) {
  if (!ctx) return OTDR_E_INVALID_ARG;
  if (!ctx->has_problem) return fail(ctx, OTDR_E_STATE, "load_state before set_problem");
  if (!X || !phi || !psi || !a || !b || !r || !s)
    return fail(ctx, OTDR_E_INVALID_ARG, "load_state needs every state buffer");
  return guarded(ctx, [&] {
    if (ctx->f64()) ctx->upload_rows<double>((double*)ctx->X, X);
    else ctx->upload_rows<float>((float*)ctx->X, X);
    ctx->upload_vec_rows(ctx->phi, phi);
    ctx->upload_vec_rows(ctx->a, a);
    ctx->upload_vec_rows(ctx->r, r);
    CK(cudaMemcpy(ctx->psi, psi, size_t(ctx->n) * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->b, b, size_t(ctx->n) * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->s, s, size_t(ctx->n) * 8, cudaMemcpyHostToDevice));
    std::memset(ctx->h_ctl, 0, sizeof(Ctl));
    ctx->h_ctl->theta[0] = ctx->h_ctl->theta[1] = theta;
    ctx->h_ctl->eta = eta;
    ctx->h_ctl->k = k;
    ctx->push_ctl();
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->has_state = true;
    return OTDR_OK;
  });
}

otdr_status otdr_dev_step(otdr_dev* ctx, double rho, int64_t iters) {
  if (!ctx) return OTDR_E_INVALID_ARG;
  if (!ctx->has_state) return fail(ctx, OTDR_E_STATE, "step before set_state");
  if (iters < 0) return fail(ctx, OTDR_E_INVALID_ARG, "iters must be >= 0");
  return guarded(ctx, [&] {
    ctx->pull_ctl();
    ctx->h_ctl->done = 0;
    ctx->h_ctl->fused_shifted = 0;
    ctx->push_ctl();
    ctx->set_rho_params(rho);
    ctx->prm.solving = 0;
    ctx->prm.fused = 0;
    ctx->prm.record_trace = 0;
    ctx->push_prm();
    ctx->run_raw(iters);
    CK(cudaStreamSynchronize(ctx->stream));
    return OTDR_OK;
  });
}

otdr_status otdr_dev_time_steps(otdr_dev* ctx, double rho, int64_t iters, double* ms) {
  if (!ctx || !ms) return OTDR_E_INVALID_ARG;
  if (!ctx->has_state) return fail(ctx, OTDR_E_STATE, "time_steps before set_state");
  return guarded(ctx, [&] {
    ctx->pull_ctl();
    ctx->h_ctl->done = 0;
    ctx->h_ctl->fused_shifted = 0;
    ctx->push_ctl();
    ctx->set_rho_params(rho);
    ctx->prm.solving = 0;
    ctx->prm.fused = 0;
    ctx->prm.record_trace = 0;
    ctx->push_prm();
    if (iters >= 16 && !ctx->stream_active(false, false) && !ctx->resident_active(false, false) &&
        !ctx->gl_stream_active(false, false))
      ctx->get_graph(0, 16, false, false);  // instantiate outside the timing
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaEventRecord(ctx->ev0, ctx->stream));
    ctx->run_raw(iters);
    CK(cudaEventRecord(ctx->ev1, ctx->stream));
    CK(cudaEventSynchronize(ctx->ev1));
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, ctx->ev0, ctx->ev1));
    *ms = t;
    return OTDR_OK;
  });
}

otdr_status otdr_dev_profile(otdr_dev* ctx, double rho, int64_t iters, otdr_kernel_times* out) {
  if (!ctx || !out) return OTDR_E_INVALID_ARG;
  if (!ctx->has_state) return fail(ctx, OTDR_E_STATE, "profile before set_state");
  return guarded(ctx, [&] {
    ctx->pull_ctl();
    ctx->h_ctl->done = 0;
    ctx->h_ctl->fused_shifted = 0;
    ctx->push_ctl();
    ctx->set_rho_params(rho);
    ctx->prm.solving = 0;
    ctx->prm.fused = 0;
    ctx->prm.record_trace = 0;
    ctx->push_prm();
    cudaEvent_t ev[5];
    for (auto& e : ev) CK(cudaEventCreate(&e));
    double acc[4] = {0, 0, 0, 0};
    for (int64_t t = 0; t < iters; ++t) {
      CK(cudaEventRecord(ev[0], ctx->stream));
      ctx->launch_sweep(false, false);
      CK(cudaEventRecord(ev[1], ctx->stream));
      ctx->launch_reduce(false, false);
      CK(cudaEventRecord(ev[2], ctx->stream));
      ctx->launch_exchange(ctx->exch, size_t(ctx->n) + 3);
      CK(cudaEventRecord(ev[3], ctx->stream));
      ctx->launch_update(0, 0, 0);
      CK(cudaEventRecord(ev[4], ctx->stream));
      ctx->check_launch();
      CK(cudaEventSynchronize(ev[4]));
      for (int k = 0; k < 4; ++k) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ev[k], ev[k + 1]));
        acc[k] += ms;
      }
    }
    for (auto& e : ev) cudaEventDestroy(e);
    const double it = double(std::max<int64_t>(iters, 1));
    out->sweep_ms = acc[0] / it;
    out->reduce_ms = acc[1] / it;
    out->exchange_ms = acc[2] / it;
    out->update_ms = acc[3] / it;
    out->iterations = iters;
    out->sweep_bytes = double(ctx->m_loc) * double(ctx->n) * 3.0 * double(ctx->esz);
    return OTDR_OK;
  });
}

otdr_status otdr_dev_solve(otdr_dev* ctx, const otdr_solve_opts* o, otdr_solve_result* res) {
  if (!ctx || !o || !res) return OTDR_E_INVALID_ARG;
  if (o->max_iter <= 0)
    return fail(ctx, OTDR_E_ZERO_ITERS,
                "max_iter must be positive, got " + std::to_string((long long)o->max_iter));
  if (o->check_every <= 0) return fail(ctx, OTDR_E_INVALID_ARG, "check_every must be positive");
  if (!(o->tol_primal > 0.0)) return fail(ctx, OTDR_E_INVALID_ARG, "tol_primal must be positive");
  if (o->has_tol_gap && !(o->tol_gap > 0.0))
    return fail(ctx, OTDR_E_INVALID_ARG, "tol_gap must be positive when set");
  if (!ctx->has_state) return fail(ctx, OTDR_E_STATE, "solve before set_state");
  return guarded(ctx, [&] {
    const double rho = o->rho > 0.0 ? o->rho : 2.0 / double(ctx->m_glob + ctx->n);
    const bool track = o->record_trace != 0;
    const bool cert = o->has_tol_gap || o->record_trace;
    ctx->set_rho_params(rho);
    ctx->prm.tol_primal = o->tol_primal;
    ctx->prm.tol_gap = o->has_tol_gap ? o->tol_gap : 0.0;
    ctx->prm.has_tol_gap = o->has_tol_gap ? 1 : 0;
    ctx->prm.max_iter = o->max_iter;
    ctx->prm.check_every = o->check_every;
    ctx->prm.record_trace = track ? 1 : 0;
    ctx->prm.deterministic = o->deterministic ? 1 : 0;
    // fused even/odd (solver.cpp:127-177) is pinned entry-wise equal to the
    // unfused loop (test_solver.cpp:342-357). With fp32 storage the even step's
    // B = X - rho C is an O(rho) quantity whose fp32 rounding grows with the
    // plan size, and the unfused sweep is also the faster one
    // once X is compressible -- so fp32 storage runs `fused` on the unfused
    // kernels; fp64 storage keeps the in-place even/odd buffer.
    ctx->prm.fused = (o->fused && ctx->f64()) ? 1 : 0;
    ctx->prm.solving = 1;
    if (track) {
      const long long cap = o->max_iter / o->check_every + 2;
      if (cap > ctx->trace_cap) {
        if (ctx->d_trace) cudaFree(ctx->d_trace);
        ctx->d_trace = dalloc<otdrk::TraceRow>(size_t(cap));
        ctx->trace_cap = cap;
        ctx->invalidate_graphs();
      }
    }
    ctx->prm.trace_cap = ctx->trace_cap;
    ctx->push_prm();
    ctx->pull_ctl();
    Ctl& c = *ctx->h_ctl;
    c.k0 = c.k;
    c.done = 0;
    c.termination = otdrk::TERM_MAXITER;
    c.want_cert = 0;
    c.fused_shifted = 0;
    c.best = std::numeric_limits<double>::infinity();
    c.last_improvement = 0;
    c.supp_changed = 0;
    c.supp_count = 0;
    c.support_last_change = 0;
    c.trace_len = 0;
    c.cnt_reduce = c.cnt_update = c.cnt_cert = 0;
    ctx->push_ctl();
    // The support mask of X_0 (solver.cpp:133-143) is implicit: the tracking
    // sweep compares each entry's old and new sign.
    CK(cudaStreamSynchronize(ctx->stream));
    const bool resident = ctx->resident_active(track, cert);
    // tol_gap without a trace runs on the persistent kernels: a launch stops at
    // a check iteration with r_primal <= tol and the certificate kernels decide
    const bool gap_only = o->has_tol_gap && !track && !ctx->prm.fused;
    const bool pcert = cert && !gap_only;
    const bool gl_streaming = !resident && ctx->gl_stream_active(track, pcert);
    const bool streaming = !resident && (ctx->stream_active(track, pcert) || gl_streaming);
    const bool use_while = ctx->comm == nullptr;
    const int body = 4;
    cudaGraphExec_t ex = nullptr;
    if (!resident && !streaming)
      ex = use_while ? ctx->get_graph(1, body, track, cert) : ctx->get_graph(0, 8, track, cert);
    CK(cudaEventRecord(ctx->ev0, ctx->stream));
    otdrk::stamp_t0_kernel<<<1, 1, 0, ctx->stream>>>(ctx->d_ctl);
    if (resident) {
      ctx->launch_resident(0);
      ctx->check_launch();
    } else if (streaming) {
      for (;;) {
        if (gl_streaming) ctx->launch_gl_stream(0);
        else ctx->launch_stream(0);
        ctx->check_launch();
        if (!gap_only) break;
        ctx->pull_ctl();
        if (ctx->h_ctl->done || !ctx->h_ctl->want_cert) break;
        ctx->launch_cert(0, 0, 0);  // certificate + the reference's stopping decision
        ctx->check_launch();
        ctx->pull_ctl();
        if (ctx->h_ctl->done) break;
      }
    } else if (use_while) {
      CK(cudaGraphLaunch(ex, ctx->stream));
    } else {
      for (;;) {
        CK(cudaGraphLaunch(ex, ctx->stream));
        ctx->pull_ctl();
        if (ctx->h_ctl->done) break;
      }
    }
    CK(cudaEventRecord(ctx->ev1, ctx->stream));
    CK(cudaEventSynchronize(ctx->ev1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    ctx->pull_ctl();
    if (ctx->h_ctl->termination == otdrk::TERM_NONFINITE) {
      const long long kk = ctx->h_ctl->k - ctx->h_ctl->k0;
      return fail(ctx, OTDR_E_NONFINITE,
                  "non-finite iterate at iteration " + std::to_string(kk) +
                      " (check rho and regularizer parameters)");
    }
    // Materialise X after an even fused iteration, then the objective.
    if (ctx->prm.fused && ctx->h_ctl->fused_shifted) {
      const long long cnt = ctx->m_loc * ctx->ld;
      if (ctx->f64())
        otdrk::unshift_kernel<double><<<4 * kNumSMs, 256, 0, ctx->stream>>>((double*)ctx->X, (const double*)ctx->C, ctx->d_prm, cnt);
      else
        otdrk::unshift_kernel<float><<<4 * kNumSMs, 256, 0, ctx->stream>>>((float*)ctx->X, (const float*)ctx->C, ctx->d_prm, cnt);
      ctx->check_launch();
      ctx->h_ctl->fused_shifted = 0;
      ctx->push_ctl();
    }
    if (!resident) {  // the resident kernel already evaluated the objective on chip
      ctx->launch_cert(1, 0, 0);
      ctx->check_launch();
    }
    ctx->pull_ctl();
    res->iterations = ctx->h_ctl->k;
    res->termination = ctx->h_ctl->termination;
    res->rho = rho;
    res->r_primal = ctx->h_ctl->r_primal;
    res->objective = ctx->h_ctl->objective;
    res->support_last_change = track ? ctx->h_ctl->support_last_change : -1;
    res->trace_rows = track ? ctx->h_ctl->trace_len : 0;
    res->device_ms = ms;
    ctx->prm.solving = 0;
    ctx->prm.fused = 0;
    ctx->push_prm();
    return OTDR_OK;
  });
}

otdr_status otdr_dev_get_state(otdr_dev* ctx, double* X, double* phi, double* psi, double* a,
                               double* b, double* r, double* s, double* theta, double* eta,
                               int64_t* k) {
  if (!ctx) return OTDR_E_INVALID_ARG;
  if (!ctx->has_state) return fail(ctx, OTDR_E_STATE, "get_state before set_state");
  return guarded(ctx, [&] {
    CK(cudaStreamSynchronize(ctx->stream));
    if (X) {
      if (ctx->f64()) ctx->download_rows<double>(X, (const double*)ctx->X);
      else ctx->download_rows<float>(X, (const float*)ctx->X);
    }
    if (phi) ctx->download_vec_rows(phi, ctx->phi);
    if (a) ctx->download_vec_rows(a, ctx->a);
    if (r) ctx->download_vec_rows(r, ctx->r);
    if (psi) CK(cudaMemcpy(psi, ctx->psi, size_t(ctx->n) * 8, cudaMemcpyDeviceToHost));
    if (b) CK(cudaMemcpy(b, ctx->b, size_t(ctx->n) * 8, cudaMemcpyDeviceToHost));
    if (s) CK(cudaMemcpy(s, ctx->s, size_t(ctx->n) * 8, cudaMemcpyDeviceToHost));
    ctx->pull_ctl();
    if (theta) *theta = ctx->h_ctl->theta[ctx->h_ctl->k & 1];
    if (eta) *eta = ctx->h_ctl->eta;
    if (k) *k = ctx->h_ctl->k;
    return OTDR_OK;
  });
}

otdr_status otdr_dev_objective(otdr_dev* ctx, double* out) {
  if (!ctx || !out) return OTDR_E_INVALID_ARG;
  if (!ctx->has_state) return fail(ctx, OTDR_E_STATE, "objective before set_state");
  return guarded(ctx, [&] {
    ctx->launch_cert(1, 0, 0);
    ctx->check_launch();
    ctx->pull_ctl();
    *out = ctx->h_ctl->objective;
    return OTDR_OK;
  });
}

otdr_status otdr_dev_duality_gap(otdr_dev* ctx, double rho, otdr_certificate* out) {
  if (!ctx || !out) return OTDR_E_INVALID_ARG;
  if (!ctx->has_state) return fail(ctx, OTDR_E_STATE, "duality_gap before set_state");
  return guarded(ctx, [&] {
    ctx->set_rho_params(rho);
    ctx->prm.solving = 0;
    ctx->prm.fused = 0;
    ctx->prm.record_trace = 0;
    ctx->prm.has_tol_gap = 0;
    ctx->prm.check_every = 1;
    ctx->prm.max_iter = std::numeric_limits<long long>::max();
    ctx->push_prm();
    ctx->pull_ctl();
    ctx->h_ctl->want_cert = 1;
    ctx->h_ctl->done = 0;
    ctx->push_ctl();
    ctx->launch_cert(0, 0, 0);
    ctx->check_launch();
    ctx->pull_ctl();
    out->dual_value = ctx->h_ctl->dual_value;
    out->gap = ctx->h_ctl->gap;
    out->dual_residual = ctx->h_ctl->dres;
    ctx->h_ctl->done = 0;
    ctx->h_ctl->want_cert = 0;
    ctx->push_ctl();
    CK(cudaStreamSynchronize(ctx->stream));
    return OTDR_OK;
  });
}

otdr_status otdr_dev_get_trace(otdr_dev* ctx, otdr_trace_row* rows, int64_t cap, int64_t* count) {
  if (!ctx) return OTDR_E_INVALID_ARG;
  return guarded(ctx, [&] {
    ctx->pull_ctl();
    const long long have = std::min<long long>(ctx->h_ctl->trace_len, ctx->trace_cap);
    if (count) *count = have;
    const long long take = std::min<long long>(have, cap);
    if (take > 0 && rows) {
      static_assert(sizeof(otdrk::TraceRow) == sizeof(otdr_trace_row), "trace row layout");
      CK(cudaMemcpy(rows, ctx->d_trace, size_t(take) * sizeof(otdr_trace_row),
                    cudaMemcpyDeviceToHost));
    }
    return OTDR_OK;
  });
}

}  // extern "C"

#include "otdr_batch.cuh"
