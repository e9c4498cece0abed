// otdr_batch.cuh -- batched entry point (include/otdr_dev.h, otdr_batch_*);
// compiled as part of otdr_dev.cu's translation unit.
//
// B problems of one shape; problem b is owned by thread-block cluster b, whose
// G CTAs keep the problem's C and X resident in shared memory for the whole
// solve and exchange column sums / psi through distributed shared memory
// (resident_kernel<T, true>, otdr_resident.cuh). One launch solves the batch;
// the hardware schedules clusters as SMs free up, so problems that converge
// early release their SMs to the remaining ones.
#pragma once
namespace {

struct BErr {
  otdr_status code;
  std::string msg;
};

#define BCK(expr)                                                                    \
  do {                                                                               \
    cudaError_t e_ = (expr);                                                         \
    if (e_ != cudaSuccess)                                                           \
      throw BErr{OTDR_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)};   \
  } while (0)

template <typename T>
T* balloc(size_t count) {
  void* p = nullptr;
  BCK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
  return static_cast<T*>(p);
}

}  // namespace

struct otdr_batch {
  int device = 0;
  int storage = OTDR_STORE_F32;
  size_t esz = 4;
  long long B = 0, m = 0, n = 0, ld = 0;
  int G = 0, R = 0;
  size_t smem = 0;
  // streaming mode: one CTA per problem, C / X streamed from HBM every iteration
  bool use_stream = false;
  int bs_nch = 0, bs_nsets = 0;
  size_t bs_smem = 0;
  static constexpr int kBSD = 6;
  int bs_nt = 256;  // threads per problem CTA (OTDR_BATCH_THREADS=512: one CTA per SM)
  int bs_cs = 2;    // CTAs per problem (OTDR_BATCH_CLUSTER=1: one CTA per problem)
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::string err;
  void* C = nullptr;
  void* X = nullptr;
  size_t x_vmm = 0;  // mapped size when X is a compressible VMM allocation
  bool x_comp = false;
  double *p = nullptr, *q = nullptr, *phi = nullptr, *psi = nullptr, *a = nullptr, *b = nullptr,
         *r = nullptr, *s = nullptr;
  otdrk::Ctl* ctl = nullptr;
  otdrk::Params* prm = nullptr;
  std::vector<double> hp, hq;
  int reg = OTDR_REG_NONE;
  double alpha = 0.0;
  bool has_problems = false;

  bool f64() const { return storage == OTDR_STORE_F64; }

  void release() {
    if (x_vmm) {
      comp_free(X, x_vmm);
      X = nullptr;
    }
    void* ptrs[] = {C, X, p, q, phi, psi, a, b, r, s, ctl, prm};
    for (void* ptr : ptrs)
      if (ptr) cudaFree(ptr);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (stream) cudaStreamDestroy(stream);
  }

  template <typename T>
  void upload_costs(const double* costs) {
    // row-major problems -> padded rows of width ld (pad columns are 0)
    std::vector<T> buf(size_t(B * m * ld), T(0));
    for (long long t = 0; t < B * m; ++t)
      for (long long j = 0; j < n; ++j) buf[size_t(t * ld + j)] = T(costs[t * n + j]);
    BCK(cudaMemcpy(C, buf.data(), buf.size() * sizeof(T), cudaMemcpyHostToDevice));
  }

  template <typename T, int NT, int CS>
  void launch_stream_nt() {
    auto kern = otdrk::bstream_kernel<T, sizeof(T) == 8, kBSD, NT, CS>;
    BCK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bs_smem)));
    otdrk::BStreamArgs ba{X, C, m * ld, phi, a, r, p, psi, b, s, q, ctl, prm, m, n, ld,
                          bs_nch, bs_nsets, reg == OTDR_REG_QUAD ? otdrk::REG_QUAD : otdrk::REG_NONE};
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(unsigned(B * CS), 1, 1);
    lc.blockDim = dim3(NT, 1, 1);
    lc.dynamicSmemBytes = bs_smem;
    lc.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(CS);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    BCK(cudaLaunchKernelEx(&lc, kern, ba));
    BCK(cudaGetLastError());
  }
  template <typename T>
  void launch_stream() {
    if (bs_cs == 4) {
      if (bs_nt == 512) launch_stream_nt<T, 512, 4>();
      else launch_stream_nt<T, 256, 4>();
    } else if (bs_cs == 2) {
      if (bs_nt == 512) launch_stream_nt<T, 512, 2>();
      else launch_stream_nt<T, 256, 2>();
    } else {
      if (bs_nt == 512) launch_stream_nt<T, 512, 1>();
      else launch_stream_nt<T, 256, 1>();
    }
  }

  template <typename T>
  void launch() {
    if (use_stream) {
      launch_stream<T>();
      return;
    }
    auto kern = otdrk::resident_kernel<T, true>;
    BCK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    if (G > 8) BCK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    otdrk::ResidentArgs ra{X, C, m * ld, phi, a, r, p, psi, b, s, q, ctl, prm, nullptr,
                           m, n, ld, R, G,
                           reg == OTDR_REG_QUAD ? otdrk::REG_QUAD : otdrk::REG_NONE, 0};
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(unsigned(B * G), 1, 1);
    lc.blockDim = dim3(otdrk::kRT, 1, 1);
    lc.dynamicSmemBytes = smem;
    lc.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(G);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    BCK(cudaLaunchKernelEx(&lc, kern, ra));
    BCK(cudaGetLastError());
  }
};

namespace {

otdr_status bfail(otdr_batch* bt, otdr_status code, const std::string& msg) {
  if (bt) bt->err = msg;
  return code;
}

template <typename F>
otdr_status bguard(otdr_batch* bt, F&& f) {
  try {
    BCK(cudaSetDevice(bt->device));
    return f();
  } catch (const BErr& e) {
    return bfail(bt, e.code, e.msg);
  } catch (const std::exception& e) {
    return bfail(bt, OTDR_E_CUDA, e.what());
  }
}

}  // namespace

extern "C" {

otdr_status otdr_batch_create(int device, otdr_storage storage, int64_t batch, int64_t m,
                              int64_t n, otdr_batch** out) {
  if (!out) return OTDR_E_INVALID_ARG;
  *out = nullptr;
  if (batch < 1 || m < 1 || n < 1) return OTDR_E_DIMENSION;
  if (!otdr_dev_cuda_available()) return OTDR_E_CUDA;
  otdr_batch* bt = new otdr_batch();
  bt->device = device;
  bt->storage = storage == OTDR_STORE_F64 ? OTDR_STORE_F64 : OTDR_STORE_F32;
  bt->esz = bt->f64() ? 8 : 4;
  bt->B = batch;
  bt->m = m;
  bt->n = n;
  const long long vec = bt->f64() ? 2 : 4;
  bt->ld = (n + vec - 1) / vec * vec;
  try {
    BCK(cudaSetDevice(device));
    int max_smem = 0;
    BCK(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    for (int G : {4, 8, 16}) {  // smallest cluster whose per-CTA tiles fit
      const long long R = (m + G - 1) / G;
      const size_t bytes = bt->f64() ? otdrk::resident_smem_bytes<double>(R, n, bt->ld)
                                     : otdrk::resident_smem_bytes<float>(R, n, bt->ld);
      if (bytes + 2048 <= size_t(max_smem)) {
        bt->G = G;
        bt->R = int(R);
        bt->smem = bytes;
        break;
      }
    }
    {  // streaming mode (default when it fits): one CTA per problem
      const long long vecw = 32 * (bt->f64() ? 2 : 4);
      const long long nch = (bt->ld + vecw - 1) / vecw;
      if (const char* bn = std::getenv("OTDR_BATCH_THREADS")) bt->bs_nt = std::atoi(bn) == 512 ? 512 : 256;
      if (const char* bc = std::getenv("OTDR_BATCH_CLUSTER")) bt->bs_cs = std::atoi(bc) == 1 ? 1 : std::atoi(bc) == 4 ? 4 : 2;
      const int nw = bt->bs_nt / 32;
      if (nch <= nw) {
        bt->bs_nch = int(nch);
        bt->bs_nsets = int(nw / nch);
        bt->bs_smem = bt->bs_nt == 512
                          ? otdrk::bstream_smem_bytes<double, otdr_batch::kBSD, 512>(m, bt->ld, bt->bs_nch, bt->bs_nsets)
                          : otdrk::bstream_smem_bytes<double, otdr_batch::kBSD, 256>(m, bt->ld, bt->bs_nch, bt->bs_nsets);
        const char* bm = std::getenv("OTDR_BATCH");
        bt->use_stream = bt->bs_smem + 1024 <= size_t(max_smem) && !(bm && std::strcmp(bm, "resident") == 0);
      }
    }
    if (bt->G == 0 && !bt->use_stream) {
      delete bt;
      return OTDR_E_UNSUPPORTED;
    }
    BCK(cudaStreamCreateWithFlags(&bt->stream, cudaStreamNonBlocking));
    BCK(cudaEventCreate(&bt->ev0));
    BCK(cudaEventCreate(&bt->ev1));
    const size_t mat = size_t(batch * m * bt->ld) * bt->esz;
    BCK(cudaMalloc(&bt->C, mat));
    {  // the batch's plans in compressible HBM, as for one engine (otdr_dev.cu)
      std::string cm = mat >= (size_t(16) << 20) ? "x" : "off";
      if (const char* e = std::getenv("OTDR_COMPRESS")) cm = e;
      double cap_gb = 3.2;
      if (const char* e = std::getenv("OTDR_COMPRESS_GB")) cap_gb = std::atof(e);
      if (cm.find('x') != std::string::npos)
        bt->X = comp_malloc(device, mat, std::min(mat, size_t(std::max(0.0, cap_gb) * 1e9)), &bt->x_vmm,
                            &bt->x_comp);
      if (!bt->X) bt->x_vmm = 0;
    }
    if (!bt->X) BCK(cudaMalloc(&bt->X, mat));
    BCK(cudaMemset(bt->C, 0, mat));
    BCK(cudaMemset(bt->X, 0, mat));
    bt->p = balloc<double>(size_t(batch * m));
    bt->phi = balloc<double>(size_t(batch * m));
    bt->a = balloc<double>(size_t(batch * m));
    bt->r = balloc<double>(size_t(batch * m));
    bt->q = balloc<double>(size_t(batch * n));
    bt->psi = balloc<double>(size_t(batch * n));
    bt->b = balloc<double>(size_t(batch * n));
    bt->s = balloc<double>(size_t(batch * n));
    bt->ctl = balloc<otdrk::Ctl>(size_t(batch));
    bt->prm = balloc<otdrk::Params>(1);
  } catch (const BErr& e) {
    bt->release();
    delete bt;
    return e.code;
  }
  *out = bt;
  return OTDR_OK;
}

void otdr_batch_destroy(otdr_batch* bt) {
  if (!bt) return;
  cudaSetDevice(bt->device);
  bt->release();
  delete bt;
}

const char* otdr_batch_last_error(const otdr_batch* bt) { return bt ? bt->err.c_str() : ""; }

otdr_status otdr_batch_set_problems(otdr_batch* bt, const double* costs, const double* p,
                                    const double* q) {
  if (!bt) return OTDR_E_INVALID_ARG;
  if (!costs || !p || !q) return bfail(bt, OTDR_E_INVALID_ARG, "null problem buffer");
  return bguard(bt, [&] {
    if (bt->f64()) bt->upload_costs<double>(costs);
    else bt->upload_costs<float>(costs);
    bt->hp.assign(p, p + bt->B * bt->m);
    bt->hq.assign(q, q + bt->B * bt->n);
    BCK(cudaMemcpy(bt->p, p, size_t(bt->B * bt->m) * 8, cudaMemcpyHostToDevice));
    BCK(cudaMemcpy(bt->q, q, size_t(bt->B * bt->n) * 8, cudaMemcpyHostToDevice));
    bt->has_problems = true;
    return OTDR_OK;
  });
}

otdr_status otdr_batch_build_sqdist_costs(otdr_batch* bt, const double* src, const double* tgt,
                                          int d, const double* p, const double* q) {
  if (!bt) return OTDR_E_INVALID_ARG;
  if (!src || !tgt || !p || !q || d < 1)
    return bfail(bt, OTDR_E_INVALID_ARG, "bad point cloud arguments");
  return bguard(bt, [&] {
    const long long B = bt->B, m = bt->m, n = bt->n;
    double* d_src = balloc<double>(size_t(B * m * d));
    double* d_tgt = balloc<double>(size_t(B * n * d));
    double* d_mx = balloc<double>(size_t(B));
    unsigned long long* d_bits = balloc<unsigned long long>(size_t(B));
    BCK(cudaMemcpy(d_src, src, size_t(B * m * d) * 8, cudaMemcpyHostToDevice));
    BCK(cudaMemcpy(d_tgt, tgt, size_t(B * n * d) * 8, cudaMemcpyHostToDevice));
    BCK(cudaMemset(d_bits, 0, size_t(B) * 8));
    for (long long pb = 0; pb < B; ++pb) {
      const double* s = d_src + pb * m * d;
      const double* t = d_tgt + pb * n * d;
      unsigned long long* bits = d_bits + pb;
      double* mx = d_mx + pb;
      if (bt->f64()) {
        double* Cb = static_cast<double*>(bt->C) + pb * m * bt->ld;
        otdrk::sqdist_kernel<double><<<64, 256, 0, bt->stream>>>(Cb, s, t, d, m, n, bt->ld, mx, bits, 0);
        BCK(cudaMemcpyAsync(mx, bits, 8, cudaMemcpyDeviceToDevice, bt->stream));
        otdrk::sqdist_kernel<double><<<64, 256, 0, bt->stream>>>(Cb, s, t, d, m, n, bt->ld, mx, bits, 1);
      } else {
        float* Cb = static_cast<float*>(bt->C) + pb * m * bt->ld;
        otdrk::sqdist_kernel<float><<<64, 256, 0, bt->stream>>>(Cb, s, t, d, m, n, bt->ld, mx, bits, 0);
        BCK(cudaMemcpyAsync(mx, bits, 8, cudaMemcpyDeviceToDevice, bt->stream));
        otdrk::sqdist_kernel<float><<<64, 256, 0, bt->stream>>>(Cb, s, t, d, m, n, bt->ld, mx, bits, 1);
      }
    }
    BCK(cudaGetLastError());
    BCK(cudaStreamSynchronize(bt->stream));
    cudaFree(d_src);
    cudaFree(d_tgt);
    cudaFree(d_mx);
    cudaFree(d_bits);
    bt->hp.assign(p, p + B * m);
    bt->hq.assign(q, q + B * n);
    BCK(cudaMemcpy(bt->p, p, size_t(B * m) * 8, cudaMemcpyHostToDevice));
    BCK(cudaMemcpy(bt->q, q, size_t(B * n) * 8, cudaMemcpyHostToDevice));
    bt->has_problems = true;
    return OTDR_OK;
  });
}

otdr_status otdr_batch_set_regularizer(otdr_batch* bt, otdr_reg_kind kind, double alpha) {
  if (!bt) return OTDR_E_INVALID_ARG;
  if (kind == OTDR_REG_GROUP_LASSO)
    return bfail(bt, OTDR_E_UNSUPPORTED, "batched entry point covers zero / quadratic");
  if (kind == OTDR_REG_QUAD && !(alpha > 0.0 && std::isfinite(alpha)))
    return bfail(bt, OTDR_E_INVALID_ARG, "quadratic regularizer needs alpha > 0");
  bt->reg = kind;
  bt->alpha = kind == OTDR_REG_QUAD ? alpha : 0.0;
  return OTDR_OK;
}

otdr_status otdr_batch_solve(otdr_batch* bt, const otdr_solve_opts* o, otdr_solve_result* res) {
  if (!bt || !o || !res) return OTDR_E_INVALID_ARG;
  if (o->max_iter <= 0)
    return bfail(bt, OTDR_E_ZERO_ITERS,
                 "max_iter must be positive, got " + std::to_string((long long)o->max_iter));
  if (o->check_every <= 0) return bfail(bt, OTDR_E_INVALID_ARG, "check_every must be positive");
  if (!(o->tol_primal > 0.0)) return bfail(bt, OTDR_E_INVALID_ARG, "tol_primal must be positive");
  if (o->has_tol_gap || o->record_trace || o->fused)
    return bfail(bt, OTDR_E_UNSUPPORTED, "batched solve: tol_gap / trace / fused not supported");
  if (!bt->has_problems) return bfail(bt, OTDR_E_STATE, "solve before set_problems");
  return bguard(bt, [&] {
    const long long B = bt->B, m = bt->m, n = bt->n;
    const double rho = o->rho > 0.0 ? o->rho : 2.0 / double(m + n);
    otdrk::Params prm{};
    prm.rho = rho;
    prm.alpha = bt->alpha;
    prm.quad_d = 1.0 + rho * bt->alpha;
    prm.quad_inv = 1.0 / prm.quad_d;
    prm.tol_primal = o->tol_primal;
    prm.max_iter = o->max_iter;
    prm.check_every = o->check_every;
    prm.solving = 1;
    BCK(cudaMemcpy(bt->prm, &prm, sizeof(prm), cudaMemcpyHostToDevice));
    // make_state from default_init per problem (solver.cpp:59-93) with X0 = 0:
    // r = -p, s = -q, a = n phi0 + r, b = m psi0 + s, theta = -1/(m+n).
    const double mn = double(m + n);
    const double ph = (1.0 + double(m) / mn) / (3.0 * mn);
    const double ps = (1.0 + double(n) / mn) / (3.0 * mn);
    std::vector<double> vphi(size_t(B * m), ph), vpsi(size_t(B * n), ps), vr(size_t(B * m)),
        vs(size_t(B * n)), va(size_t(B * m)), vb(size_t(B * n));
    for (long long t = 0; t < B * m; ++t) {
      vr[size_t(t)] = 0.0 - bt->hp[size_t(t)];
      va[size_t(t)] = double(n) * ph + vr[size_t(t)];
    }
    for (long long t = 0; t < B * n; ++t) {
      vs[size_t(t)] = 0.0 - bt->hq[size_t(t)];
      vb[size_t(t)] = double(m) * ps + vs[size_t(t)];
    }
    BCK(cudaMemcpy(bt->phi, vphi.data(), vphi.size() * 8, cudaMemcpyHostToDevice));
    BCK(cudaMemcpy(bt->psi, vpsi.data(), vpsi.size() * 8, cudaMemcpyHostToDevice));
    BCK(cudaMemcpy(bt->r, vr.data(), vr.size() * 8, cudaMemcpyHostToDevice));
    BCK(cudaMemcpy(bt->s, vs.data(), vs.size() * 8, cudaMemcpyHostToDevice));
    BCK(cudaMemcpy(bt->a, va.data(), va.size() * 8, cudaMemcpyHostToDevice));
    BCK(cudaMemcpy(bt->b, vb.data(), vb.size() * 8, cudaMemcpyHostToDevice));
    BCK(cudaMemset(bt->X, 0, size_t(B * m * bt->ld) * bt->esz));
    std::vector<otdrk::Ctl> ctl(static_cast<size_t>(B));
    for (auto& c : ctl) {
      std::memset(&c, 0, sizeof(c));
      c.theta[0] = c.theta[1] = (0.0 - 1.0) / mn;
      c.best = std::numeric_limits<double>::infinity();
      c.termination = otdrk::TERM_MAXITER;
    }
    BCK(cudaMemcpy(bt->ctl, ctl.data(), ctl.size() * sizeof(otdrk::Ctl), cudaMemcpyHostToDevice));
    BCK(cudaEventRecord(bt->ev0, bt->stream));
    if (bt->f64()) bt->launch<double>();
    else bt->launch<float>();
    BCK(cudaEventRecord(bt->ev1, bt->stream));
    BCK(cudaEventSynchronize(bt->ev1));
    float ms = 0.f;
    BCK(cudaEventElapsedTime(&ms, bt->ev0, bt->ev1));
    BCK(cudaMemcpy(ctl.data(), bt->ctl, ctl.size() * sizeof(otdrk::Ctl), cudaMemcpyDeviceToHost));
    long long nonfinite = -1;
    for (long long pb = 0; pb < B; ++pb) {
      const otdrk::Ctl& c = ctl[size_t(pb)];
      otdr_solve_result& rr = res[pb];
      rr.iterations = c.k;
      rr.termination = c.termination == otdrk::TERM_NONFINITE ? OTDR_TERM_MAXITER : c.termination;
      rr.rho = rho;
      rr.r_primal = c.r_primal;
      rr.objective = c.objective;
      rr.support_last_change = -1;
      rr.trace_rows = 0;
      rr.device_ms = ms;
      if (c.termination == otdrk::TERM_NONFINITE && nonfinite < 0) nonfinite = pb;
    }
    if (nonfinite >= 0)
      return bfail(bt, OTDR_E_NONFINITE,
                   "non-finite iterate at iteration " + std::to_string(ctl[size_t(nonfinite)].k) +
                       " (check rho and regularizer parameters) in problem " +
                       std::to_string(nonfinite));
    return OTDR_OK;
  });
}

otdr_status otdr_batch_get_plans(otdr_batch* bt, double* X, double* phi, double* psi) {
  if (!bt) return OTDR_E_INVALID_ARG;
  return bguard(bt, [&] {
    const long long B = bt->B, m = bt->m, n = bt->n, ld = bt->ld;
    if (X) {
      if (bt->f64()) {
        std::vector<double> buf(size_t(B * m * ld));
        BCK(cudaMemcpy(buf.data(), bt->X, buf.size() * 8, cudaMemcpyDeviceToHost));
        for (long long t = 0; t < B * m; ++t)
          std::memcpy(X + t * n, buf.data() + t * ld, size_t(n) * 8);
      } else {
        std::vector<float> buf(size_t(B * m * ld));
        BCK(cudaMemcpy(buf.data(), bt->X, buf.size() * 4, cudaMemcpyDeviceToHost));
        for (long long t = 0; t < B * m; ++t)
          for (long long j = 0; j < n; ++j) X[t * n + j] = double(buf[size_t(t * ld + j)]);
      }
    }
    if (phi) BCK(cudaMemcpy(phi, bt->phi, size_t(B * m) * 8, cudaMemcpyDeviceToHost));
    if (psi) BCK(cudaMemcpy(psi, bt->psi, size_t(B * n) * 8, cudaMemcpyDeviceToHost));
    return OTDR_OK;
  });
}

otdr_status otdr_batch_get_state(otdr_batch* bt, double* X, double* phi, double* psi, double* a,
                                 double* b, double* r, double* s, double* theta, double* eta,
                                 int64_t* k) {
  if (!bt) return OTDR_E_INVALID_ARG;
  const otdr_status st = otdr_batch_get_plans(bt, X, phi, psi);
  if (st != OTDR_OK) return st;
  return bguard(bt, [&] {
    const long long B = bt->B, m = bt->m, n = bt->n;
    // both batched kernels leave a, r (rows) and b, s (columns) in global memory
    if (a) BCK(cudaMemcpy(a, bt->a, size_t(B * m) * 8, cudaMemcpyDeviceToHost));
    if (r) BCK(cudaMemcpy(r, bt->r, size_t(B * m) * 8, cudaMemcpyDeviceToHost));
    if (b) BCK(cudaMemcpy(b, bt->b, size_t(B * n) * 8, cudaMemcpyDeviceToHost));
    if (s) BCK(cudaMemcpy(s, bt->s, size_t(B * n) * 8, cudaMemcpyDeviceToHost));
    if (theta || eta || k) {
      std::vector<otdrk::Ctl> ctl(static_cast<size_t>(B));
      BCK(cudaMemcpy(ctl.data(), bt->ctl, ctl.size() * sizeof(otdrk::Ctl), cudaMemcpyDeviceToHost));
      for (long long pb = 0; pb < B; ++pb) {
        const otdrk::Ctl& c = ctl[size_t(pb)];
        if (theta) theta[pb] = c.theta[c.k & 1];
        if (eta) eta[pb] = c.eta;
        if (k) k[pb] = c.k;
      }
    }
    return OTDR_OK;
  });
}

}  // extern "C"
