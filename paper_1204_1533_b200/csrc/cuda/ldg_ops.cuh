// ldg_ops.cuh -- host-side launchers, one table of function pointers per
// compile-time configuration (D, p, physics, Riemann solver).
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>
#include <string>
#include <cstring>

#include "ldg_kernels.cuh"

namespace ldg {

// Everything a launcher needs, independent of the template configuration.
struct DevCtx {
  cudaStream_t stream = nullptr;
  // basis tables (host copies, folded): phi[np][nq], dq[np][nq], mi[np][2], cc[np][np][nq]
  const double* phi = nullptr;
  const double* dq = nullptr;
  const double* mi = nullptr;
  const double* cc = nullptr;
  PhysParams pp{};
  const int32_t* order = nullptr;
  const double* metric = nullptr;
  const int2* conn = nullptr;
  const double* bcv = nullptr;
  const int32_t* bck = nullptr;
  int noslip = 0;
  const int32_t* bface = nullptr;  // per-line-end boundary data (ldg_set_boundary_function)
  const double* bvals = nullptr;
  int pc_inverse = 0;  // block-Jacobi mode: 0 LU solves, 1 explicit block inverse
  const double* source = nullptr;
  DevError* err = nullptr;
  // face sharing of the endpoint flux Jacobians (null = every line end computes its own)
  const int2* fpart = nullptr;        // [k][2D]: partner {k', 2 dir' + side'} or {-1, 0}
  const int32_t* owned = nullptr;     // owned faces k*2D + ds, chunk by chunk
  const int32_t* inv_order = nullptr; // reference element -> processing index
  const int64_t* owned_off = nullptr; // host: chunk c owns owned[owned_off[c] .. owned_off[c+1])
  const int32_t* bspec = nullptr;     // slip-wall / Neumann boundary faces, chunk by chunk
  const int64_t* bspec_off = nullptr; // host offsets into bspec
  int E = 0;
  int spmv_order = 0;  // LDG_OPT_SPMV_ROW_ORDER: 0 auto, 1 forward, 2 reverse
  long long* launches = nullptr;
};

struct Ops {
  int D, P, PH, RI, M, NP, NQ, NPE, NL, MD, NS11, NS12, B11, B12, R12, NT, TPE, METP, MET_NV, MET_NE;
  size_t jac_smem;
  size_t endjac_per_elem;  // doubles of endpoint-Jacobian scratch per element
  size_t (*scratch_elems)(int E);  // doubles of scratch for E elements (chunked)
  int (*chunk_elems)(int E);       // elements per Jacobian assembly chunk
  cudaError_t (*residual)(const DevCtx&, const double* U, const double* Q, double* R);
  cudaError_t (*gradient)(const DevCtx&, const double* U, double* Q);
  cudaError_t (*jacobian)(const DevCtx&, const double* U, const double* Q, double* SE, double* K11,
                          double* K12);
  cudaError_t (*k21)(const DevCtx&, double* K21);
  cudaError_t (*spmv11)(const DevCtx&, const double* V11, const double* x, double* y);
  cudaError_t (*spmv11_zc)(const DevCtx&, const double* V11, const double* x, double* y);  // y mapped host
  cudaError_t (*spmv12)(const DevCtx&, const double* V12, const double* w, double* y);
  cudaError_t (*spmv21)(const DevCtx&, const double* V21, const double* v, double* w);
  cudaError_t (*split)(const DevCtx&, const double* V11, const double* V12, const double* v,
                       const double* w, double adt, double* y);
  int pc_ne;  // unknowns per element of the block-Jacobi blocks (0: not supported)
  cudaError_t (*pc_build)(const DevCtx&, const double* V11, const double* V12, const double* V21, double adt,
                          double* LUc, int32_t* piv, int* bad);
  cudaError_t (*pc_apply)(const DevCtx&, const double* LUc, const int32_t* piv, const double* r, double* z);
  int pc_line_nb;  // line-ADI block size (p+1) m (0: not supported)
  cudaError_t (*pc_line_build)(const DevCtx&, const double* V11, const double* V12, const double* V21, double adt,
                               double* LUc, int32_t* piv, int* bad);
  cudaError_t (*pc_line_apply)(const DevCtx&, const double* LUc, const int32_t* piv, const double* r, double* z);
};

// Persistent-grid size of a kernel on the CURRENT device (the context's
// device: every C-ABI entry point makes it current): sets the dynamic
// shared-memory attribute and measures occupancy once per (kernel, device);
// thread-safe (launches from several host threads / contexts).
inline int persistent_grid(const void* kernel, int threads, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> cache;
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find({kernel, dev});
    if (it != cache.end()) return it->second;
  }
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  int per_sm = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (per_sm > 0 ? per_sm : 1) * sms;
  std::lock_guard<std::mutex> g(mu);
  cache[{kernel, dev}] = grid;
  return grid;
}

template <class C>
struct Launch {
  // line threads per residual CTA (EPB = elements per batch); measured: 64
  // for 2-D (C2 residual 35.9 -> 34.5 us: smaller batches, more CTAs per SM),
  // 128 for 3-D (C4: 64 is 1.6 % slower)
  static constexpr int RES_LINES = C::D == 2 ? 64 : 128;
  static constexpr int EPB = RES_LINES / C::LPE > 0 ? RES_LINES / C::LPE : 1;
  static constexpr int RTHREADS = (EPB * C::LPE + 31) / 32 * 32;

  static KParams<C> params(const DevCtx& d) {
    KParams<C> kp;
    std::memcpy(kp.bt.phi, d.phi, sizeof(kp.bt.phi));
    std::memcpy(kp.bt.dq, d.dq, sizeof(kp.bt.dq));
    std::memcpy(kp.bt.mi, d.mi, sizeof(kp.bt.mi));
    std::memcpy(kp.bt.cc, d.cc, sizeof(kp.bt.cc));
    kp.pp = d.pp;
    kp.order = d.order;
    kp.metric = d.metric;
    kp.conn = d.conn;
    kp.bcv = d.bcv;
    kp.bck = d.bck;
    kp.noslip = d.noslip;
    kp.bface = d.bface;
    kp.bvals = d.bvals;
    kp.source = d.source;
    kp.err = d.err;
    kp.fpart = d.fpart;
    kp.owned = d.owned;
    kp.inv_order = d.inv_order;
    kp.E = d.E;
    return kp;
  }
  static void count(const DevCtx& d) {
    if (d.launches) ++*d.launches;
  }

  // Residual.  Kernel choice (measured on B200, bench.py --config N): the
  // flattened flux-parallel kernel k_residual_f wins where the per-line work
  // is long (second-order physics: viscous fluxes and the gradient at every
  // point); the thread-per-line kernel k_residual_p wins for Euler.
  static cudaError_t residual(const DevCtx& d, const double* U, const double* Q, double* R) {
    if (C::SECOND) return residual_f(d, U, Q, R);
    using RP = ResP<C, EPB>;
    const size_t smem = sizeof(double) * RP::TOTAL;
    const int grid_max = persistent_grid(reinterpret_cast<const void*>(k_residual_p<C, EPB>), RP::THREADS, smem);
    const int nbatch = (d.E + EPB - 1) / EPB;
    const int grid = nbatch < grid_max ? nbatch : grid_max;
    k_residual_p<C, EPB><<<grid, RP::THREADS, smem, d.stream>>>(params(d), U, Q, R);
    count(d);
    return cudaGetLastError();
  }
  static cudaError_t residual_f(const DevCtx& d, const double* U, const double* Q, double* R) {
    constexpr int EF = ResFEpb<C>::value;
    using RP = ResF<C, EF>;
    const size_t smem = sizeof(double) * RP::TOTAL;
    const int grid_max = persistent_grid(reinterpret_cast<const void*>(k_residual_f<C, EF>), RP::THREADS, smem);
    const int nbatch = (d.E + EF - 1) / EF;
    const int grid = nbatch < grid_max ? nbatch : grid_max;
    k_residual_f<C, EF><<<grid, RP::THREADS, smem, d.stream>>>(params(d), U, Q, R);
    count(d);
    return cudaGetLastError();
  }
  static cudaError_t gradient(const DevCtx& d, const double* U, double* Q) {
    if (!C::SECOND) return cudaSuccess;
    constexpr int EF = GradFEpb<C>::value;
    using GP = GradF<C, EF>;
    const size_t smem = sizeof(double) * GP::TOTAL;
    const int grid_max = persistent_grid(reinterpret_cast<const void*>(k_gradient_f<C, EF>), GP::THREADS, smem);
    const int nbatch = (d.E + EF - 1) / EF;
    const int grid = nbatch < grid_max ? nbatch : grid_max;
    k_gradient_f<C, EF><<<grid, GP::THREADS, smem, d.stream>>>(params(d), U, Q);
    count(d);
    return cudaGetLastError();
  }
  static constexpr size_t jac_smem() { return sizeof(double) * JacSmem<C>::TOTAL; }
  static constexpr int EJ_SEEDS = C::M;  // seeds per k_endjac thread (primal shared)
  // Elements per assembly chunk: the endpoint-Jacobian scratch of one chunk
  // stays within 512 MB.  Measured: fewer, larger chunks beat L2-sized ones
  // (kernel ramps and tails per chunk outweigh the scratch re-read; C2 one
  // chunk 0.252 vs 0.262 ms, C4 17.1 vs 18.3 ms).
  static int chunk_elems(int E) {
    const long long per = static_cast<long long>(SeLay<C>::PER_ELEM) * 8;
    long long n = (512LL << 20) / (per > 0 ? per : 1);
    if (n < 1024) n = 1024;
    // persistent line-streaming assembly: whole rounds of one element per SM
    // (B200: 148 SMs), so no SM idles through a chunk's last round
    if (JAC_KIND == 1 && n >= 4 * 148) n -= n % 148;
    return static_cast<int>(n < E ? n : E);
  }
  // Assembly kernel family of this configuration (compile-time):
  //   k_jacobian_p  persistent element units with a TMA prefetch ring (2-D, 3-D p <= 3)
  //   k_jac_s3      3-D line streaming (element flux-Jacobian set beyond shared memory)
  //   k_jacobian    one CTA per slab / line work unit (fallback)
  static constexpr int JAC_KIND = JacP<C>::OK ? 0 : ((C::D == 3 && C::WU != 0 && JacS3<C>::OK) ? 1 : 2);
  static cudaError_t jacobian(const DevCtx& d, const double* U, const double* Q, double* SE, double* K11,
                              double* K12) {
    constexpr int IPS = EndJac<C>::items(EJ_SEEDS);
    const size_t smem = jac_smem();
    const size_t psmem = sizeof(double) * JacP<C>::TOTAL;
    const size_t s3smem = sizeof(double) * JacS3<C>::TOTAL;
    int grid_max = 0;
    if (JAC_KIND == 0)
      grid_max = persistent_grid(reinterpret_cast<const void*>(k_jacobian_p<C>), JacThreads<C>::value, psmem);
    else if (JAC_KIND == 1)
      grid_max = persistent_grid(reinterpret_cast<const void*>(k_jac_s3<C>), JacS3<C>::THREADS, s3smem);
    else
      persistent_grid(reinterpret_cast<const void*>(k_jacobian<C>), JacThreads<C>::value, smem);
    const int chunk = chunk_elems(d.E);
    for (int kb = 0, ci = 0; kb < d.E; kb += chunk, ++ci) {
      const int ke = kb + chunk < d.E ? kb + chunk : d.E;
      // faces whose endpoint Jacobians this chunk computes
      const long long ob = d.owned ? d.owned_off[ci] : 0;
      const long long oe = d.owned ? d.owned_off[ci + 1] : static_cast<long long>(ke - kb) * 2 * C::D;
      const long long nf = oe - ob;
      // (fused configurations: the persistent assembly computes the endpoint
      // Jacobians itself)
      const bool fused = JacP<C>::FE && JAC_KIND == 0;
      if (!fused) {
        // (group-major scratch: one warp per (face, pass item), see k_endjac)
        const long long items = SeLay<C>::GM ? nf * IPS * 32 : nf * C::NL * IPS;
        k_endjac<C, EJ_SEEDS, false><<<static_cast<int>((items + 127) / 128), 128, 0, d.stream>>>(
            params(d), U, Q, SE, kb, ke, ob, oe, d.owned);
        count(d);
      }
      // slip-wall / Neumann boundary ends of the chunk (general kinds)
      if (d.bspec && d.bspec_off[ci + 1] > d.bspec_off[ci]) {
        const long long sb = d.bspec_off[ci], se = d.bspec_off[ci + 1];
        const long long items = (se - sb) * C::NL * EndJac<C>::items(1);
        k_endjac<C, 1, true><<<static_cast<int>((items + 127) / 128), 128, 0, d.stream>>>(
            params(d), U, Q, SE, kb, ke, sb, se, d.bspec);
        count(d);
      }
      const int n = ke - kb;
      const int grid = n < grid_max ? n : grid_max;
      if (JAC_KIND == 0) {
        k_jacobian_p<C><<<grid, JacThreads<C>::value, psmem, d.stream>>>(params(d), U, Q, SE, K11, K12, kb, ke);
      } else if (JAC_KIND == 1) {
        k_jac_s3<C><<<grid, JacS3<C>::THREADS, s3smem, d.stream>>>(params(d), U, Q, SE, K11, K12, kb, ke);
      } else {
        k_jacobian<C><<<(ke - kb) * C::UPE, JacThreads<C>::value, smem, d.stream>>>(params(d), U, Q, SE, K11,
                                                                                    K12, kb);
      }
      count(d);
    }
    return cudaGetLastError();
  }
  static size_t scratch_elems(int E) { return static_cast<size_t>(chunk_elems(E)) * SeLay<C>::PER_ELEM; }
  static cudaError_t k21(const DevCtx& d, double* K21) {
    if (!C::SECOND) return cudaSuccess;
    k_k21<C><<<d.E * C::UPE, 128, 0, d.stream>>>(params(d), K21);
    count(d);
    return cudaGetLastError();
  }
  static int rgrid(const DevCtx& d) {
    const long long rows = static_cast<long long>(d.E) * C::NPE;
    return static_cast<int>((rows + 127) / 128);
  }
  // one thread per (row, component), rows in groups of 32 per warp
  static int rgrid_m(const DevCtx& d) {
    const long long rows = static_cast<long long>(d.E) * C::NPE;
    const long long threads = (rows + 31) / 32 * 32 * C::M;
    return static_cast<int>((threads + 127) / 128);
  }
  // reverse row order for small stores (see k_spmv11); LDG_OPT_SPMV_ROW_ORDER forces it
  static int spmv_rev(const DevCtx& d) {
    if (d.spmv_order) return d.spmv_order == 2;
    const double store = 8.0 * d.E * C::NPE * C::NS11 * C::B11;
    return store <= static_cast<double>(1LL << 30) ? 1 : 0;
  }
  static cudaError_t spmv11(const DevCtx& d, const double* V11, const double* x, double* y) {
    k_spmv11<C, false><<<rgrid_m(d), 128, 0, d.stream>>>(params(d), V11, nullptr, x, nullptr, 0.0, y, spmv_rev(d));
    count(d);
    return cudaGetLastError();
  }
  static cudaError_t spmv11_zc(const DevCtx& d, const double* V11, const double* x, double* y) {
    k_spmv11<C, false, true><<<rgrid_m(d), 128, 0, d.stream>>>(params(d), V11, nullptr, x, nullptr, 0.0, y,
                                                               spmv_rev(d));
    count(d);
    return cudaGetLastError();
  }
  static cudaError_t spmv12(const DevCtx& d, const double* V12, const double* w, double* y) {
    if (!C::SECOND) return cudaSuccess;
    k_spmv12<C><<<rgrid_m(d), 128, 0, d.stream>>>(params(d), V12, w, y);
    count(d);
    return cudaGetLastError();
  }
  static cudaError_t spmv21(const DevCtx& d, const double* V21, const double* v, double* w) {
    if (!C::SECOND) return cudaSuccess;
    // one thread per row (measured C5: one thread per (row, component) 2.35 vs 1.97 ms)
    k_spmv21<C><<<rgrid(d), 128, 0, d.stream>>>(params(d), V21, v, w);
    count(d);
    return cudaGetLastError();
  }
  static cudaError_t split(const DevCtx& d, const double* V11, const double* V12, const double* v,
                           const double* w, double adt, double* y) {
    if (MvT<C>::OK) {
      // second-order physics: TMA tile streaming of K11 + K12 (k_mv_tiles)
      const size_t smem = sizeof(double) * MvT<C>::TOTAL;
      const int grid = persistent_grid(reinterpret_cast<const void*>(k_mv_tiles<C>), MvT<C>::THREADS, smem);
      k_mv_tiles<C><<<grid, MvT<C>::THREADS, smem, d.stream>>>(params(d), V11, V12, v, w, adt, y);
      count(d);
      return cudaGetLastError();
    }
    k_spmv11<C, true><<<rgrid_m(d), 128, 0, d.stream>>>(params(d), V11, V12, v, w, adt, y, spmv_rev(d));
    count(d);
    return cudaGetLastError();
  }

  template <bool INV>
  static void pc_build_t(const DevCtx& d, const double* V11, const double* V12, const double* V21, double adt,
                         double* LUc, int32_t* piv, int* bad) {
    using PC = PcCfg<C, INV>;
    persistent_grid(reinterpret_cast<const void*>(k_pc_build<C, INV>), PC::THREADS, PC::smem());
    k_pc_build<C, INV><<<d.E, PC::THREADS, PC::smem(), d.stream>>>(params(d), V11, V12, V21, adt, LUc, piv, bad);
  }
  static cudaError_t pc_build(const DevCtx& d, const double* V11, const double* V12, const double* V21, double adt,
                              double* LUc, int32_t* piv, int* bad) {
    if (!PcCfg<C>::OK) return cudaErrorNotSupported;
    if (d.pc_inverse) pc_build_t<true>(d, V11, V12, V21, adt, LUc, piv, bad);
    else pc_build_t<false>(d, V11, V12, V21, adt, LUc, piv, bad);
    count(d);
    return cudaGetLastError();
  }
  static cudaError_t pc_apply(const DevCtx& d, const double* LUc, const int32_t* piv, const double* r, double* z) {
    if (!PcCfg<C>::OK) return cudaErrorNotSupported;
    if (d.pc_inverse) k_pc_apply<C, true><<<(d.E + 3) / 4, 128, 0, d.stream>>>(params(d), LUc, piv, r, z);
    else k_pc_apply_lu2<C><<<(d.E + 4 * LDG_PC_EPW - 1) / (4 * LDG_PC_EPW), 128, 0, d.stream>>>(params(d), LUc, piv,
                                                                                              r, z);
    count(d);
    return cudaGetLastError();
  }
  static cudaError_t pc_line_build(const DevCtx& d, const double* V11, const double* V12, const double* V21,
                                   double adt, double* LUc, int32_t* piv, int* bad) {
    using PL = PcLine<C>;
    if (!PL::OK) return cudaErrorNotSupported;
    persistent_grid(reinterpret_cast<const void*>(k_pc_line_build<C>), PL::THREADS, PL::smem());
    k_pc_line_build<C><<<dim3(d.E, C::D), PL::THREADS, PL::smem(), d.stream>>>(params(d), V11, V12, V21, adt, LUc,
                                                                              piv, bad);
    count(d);
    return cudaGetLastError();
  }
  static cudaError_t pc_line_apply(const DevCtx& d, const double* LUc, const int32_t* piv, const double* r,
                                   double* z) {
    if (!PcLine<C>::OK) return cudaErrorNotSupported;
    k_pc_line_apply<C><<<d.E, 256, 0, d.stream>>>(params(d), LUc, piv, r, z);
    count(d);
    return cudaGetLastError();
  }
  static const Ops* table() {
    static const Ops ops = {C::D, C::P, C::PH, C::RI, C::M, C::NP, C::NQ, C::NPE, C::NL, C::MD,
                            C::NS11, C::NS12, C::B11, C::B12, C::R12, C::NT, C::TPE, C::METP,
                            C::MET_NV, C::MET_NE, jac_smem(), SeLay<C>::PER_ELEM, scratch_elems, chunk_elems, residual, gradient, jacobian, k21,
                            spmv11, spmv11_zc, spmv12, spmv21, split, PcCfg<C>::OK ? PcCfg<C>::NE : 0, pc_build, pc_apply,
                            PcLine<C>::OK ? PcLine<C>::NB : 0, pc_line_build, pc_line_apply};
    return &ops;
  }
};

}  // namespace ldg

#define LDG_OPS_NAME(D, P, PH, RI) ldg_ops_##D##_##P##_##PH##_##RI
#define LDG_DECLARE_OPS(D, P, PH, RI) const ldg::Ops* LDG_OPS_NAME(D, P, PH, RI)();
#define LDG_DEFINE_OPS(D, P, PH, RI) \
  const ldg::Ops* LDG_OPS_NAME(D, P, PH, RI)() { return ldg::Launch<ldg::Cfg<D, P, PH, RI>>::table(); }
