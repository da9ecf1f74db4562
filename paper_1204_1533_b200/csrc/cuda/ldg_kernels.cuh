// ldg_kernels.cuh -- sm_100a kernels of the Line-DG hot path.
//
// Work decomposition:
//   * residual / gradient: one thread per 1-D coordinate line (all m
//     components), EPB elements per CTA.  The element's nodal states are
//     staged in shared memory; the (p+1) x n_q line contractions run in
//     registers with the basis tables as compile-time-indexed constant-bank
//     operands; per-direction line results meet in shared memory, so no
//     atomics are needed (PAPER.md:285 sums r^(n) over directions).
//   * Jacobian: one CTA per row tile (2-D: one element, 3-D: one x2-slab of
//     an element).  Flux Jacobians at quadrature points / line ends come
//     from a forward-mode Dual<N>; the line blocks
//     B(i,t) = sum_q dq[i][q] phi[t][q] A_q are formed by one thread per
//     (line, a, b) with all coefficients as constants, staged in shared
//     memory in the store's layout and written with 16-byte coalesced
//     stores.  Rows are never shared between CTAs: no atomics.
//   * SpMV: one thread per node row; the store is interleaved so a warp's
//     value loads are contiguous; in-element column nodes are implied by the
//     row's position on its lines, neighbour columns come from the face
//     connectivity (no column-index stream).
#pragma once

#include <type_traits>

#include "ldg_device.cuh"

namespace ldg {

template <class C>
struct KParams {
  BasisTab<C::NP, C::NQ> bt;
  PhysParams pp;
  const int32_t* order;  // processing index k -> reference element e
  const double* metric;  // [k][METP]
  const int2* conn;      // [k][D][2]
  const double* bcv;     // [nbc][M] boundary data (Dirichlet / far-field state, Neumann flux)
  const int32_t* bck;    // [nbc] boundary kind (BcKindDev)
  int noslip;            // number of no-slip-wall boundary conditions (K21 wall terms)
  const int32_t* bface;  // [k][2D] boundary-face index into bvals, -1: constant data (null: none)
  const double* bvals;   // [bface][NL][M] boundary data per line end (ldg_set_boundary_function)
  const double* source;  // reference numbering, may be null
  DevError* err;
  const int2* fpart;     // [k][2D] face partner {k', 2 dir' + side'} ({-1, 0}: none)
  const int32_t* inv_order;  // reference element e -> processing index k
  const int32_t* owned;  // owned faces (k*2D + ds) of the Jacobian chunks, or null
  int E;                 // elements
};

// Numerical flux F_hat.n at a boundary line end (SPEC.md:266,
// 366-368), bc = boundary index, n the non-normalised outward normal, nn = |n|:
//   Dirichlet / characteristic: Riemann flux against g (the prescribed /
//     free-stream state) + viscous F(u_in, q_in).n + C11_bd |n| (u_in - g);
//   slip wall: Riemann flux against the mirrored-normal-momentum ghost of
//     u_in + viscous F(u_in, q_in).n (no penalty);
//   Neumann: the prescribed normal flux g_N |n| (no other term).
// T = double or Dual<N> in u_in; TQ the type of q_in.
// Boundary data of one line end: per-node values from a boundary function
// (ldg_set_boundary_function: the reference's std::function g_D / g_N / far
// state evaluated at the end node) or the boundary condition's constants.
template <class C>
__device__ __forceinline__ const double* bnd_g(const KParams<C>& kp, int bc, int k, int ds, int line) {
  if (kp.bface) {
    const int f = __ldg(kp.bface + static_cast<size_t>(k) * 2 * C::D + ds);
    if (f >= 0) return kp.bvals + (static_cast<size_t>(f) * C::NL + line) * C::M;
  }
  return kp.bcv + bc * C::M;
}

template <class C, class T, class TQ>
__device__ __forceinline__ void bnd_flux(const KParams<C>& kp, int bc, const double* g, const T* ui, const TQ* qi,
                                         const double* n, double nn, T* fh, bool& ok) {
  constexpr int M = C::M, D = C::D;
  const int kind = __ldg(kp.bck + bc);
#pragma unroll
  for (int c = 0; c < M; ++c) fh[c] = T(0.0);
  if (kind == BC_NEUMANN) {
#pragma unroll
    for (int c = 0; c < M; ++c) fh[c] = T(__ldg(g + c) * nn);
    return;
  }
  if (C::HAS_INV) {
    T uo[M];
    bc_ghost<D, M>(kind, g, ui, n, uo);
    if (C::RI == LDG_ROE) roe_fn<D>(uo, ui, n, kp.pp.gamma, fh, ok);
    else llf_fn<D>(uo, ui, n, kp.pp.gamma, fh, ok);
  }
  if (C::SECOND) {
    T fv[M];
    visc_fn<D, C::PH, T, TQ, T>(ui, qi, n, kp.pp, fv, ok);
    if (kind == BC_SLIP_WALL) {
#pragma unroll
      for (int c = 0; c < M; ++c) fh[c] = fh[c] + fv[c];
    } else if (kind == BC_NO_SLIP) {
      // momentum: Dirichlet zero velocity (penalty on m - 0); density row of F
      // is zero; energy: zero normal flux (adiabatic, no wall work)
      const double c11 = kp.pp.c11bd / (D == 2 ? nn : sqrt(nn));
      fh[0] = fh[0] + fv[0];
#pragma unroll
      for (int c = 1; c < M - 1; ++c) fh[c] = fh[c] + (fv[c] + (c11 * nn) * ui[c]);
    } else {
      const double c11 = kp.pp.c11bd / (D == 2 ? nn : sqrt(nn));
#pragma unroll
      for (int c = 0; c < M; ++c) fh[c] = fh[c] + (fv[c] + (c11 * nn) * (ui[c] - __ldg(g + c)));
    }
  }
}
// u_hat of the auxiliary gradient at a boundary end: g (Dirichlet-type,
// PAPER.md:573) or the interior trace (Neumann-type with C22 = 0,
// PAPER.md:580; slip wall)
template <class C>
__device__ __forceinline__ bool bnd_uhat_inner(const KParams<C>& kp, int bc) {
  const int kind = __ldg(kp.bck + bc);
  return kind == BC_NEUMANN || kind == BC_SLIP_WALL;
}
// u_hat of component c at a boundary end with interior trace uin: the
// no-slip adiabatic wall is mixed -- zero momentum (Dirichlet
// velocity), interior density and energy (Neumann-type, C22 = 0)
template <class C>
__device__ __forceinline__ double bnd_uhat(const KParams<C>& kp, int bc, const double* g, int c, double uin) {
  const int kind = __ldg(kp.bck + bc);
  if (kind == BC_NO_SLIP) return (c == 0 || c == C::M - 1) ? uin : 0.0;
  if (kind == BC_NEUMANN || kind == BC_SLIP_WALL) return uin;
  return __ldg(g + c);
}

static constexpr int LDG_VISC_DU = 1;  // closed-form viscous dF/du (1) or dual numbers (0)
constexpr bool VISC_DU_CLOSED = LDG_VISC_DU != 0;

static constexpr int LDG_JAC_SMEMTAB = 0;  // tuning knob: assembly basis coefficients from shared memory (1) or the constant bank (0); measured: the constant bank wins (C2 0.266 vs 0.311 ms) despite its spills
constexpr int JAC_SMEMTAB = LDG_JAC_SMEMTAB;
static constexpr int LDG_JAC_CHAINS = 1;  // assembly: line-block sums as one (1) or two (2) dependent DFMA chains
constexpr int JAC_CHAINS = LDG_JAC_CHAINS;
  // 0 constant bank, 1 shared (scalar), 2 shared (pairs)
// ---------------------------------------------------------------- helpers

// f(integral_constant<int, 0>) ... f(integral_constant<int, N - 1>)
template <int N, int I = 0, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    static_for<N, I + 1>(f);
  }
}

template <class C>
__device__ __forceinline__ int node_on_line(int dir, int line, int t) {
  constexpr int NP = C::NP;
  if (C::D == 2) return dir == 0 ? t + NP * line : line + NP * t;
  const int l1 = line % NP, l2 = line / NP;
  if (dir == 0) return t + NP * l1 + NP * NP * l2;
  if (dir == 1) return l1 + NP * t + NP * NP * l2;
  return l1 + NP * l2 + NP * NP * t;
}

// Line index of the dir-line through node `nd`, and the node's position on it.
template <class C>
__device__ __forceinline__ void line_of(int dir, int nd, int& line, int& pos) {
  constexpr int NP = C::NP;
  const int x0 = nd % NP, x1 = (nd / NP) % NP, x2 = nd / (NP * NP);
  if (C::D == 2) {
    line = dir == 0 ? x1 : x0;
    pos = dir == 0 ? x0 : x1;
  } else {
    if (dir == 0) { line = x1 + NP * x2; pos = x0; }
    else if (dir == 1) { line = x0 + NP * x2; pos = x1; }
    else { line = x0 + NP * x1; pos = x2; }
  }
}

__device__ __forceinline__ int conn_node(int packed, int line, int NP) {
  const int c0 = packed & 0xff;
  const int c1 = static_cast<int8_t>((packed >> 8) & 0xff);
  const int c2 = static_cast<int8_t>((packed >> 16) & 0xff);
  return c0 + c1 * (line % NP) + c2 * (line / NP);
}
__device__ __forceinline__ int conn_sign(int packed) { return (packed >> 24) & 1 ? 1 : -1; }

// K11 slot of column node `col` on the dir-line through row (pos = row's
// position on that line).  Slots: dir-0 line nodes t (self included), then
// for dir d >= 1 the P non-self nodes, then neighbours 2*dir+side.
template <class C>
__device__ __forceinline__ int inel_slot(int dir, int pos, int t) {
  if (dir == 0) return t;
  return C::NP + (dir - 1) * C::P + (t < pos ? t : t - 1);
}

template <class C>
__device__ __forceinline__ void cp_elem(double* dst, const double* __restrict__ src, int n, int tid,
                                        int nthr) {
  // 16-byte vector copy when both sides are aligned (n even and src aligned).
  if ((n & 1) == 0 && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
    const double2* s2 = reinterpret_cast<const double2*>(src);
    double2* d2 = reinterpret_cast<double2*>(dst);
    for (int i = tid; i < n / 2; i += nthr) d2[i] = __ldg(s2 + i);
  } else {
    for (int i = tid; i < n; i += nthr) dst[i] = __ldg(src + i);
  }
}


// Physical-state failure on a line: report the first nodal state on the line
// that is itself non-physical (rho <= 0 or p <= 0), else the line's first node
// (the failure was at an interpolated quadrature state).
template <class C>
__device__ __noinline__ void report_line(const KParams<C>& kp, int e, int dir, int line,
                                         const double* su) {
  constexpr int M = C::M, D = C::D;
  int bad = node_on_line<C>(dir, line, 0);
  if (C::HAS_INV) {
    for (int t = 0; t < C::NP; ++t) {
      const int nd = node_on_line<C>(dir, line, t);
      const double* u = su + nd * M;
      double m2 = 0.0;
      for (int d = 0; d < D; ++d) m2 += u[1 + d] * u[1 + d];
      const double p = (kp.pp.gamma - 1.0) * (u[D + 1] - 0.5 * m2 / u[0]);
      if (!(u[0] > 0.0) || !(p > 0.0)) {
        bad = nd;
        break;
      }
    }
  }
  report_bad_state<double, M>(kp.err, e, bad, su + bad * M);
}

// ------------------------------------------------------ async copy helpers
// TMA 1-D bulk copies global -> shared completing on an mbarrier
// (cp.async.bulk ... mbarrier::complete_tx, SASS UBLKCP) and Ampere-style
// cp.async gathers (LDGSTS) for the scattered neighbour traces.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* sdst, const void* gsrc, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Same with an L2 evict-first policy (data read exactly once).
__device__ __forceinline__ void tma_load_1d_once(void* sdst, const void* gsrc, unsigned bytes, uint64_t* bar) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          smem_u32(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
// N consecutive doubles: 16-byte copies when N is even (source and destination
// are then 16-byte aligned: nodal traces of m or m*D doubles at multiples of
// N doubles from 16-byte-aligned bases), else 8-byte copies.
template <int N>
__device__ __forceinline__ void cp_async_run(double* sdst, const double* gsrc) {
  if (N % 2 == 0) {
#pragma unroll
    for (int c = 0; c < N; c += 2) cp_async16(sdst + c, gsrc + c);
  } else {
#pragma unroll
    for (int c = 0; c < N; ++c) cp_async8(sdst + c, gsrc + c);
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Staged tile -> global, asynchronous: TMA bulk copy (cp.async.bulk, SASS
// UBLKCP) issued by thread 0 when size and both addresses are 16-byte
// multiples (else plain stores).  store_wait() returns once the copy has read
// the staging buffer (thread 0 waits on its bulk group, then a CTA barrier).
__device__ __forceinline__ void store_issue(double* __restrict__ gdst, const double* ssrc, int n, int tid,
                                            int nthr) {
  const unsigned bytes = static_cast<unsigned>(n) * 8u;
  const bool bulk = (bytes % 16u) == 0 && aligned16(gdst) && aligned16(ssrc);
  if (bulk) {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst),
                   "r"(smem_u32(ssrc)), "r"(bytes)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
  } else {
    __syncthreads();
    for (int i = tid; i < n; i += nthr) gdst[i] = ssrc[i];
  }
}
__device__ __forceinline__ void store_wait(int tid) {
  if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
  __syncthreads();
}

// Staged tile -> global.  TMA bulk copy (cp.async.bulk, SASS UBLKCP) when the
// size and both addresses are 16-byte multiples, else 16/8-byte stores.
// Must be reached by all threads of the CTA; returns with the smem source
// free for reuse.
__device__ __forceinline__ void store_tile(double* __restrict__ gdst, const double* ssrc, int n, int tid,
                                           int nthr) {
  const unsigned bytes = static_cast<unsigned>(n) * 8u;
  const bool bulk = (bytes % 16u) == 0 && ((reinterpret_cast<uintptr_t>(gdst) & 15) == 0) &&
                    ((reinterpret_cast<uintptr_t>(ssrc) & 15) == 0);
  if (bulk) {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(ssrc));
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst), "r"(saddr),
                   "r"(bytes)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    }
    __syncthreads();
  } else {
    __syncthreads();
    for (int i = tid; i < n; i += nthr) gdst[i] = ssrc[i];
    __syncthreads();
  }
}

// ================================================= residual, persistent + TMA
// Persistent CTAs walk batches of EPB elements (grid-stride).  Two smem
// buffers: while batch i is computed from buffer i%2, the TMA engine fills the
// other buffer with batch i+1 (element states -- one bulk copy per element,
// the batch's metric and connectivity -- one bulk copy each, all completing on
// one mbarrier); the scattered neighbour traces of batch i+1 are gathered with
// cp.async as soon as its connectivity has landed.  Compute is
// thread-per-line with every operand in shared memory.
static constexpr int LDG_RES_MET_SMEM = 1;  // residual: stage the metric in the ring (1) or read it from global (0)
template <class C, int EPB>
struct ResP {
  static constexpr int ev(int x) { return (x + 1) / 2 * 2; }
  static constexpr bool METS = LDG_RES_MET_SMEM != 0;
  static constexpr int U = ev(EPB * C::NPE * C::M);
  static constexpr int Q = C::SECOND ? ev(EPB * C::NPE * C::MD) : 0;
  static constexpr int MET = METS ? EPB * C::METP : 0;
  static constexpr int CONN = ev(EPB * C::D * 2);  // int2 entries, 8 B each
  static constexpr int NB = ev(EPB * C::LPE * 2 * C::M);
  static constexpr int NBQ = C::SECOND ? ev(EPB * C::LPE * 2 * C::MD) : 0;
  static constexpr int BUF = U + Q + MET + CONN + NB + NBQ;
  // SPLIT threads per line (warp-uniform halves: the first half of the CTA
  // takes the first quadrature points and the left end of every line, the
  // second half the rest and the right end; per-half partial sums in ACC)
static constexpr int LDG_RES_SPLIT = 1;  // measured slower for C2/C4 (more warps, same latency chains): off
  static constexpr int SPLIT = LDG_RES_SPLIT;
  static constexpr int LT = (EPB * C::LPE + 31) / 32 * 32;  // line threads of one half
  static constexpr int ACC = SPLIT * EPB * C::D * C::NPE * C::M;
  static constexpr int TOTAL = 2 + 2 * BUF + ACC;  // 2 doubles hold the two mbarriers
  static constexpr bool TMA = (C::NPE * C::M) % 2 == 0 && (!C::SECOND || (C::NPE * C::MD) % 2 == 0);
  static constexpr int THREADS = SPLIT * LT;
};

static constexpr int LDG_RES_MINB = 1;  // k_residual_p min CTAs per SM (register cap)
template <class C, int EPB>
__global__ void __launch_bounds__(ResP<C, EPB>::THREADS, LDG_RES_MINB)
k_residual_p(const KParams<C> kp, const double* __restrict__ U, const double* __restrict__ Q,
             double* __restrict__ R) {
  constexpr int NP = C::NP, NQ = C::NQ, NPE = C::NPE, NL = C::NL, M = C::M, D = C::D, MD = C::MD,
                LPE = C::LPE, P = C::P;
  using RP = ResP<C, EPB>;
  extern __shared__ __align__(16) double smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  double* const bufs = smem + 2;
  double* const sacc = bufs + 2 * RP::BUF;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int nbatch = (kp.E + EPB - 1) / EPB;
  const int G = gridDim.x;
  if (static_cast<int>(blockIdx.x) >= nbatch) return;
  auto bU = [&](int bi) { return bufs + bi * RP::BUF; };
  auto bQ = [&](int bi) { return bufs + bi * RP::BUF + RP::U; };
  auto bMET = [&](int bi) { return bufs + bi * RP::BUF + RP::U + RP::Q; };
  auto bCONN = [&](int bi) { return reinterpret_cast<int2*>(bufs + bi * RP::BUF + RP::U + RP::Q + RP::MET); };
  auto bNB = [&](int bi) { return bufs + bi * RP::BUF + RP::U + RP::Q + RP::MET + RP::CONN; };
  auto bNBQ = [&](int bi) { return bufs + bi * RP::BUF + RP::U + RP::Q + RP::MET + RP::CONN + RP::NB; };
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  // bulk loads of one batch into buffer bi (thread 0 issues; TMA path)
  auto issue = [&](int batch, int bi) {
    const int k0 = batch * EPB, nb = min(EPB, kp.E - k0);
    unsigned bytes = nb * (NPE * M * 8) + (RP::METS ? nb * C::METP * 8 : 0) + nb * D * 2 * 8;
    if (C::SECOND) bytes += nb * (NPE * MD * 8);
    int ev_[EPB];
#pragma unroll
    for (int le = 0; le < EPB; ++le) ev_[le] = le < nb ? __ldg(kp.order + k0 + le) : 0;
    mbar_expect_tx(&bar[bi], bytes);
#pragma unroll
    for (int le = 0; le < EPB; ++le) {
      if (le >= nb) break;
      const size_t e = static_cast<size_t>(ev_[le]);
      tma_load_1d(bU(bi) + le * NPE * M, U + e * (NPE * M), NPE * M * 8, &bar[bi]);
      if (C::SECOND) tma_load_1d(bQ(bi) + le * NPE * MD, Q + e * (NPE * MD), NPE * MD * 8, &bar[bi]);
    }
    if (RP::METS) tma_load_1d(bMET(bi), kp.metric + static_cast<size_t>(k0) * C::METP, nb * C::METP * 8, &bar[bi]);
    tma_load_1d(bCONN(bi), kp.conn + static_cast<size_t>(k0) * D * 2, nb * D * 2 * 8, &bar[bi]);
  };
  // synchronous fallback (element chunks not 16-byte aligned)
  auto load_sync = [&](int batch, int bi) {
    const int k0 = batch * EPB, nb = min(EPB, kp.E - k0);
    for (int le = 0; le < nb; ++le) {
      const size_t e = kp.order[k0 + le];
      for (int i = tid; i < NPE * M; i += nthr) bU(bi)[le * NPE * M + i] = __ldg(U + e * (NPE * M) + i);
      if (C::SECOND)
        for (int i = tid; i < NPE * MD; i += nthr) bQ(bi)[le * NPE * MD + i] = __ldg(Q + e * (NPE * MD) + i);
    }
    if (RP::METS)
      for (int i = tid; i < nb * C::METP; i += nthr) bMET(bi)[i] = __ldg(kp.metric + static_cast<size_t>(k0) * C::METP + i);
    for (int i = tid; i < nb * D * 2; i += nthr) bCONN(bi)[i] = __ldg(kp.conn + static_cast<size_t>(k0) * D * 2 + i);
    __syncthreads();
  };
  // neighbour-trace gathers of buffer bi (all threads; needs its connectivity)
  auto gather = [&](int batch, int bi) {
    const int k0 = batch * EPB, nb = min(EPB, kp.E - k0);
    const int2* sc = bCONN(bi);
    for (int w = tid; w < nb * LPE * 2; w += nthr) {
      const int side = w & 1, lw = w >> 1, le = lw / LPE, rem = lw - le * LPE;
      const int dir = rem / NL, line = rem - dir * NL;
      const int2 cn = sc[(le * D + dir) * 2 + side];
      if (cn.x < 0) continue;
      const size_t nd = static_cast<size_t>(cn.x) * NPE + conn_node(cn.y, line, NP);
      double* dst = bNB(bi) + w * M;
      cp_async_run<M>(dst, U + nd * M);
      if (C::SECOND && conn_sign(cn.y) > 0) {
        double* dq = bNBQ(bi) + w * MD;
        cp_async_run<MD>(dq, Q + nd * MD);
      }
    }
    cp_async_commit();
  };

  const int b0 = blockIdx.x;
  if (RP::TMA) {
    if (tid == 0) {
      issue(b0, 0);
      if (b0 + G < nbatch) issue(b0 + G, 1);
    }
    mbar_wait(&bar[0], 0);
  } else {
    load_sync(b0, 0);
  }
  gather(b0, 0);
  __shared__ int sord[EPB];  // element ids of the batch (epilogue addresses)
  for (int batch = b0, it = 0; batch < nbatch; batch += G, ++it) {
    const int cur = it & 1, nxt = cur ^ 1;
    const int k0 = batch * EPB, nb = min(EPB, kp.E - k0);
    cp_async_wait_all();
    __syncthreads();
    if (tid < nb) sord[tid] = __ldg(kp.order + k0 + tid);  // lands during the line work
    // ---- lines (RP::SPLIT threads per line, warp-uniform halves; the body is
    // instantiated per half so each thread issues only its own points)
    const int half_rt = RP::SPLIT > 1 ? tid / RP::LT : 0, lt = tid - half_rt * RP::LT;
    constexpr int QH = RP::SPLIT > 1 ? (NQ + 1) / 2 : NQ;
    const int le = lt / LPE;
    auto line_work = [&](auto HC) {
      constexpr int half = decltype(HC)::value;
      const int rem = lt - le * LPE;
      const int dir = rem / NL, line = rem - dir * NL;
      const double* mk = RP::METS ? bMET(cur) + le * C::METP : kp.metric + static_cast<size_t>(k0 + le) * C::METP;
      const double* nvl = mk + (dir * NL + line) * NQ * D;
      const double* sul = bU(cur) + le * NPE * M;
      const double* sql = bQ(cur) + le * NPE * MD;
      bool ok = true;
      double r[NP][M];
#pragma unroll
      for (int i = 0; i < NP; ++i)
#pragma unroll
        for (int c = 0; c < M; ++c) r[i][c] = 0.0;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        if (RP::SPLIT > 1 && ((q < QH) != (half == 0))) continue;  // compile-time
        double uq[M], qq[C::SECOND ? MD : 1];
#pragma unroll
        for (int c = 0; c < M; ++c) uq[c] = 0.0;
        if (C::SECOND) {
#pragma unroll
          for (int c = 0; c < MD; ++c) qq[c] = 0.0;
        }
#pragma unroll
        for (int t = 0; t < NP; ++t) {
          const int nd = node_on_line<C>(dir, line, t);
          const double ph = kp.bt.phi[t][q];
#pragma unroll
          for (int c = 0; c < M; ++c) uq[c] += ph * sul[nd * M + c];
          if (C::SECOND) {
#pragma unroll
            for (int c = 0; c < MD; ++c) qq[c] += ph * sql[nd * MD + c];
          }
        }
        double nv[D];
#pragma unroll
        for (int d = 0; d < D; ++d) nv[d] = nvl[q * D + d];
        double f[M];
#pragma unroll
        for (int c = 0; c < M; ++c) f[c] = 0.0;
        if (C::HAS_INV) euler_fn<D>(uq, nv, kp.pp.gamma, f, ok);
        if (C::SECOND) {
          double fv[M];
          visc_fn<D, C::PH, double, double, double>(uq, qq, nv, kp.pp, fv, ok);
#pragma unroll
          for (int c = 0; c < M; ++c) f[c] += fv[c];
        }
#pragma unroll
        for (int i = 0; i < NP; ++i)
#pragma unroll
          for (int c = 0; c < M; ++c) r[i][c] += kp.bt.dq[i][q] * f[c];
      }
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        if (RP::SPLIT > 1 && side != half) continue;  // compile-time
        const int2 cn = bCONN(cur)[(le * D + dir) * 2 + side];
        const int S = conn_sign(cn.y);
        const int ie = side ? P : 0;
        const int nd = node_on_line<C>(dir, line, ie);
        const double* nep = mk + C::MET_NV + ((dir * 2 + side) * NL + line) * D;
        const int w = ((le * LPE + rem) << 1) | side;
        double n[D], ui[M], uo[M], fh[M];
#pragma unroll
        for (int d = 0; d < D; ++d) n[d] = nep[d];
        const double* bcp = cn.x < 0 ? bnd_g(kp, -1 - cn.x, k0 + le, dir * 2 + side, line) : nullptr;
#pragma unroll
        for (int c = 0; c < M; ++c) {
          ui[c] = sul[nd * M + c];
          uo[c] = bcp ? __ldg(bcp + c) : bNB(cur)[w * M + c];
          fh[c] = 0.0;
        }
        if (bcp) {
          double nn = n[0] * n[0];
#pragma unroll
          for (int d = 1; d < D; ++d) nn += n[d] * n[d];
          nn = sqrt(nn);
          bnd_flux<C>(kp, -1 - cn.x, bcp, ui, (C::SECOND ? sql + nd * MD : sul), n, nn, fh, ok);
        } else {
          if (C::HAS_INV) {
            if (C::RI == LDG_ROE) roe_fn<D>(uo, ui, n, kp.pp.gamma, fh, ok);
            else llf_fn<D>(uo, ui, n, kp.pp.gamma, fh, ok);
          }
          if (C::SECOND) {
            double nn = n[0] * n[0];
#pragma unroll
            for (int d = 1; d < D; ++d) nn += n[d] * n[d];
            nn = sqrt(nn);
            double fv[M];
            if (S > 0) visc_fn<D, C::PH, double, double, double>(uo, bNBQ(cur) + w * MD, n, kp.pp, fv, ok);
            else visc_fn<D, C::PH, double, double, double>(ui, sql + nd * MD, n, kp.pp, fv, ok);
#pragma unroll
            for (int c = 0; c < M; ++c) fh[c] += fv[c];
            if (kp.pp.c11 != 0.0) {
#pragma unroll
              for (int c = 0; c < M; ++c) fh[c] += kp.pp.c11 * nn * (ui[c] - uo[c]);
            }
          }
        }
#pragma unroll
        for (int i = 0; i < NP; ++i)
#pragma unroll
          for (int c = 0; c < M; ++c) r[i][c] += kp.bt.mi[i][side] * fh[c];
      }
      if (!ok) report_line<C>(kp, kp.order[k0 + le], dir, line, sul);
      double* acc = sacc + ((half * EPB + le) * D + dir) * NPE * M;
#pragma unroll
      for (int t = 0; t < NP; ++t) {
        const int nd = node_on_line<C>(dir, line, t);
#pragma unroll
        for (int c = 0; c < M; ++c) acc[nd * M + c] = r[t][c];
      }
    };
    if (le < nb) {
      if (RP::SPLIT > 1 && half_rt == 1) line_work(std::integral_constant<int, 1>{});
      else line_work(std::integral_constant<int, 0>{});
    }
    __syncthreads();
    // ---- dU/dt = S - (1/J) sum_dir r
    // (even element blocks: two entries per thread, one 16-byte store)
    constexpr int EW = (NPE * M) % 2 == 0 ? 2 : 1;
    for (int idx = tid * EW; idx < nb * NPE * M; idx += nthr * EW) {
      const int l = idx / (NPE * M), off = idx - l * NPE * M;
      const size_t e = static_cast<size_t>(sord[l]);
      double val[EW];
#pragma unroll
      for (int x = 0; x < EW; ++x) {
        const int nd = (off + x) / M;
        const double* a = sacc + l * D * NPE * M + off + x;
        double sum = a[0];
#pragma unroll
        for (int d = 1; d < D; ++d) sum = sum + a[d * NPE * M];
#pragma unroll
        for (int h = 1; h < RP::SPLIT; ++h)
#pragma unroll
          for (int d = 0; d < D; ++d) sum = sum + a[(h * EPB * D + d) * NPE * M];
        const double invJ = RP::METS ? bMET(cur)[l * C::METP + C::MET_NV + C::MET_NE + nd]
                                     : __ldg(kp.metric + static_cast<size_t>(k0 + l) * C::METP + C::MET_NV + C::MET_NE + nd);
        const double src = kp.source ? __ldg(kp.source + e * (NPE * M) + off + x) : 0.0;
        val[x] = src - invJ * sum;
      }
      double* out = R + e * (NPE * M) + off;
      if (EW == 2) *reinterpret_cast<double2*>(out) = make_double2(val[0], val[EW - 1]);
      else out[0] = val[0];
    }
    // ---- next batch: its bulk data was issued one iteration ago
    const int nbn = batch + G;
    if (nbn < nbatch) {
      if (RP::TMA) mbar_wait(&bar[nxt], ((it + 1) >> 1) & 1);
      else {
        __syncthreads();
        load_sync(nbn, nxt);
      }
      gather(nbn, nxt);
    }
    __syncthreads();  // buffer `cur` is free
    if (RP::TMA && tid == 0 && batch + 2 * G < nbatch) issue(batch + 2 * G, cur);
  }
}

// ============================== residual, persistent + TMA, flux-parallel
// Same prefetch ring as k_residual_p (TMA bulk copies of a batch's element
// states, metric and connectivity on an mbarrier; neighbour traces by
// cp.async), but the work of a batch is flattened into short independent
// items so many more warps are resident:
//   R1  one item per (element, line, quadrature point): F(u_q).nvec_q (+ the
//       viscous flux) into shared memory;
//   R2  one item per (element, line end): the Riemann (+ LDG switch) flux;
//   R3  one item per (element, node, component): the line projections
//       r = sum_q dq[i][q] F_q + mi[i][0] Fh_0 + mi[i][1] Fh_1 summed over the
//       D lines through the node, dU/dt = S - (1/J) sum (coalesced store).
// Basis tables live in shared memory (lane-dependent indices).
// Batch input ring shared by the flattened residual and gradient kernels:
// two buffers of EPB elements {U, (Q), metric, connectivity, element ids,
// neighbour traces (U; Q where the switch selects the neighbour)}; bulk data
// by TMA on one mbarrier per buffer; neighbour traces by cp.async one batch
// ahead of the bulk data, driven by a small connectivity ring.
// Element blocks of an odd number of doubles (odd NPE and odd M: 3-D p = 2, 4)
// start 8 bytes off a 16-byte boundary for odd element ids: the bulk copy then
// takes the enclosing 16-byte-aligned range (one extra double at the front or
// the back) and the element's data sit at slot offset `e & 1` (pU / pQ).
template <class C, int EPB, bool WQ>
struct BatchIO {
  static constexpr int ev(int x) { return (x + 1) / 2 * 2; }
  static constexpr bool ODDU = ((C::NPE * C::M) & 1) != 0;
  static constexpr bool ODDQ = WQ && ((C::NPE * C::MD) & 1) != 0;
  static constexpr int US = ev(C::NPE * C::M + (ODDU ? 1 : 0));            // slot stride per element
  static constexpr int QS = WQ ? ev(C::NPE * C::MD + (ODDQ ? 1 : 0)) : 0;
  static constexpr int U = EPB * US;
  static constexpr int Q = EPB * QS;
  static constexpr int MET = EPB * C::METP;
  static constexpr int CONN = ev(EPB * C::D * 2);  // int2 entries, 8 B each
  static constexpr int EID = ev((EPB + 1) / 2);    // int32 element ids
  static constexpr int NB = ev(EPB * C::LPE * 2 * C::M);
  static constexpr int NBQ = WQ ? ev(EPB * C::LPE * 2 * C::MD) : 0;
  static constexpr int BUF = U + Q + MET + CONN + EID + NB + NBQ;
  // 2 doubles hold the two mbarriers; after the buffers, a two-slot ring of
  // the connectivity one batch ahead of the bulk data (drives the gathers)
  static constexpr int SMEM = 2 + 2 * BUF + 2 * CONN;
  static constexpr long long bytes_per_elem() {
    return 8LL * (2 * (US + QS + C::METP + 2 * C::D + 1 + C::LPE * 2 * C::M + (WQ ? C::LPE * 2 * C::MD : 0)) +
                  4 * C::D);
  }
  uint64_t* bar;
  double* bufs;
  __device__ BatchIO(double* smem) : bar(reinterpret_cast<uint64_t*>(smem)), bufs(smem + 2) {}
  __device__ int2* cring(int bi) const { return reinterpret_cast<int2*>(bufs + 2 * BUF + bi * CONN); }
  __device__ double* bU(int bi) const { return bufs + bi * BUF; }
  __device__ double* bQ(int bi) const { return bufs + bi * BUF + U; }
  __device__ double* bMET(int bi) const { return bufs + bi * BUF + U + Q; }
  __device__ int2* bCONN(int bi) const { return reinterpret_cast<int2*>(bufs + bi * BUF + U + Q + MET); }
  __device__ int* eid(int bi) const { return reinterpret_cast<int*>(bufs + bi * BUF + U + Q + MET + CONN); }
  __device__ double* bNB(int bi) const { return bufs + bi * BUF + U + Q + MET + CONN + EID; }
  __device__ double* bNBQ(int bi) const { return bufs + bi * BUF + U + Q + MET + CONN + EID + NB; }
  // element le's nodal states / gradients in buffer bi
  __device__ const double* pU(int bi, int le) const {
    return bU(bi) + le * US + (ODDU ? (eid(bi)[le] & 1) : 0);
  }
  __device__ const double* pQ(int bi, int le) const {
    return bQ(bi) + le * QS + (ODDQ ? (eid(bi)[le] & 1) : 0);
  }
  __device__ void init(int tid) {
    if (tid == 0) {
      mbar_init(&bar[0], 1);
      mbar_init(&bar[1], 1);
      mbar_fence_init();
    }
  }
  // One element block of N doubles (global block index e of `base`) into the
  // slot at `dst`: returns the bytes the bulk copy will signal.  ODD blocks:
  // the enclosing aligned range of N + 1 doubles, except for the array's last
  // block at an even id (no double behind it): N - 1 doubles by bulk copy, the
  // last one by a plain load.
  template <bool ODD>
  __device__ unsigned load_block(double* dst, const double* base, size_t e, int N, int E, uint64_t* b,
                                 bool dry) const {
    const double* src = base + e * N;
    if (!ODD) {
      if (!dry) tma_load_1d(dst, src, N * 8, b);
      return N * 8;
    }
    const int par = static_cast<int>(e & 1);
    if (par == 0 && e + 1 == static_cast<size_t>(E)) {
      if (!dry) {
        tma_load_1d(dst, src, (N - 1) * 8, b);
        dst[N - 1] = __ldg(src + N - 1);
      }
      return (N - 1) * 8;
    }
    if (!dry) tma_load_1d(dst, src - par, (N + 1) * 8, b);
    return (N + 1) * 8;
  }
  // bulk loads of one batch into buffer bi (thread 0)
  __device__ void issue(const KParams<C>& kp, const double* Ug, const double* Qg, int batch, int bi) {
    constexpr int NPE = C::NPE, M = C::M, MD = C::MD, D = C::D;
    const int k0 = batch * EPB, nb = min(EPB, kp.E - k0);
    // element ids first: the bulk copies are asm volatile with a memory
    // clobber, so a load between them would wait out its full latency
    int ev_[EPB];
#pragma unroll
    for (int le = 0; le < EPB; ++le) ev_[le] = le < nb ? __ldg(kp.order + k0 + le) : 0;
    unsigned bytes = nb * C::METP * 8 + nb * D * 2 * 8;
#pragma unroll
    for (int le = 0; le < EPB; ++le) {
      if (le >= nb) break;
      const size_t e = static_cast<size_t>(ev_[le]);
      bytes += load_block<ODDU>(nullptr, Ug, e, NPE * M, kp.E, nullptr, true);
      if (WQ) bytes += load_block<ODDQ>(nullptr, Qg, e, NPE * MD, kp.E, nullptr, true);
    }
    mbar_expect_tx(&bar[bi], bytes);
#pragma unroll
    for (int le = 0; le < EPB; ++le) {
      if (le >= nb) break;
      const size_t e = static_cast<size_t>(ev_[le]);
      eid(bi)[le] = ev_[le];
      load_block<ODDU>(bU(bi) + le * US, Ug, e, NPE * M, kp.E, &bar[bi], false);
      if (WQ) load_block<ODDQ>(bQ(bi) + le * QS, Qg, e, NPE * MD, kp.E, &bar[bi], false);
    }
    tma_load_1d(bMET(bi), kp.metric + static_cast<size_t>(k0) * C::METP, nb * C::METP * 8, &bar[bi]);
    tma_load_1d(bCONN(bi), kp.conn + static_cast<size_t>(k0) * D * 2, nb * D * 2 * 8, &bar[bi]);
  }
  // neighbour traces of buffer bi (all threads; connectivity from its ring slot)
  __device__ void gather(const KParams<C>& kp, const double* Ug, const double* Qg, int batch, int bi, int tid,
                         int nthr) {
    constexpr int NPE = C::NPE, M = C::M, MD = C::MD, D = C::D, NL = C::NL, LPE = C::LPE, NP = C::NP;
    const int k0 = batch * EPB, nb = min(EPB, kp.E - k0);
    const int2* sc = cring(bi);
    for (int w = tid; w < nb * LPE * 2; w += nthr) {
      const int side = w & 1, lw = w >> 1, le = lw / LPE, rem = lw - le * LPE;
      const int dir = rem / NL, line = rem - dir * NL;
      const int2 cn = sc[(le * D + dir) * 2 + side];
      if (cn.x < 0) continue;
      const size_t nd = static_cast<size_t>(cn.x) * NPE + conn_node(cn.y, line, NP);
      double* dst = bNB(bi) + w * M;
      cp_async_run<M>(dst, Ug + nd * M);
      if (WQ && conn_sign(cn.y) > 0) {
        double* dq = bNBQ(bi) + w * MD;
        cp_async_run<MD>(dq, Qg + nd * MD);
      }
    }
  }
  // prologue: batches b0 and b0+G issued, their connectivity in the ring,
  // the traces of b0 in flight
  __device__ void start(const KParams<C>& kp, const double* Ug, const double* Qg, int b0, int G, int nbatch, int tid,
                        int nthr) {
    constexpr int D = C::D;
    if (tid == 0) {
      issue(kp, Ug, Qg, b0, 0);
      if (b0 + G < nbatch) issue(kp, Ug, Qg, b0 + G, 1);
    }
    for (int s = 0; s < 2; ++s) {
      const int b = b0 + s * G;
      if (b >= nbatch) break;
      const int k0 = b * EPB, nb = min(EPB, kp.E - k0);
      for (int i = tid; i < nb * D * 2; i += nthr) cring(s)[i] = __ldg(kp.conn + static_cast<size_t>(k0) * D * 2 + i);
    }
    __syncthreads();
    gather(kp, Ug, Qg, b0, 0, tid, nthr);
    cp_async_commit();
  }
  // head of iteration `it` (batch `batch`): its traces and bulk data are
  // resident on return; the gathers of the next batch (connectivity already
  // in the ring) and the connectivity two batches ahead are in flight behind
  // this batch's work
  __device__ void begin(const KParams<C>& kp, const double* Ug, const double* Qg, int batch, int it, int G,
                        int nbatch, int tid, int nthr) {
    constexpr int D = C::D;
    const int cur = it & 1, nxt = cur ^ 1;
    cp_async_wait_all();
    __syncthreads();
    mbar_wait(&bar[cur], (it >> 1) & 1);
    if (batch + G < nbatch) gather(kp, Ug, Qg, batch + G, nxt, tid, nthr);
    if (batch + 2 * G < nbatch) {
      const int k0 = (batch + 2 * G) * EPB, nb = min(EPB, kp.E - k0);
      for (int i = tid; i < nb * D * 2; i += nthr) cp_async8(cring(cur) + i, kp.conn + static_cast<size_t>(k0) * D * 2 + i);
    }
    cp_async_commit();
  }
  // epilogue of iteration `it`: free buffer `cur` and refill it two batches ahead
  __device__ void advance(const KParams<C>& kp, const double* Ug, const double* Qg, int batch, int it, int G,
                          int nbatch, int tid, int nthr) {
    const int cur = it & 1;
    __syncthreads();
    if (tid == 0 && batch + 2 * G < nbatch) issue(kp, Ug, Qg, batch + 2 * G, cur);
  }
};

template <class C, int EPB>
struct ResF {
  using IO = BatchIO<C, EPB, C::SECOND>;
  static constexpr int F = EPB * C::LPE * C::NQ * C::M;
  static constexpr int FH = EPB * C::LPE * 2 * C::M;
  static constexpr int TAB = IO::ev(2 * C::NP * C::NQ + 2 * C::NP);
  static constexpr int ACC = EPB * C::D * C::NPE * C::M;  // per-direction line projections
  static constexpr int TOTAL = IO::SMEM + F + FH + TAB + ACC;
  // one element per batch (the ring fills shared memory): as many warps as
  // the register file allows
static constexpr int LDG_RESF_THREADS1 = 512;
  static constexpr int THREADS = EPB == 1 ? LDG_RESF_THREADS1 : 256;
  static constexpr long long bytes_per_elem() {
    return IO::bytes_per_elem() + 8LL * (C::LPE * C::NQ * C::M + C::LPE * 2 * C::M + C::D * C::NPE * C::M);
  }
};
static constexpr int LDG_RESF_BUDGET_KB = 110;  // shared-memory budget per CTA of the flux-parallel residual / gradient measured (C3): 72 KB +40 us, 55 KB +96 us
template <class C>
struct ResFEpb {
  static constexpr long long per = ResF<C, 1>::bytes_per_elem();
  static constexpr int raw = static_cast<int>((LDG_RESF_BUDGET_KB * 1024LL) / per);
  static constexpr int value = raw < 1 ? 1 : (raw > 8 ? 8 : raw);
};

template <class C, int EPB>
__global__ void __launch_bounds__(ResF<C, EPB>::THREADS)
k_residual_f(const KParams<C> kp, const double* __restrict__ U, const double* __restrict__ Q,
             double* __restrict__ R) {
  constexpr int NP = C::NP, NQ = C::NQ, NPE = C::NPE, NL = C::NL, M = C::M, D = C::D, MD = C::MD,
                LPE = C::LPE, P = C::P;
  using RP = ResF<C, EPB>;
  extern __shared__ __align__(16) double smem[];
  typename RP::IO io(smem);
  double* const sF = smem + RP::IO::SMEM;
  double* const sFH = sF + RP::F;
  double* const sphi = sFH + RP::FH;     // phi[t][q]
  double* const sdq = sphi + NP * NQ;    // dq[i][q]
  double* const smi = sdq + NP * NQ;     // mi[i][side]
  double* const sacc = sphi + RP::TAB;   // acc[le][dir][node][c]
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int nbatch = (kp.E + EPB - 1) / EPB;
  const int G = gridDim.x;
  if (static_cast<int>(blockIdx.x) >= nbatch) return;
  io.init(tid);
  for (int i = tid; i < NP * NQ; i += nthr) {
    sphi[i] = (&kp.bt.phi[0][0])[i];
    sdq[i] = (&kp.bt.dq[0][0])[i];
  }
  for (int i = tid; i < 2 * NP; i += nthr) smi[i] = (&kp.bt.mi[0][0])[i];
  __syncthreads();
  io.start(kp, U, Q, blockIdx.x, G, nbatch, tid, nthr);
  for (int batch = blockIdx.x, it = 0; batch < nbatch; batch += G, ++it) {
    const int cur = it & 1;
    const int k0 = batch * EPB, nb = min(EPB, kp.E - k0);
    io.begin(kp, U, Q, batch, it, G, nbatch, tid, nthr);
    const int* sord = io.eid(cur);  // element ids of the batch (epilogue addresses)
    // ---- R2 (line ends) then R1 (quadrature points)
    // item space: the (heavier) line-end items padded to whole warps, then the
    // quadrature-point items; rounds alternate the thread order so the ragged
    // last round falls on the threads that had the lighter items
    const int n2 = nb * LPE * 2, n2p = (n2 + 31) / 32 * 32, n1 = nb * LPE * NQ;
    for (int base = 0, rnd = 0; base < n2p + n1; base += nthr, ++rnd) {
      const int w = base + ((rnd & 1) ? nthr - 1 - tid : tid);
      if (w >= n2p + n1 || (w >= n2 && w < n2p)) continue;
      bool ok = true;
      int le, dir, line;
      if (w < n2) {
        const int side = w & 1, lw = w >> 1;
        le = lw / LPE;
        const int rem = lw - le * LPE;
        dir = rem / NL;
        line = rem - dir * NL;
        const double* mk = io.bMET(cur) + le * C::METP;
        const double* sul = io.pU(cur, le);
        const double* sql = io.pQ(cur, le);
        const int2 cn = io.bCONN(cur)[(le * D + dir) * 2 + side];
        const int S = conn_sign(cn.y);
        const int nd = node_on_line<C>(dir, line, side ? P : 0);
        const double* nep = mk + C::MET_NV + ((dir * 2 + side) * NL + line) * D;
        double n[D], ui[M], uo[M], fh[M];
#pragma unroll
        for (int d = 0; d < D; ++d) n[d] = nep[d];
        const double* bcp = cn.x < 0 ? bnd_g(kp, -1 - cn.x, k0 + le, dir * 2 + side, line) : nullptr;
#pragma unroll
        for (int c = 0; c < M; ++c) {
          ui[c] = sul[nd * M + c];
          uo[c] = bcp ? __ldg(bcp + c) : io.bNB(cur)[w * M + c];
          fh[c] = 0.0;
        }
        if (bcp) {
          double nn = n[0] * n[0];
#pragma unroll
          for (int d = 1; d < D; ++d) nn += n[d] * n[d];
          nn = sqrt(nn);
          bnd_flux<C>(kp, -1 - cn.x, bcp, ui, (C::SECOND ? sql + nd * MD : sul), n, nn, fh, ok);
          } else {
              if (C::HAS_INV) {
              if (C::RI == LDG_ROE) roe_fn<D>(uo, ui, n, kp.pp.gamma, fh, ok);
              else llf_fn<D>(uo, ui, n, kp.pp.gamma, fh, ok);
            }
            if (C::SECOND) {
              double nn = n[0] * n[0];
#pragma unroll
              for (int d = 1; d < D; ++d) nn += n[d] * n[d];
              nn = sqrt(nn);
              double fv[M];
              if (S > 0) visc_fn<D, C::PH, double, double, double>(uo, io.bNBQ(cur) + w * MD, n, kp.pp, fv, ok);
              else visc_fn<D, C::PH, double, double, double>(ui, sql + nd * MD, n, kp.pp, fv, ok);
#pragma unroll
              for (int c = 0; c < M; ++c) fh[c] += fv[c];
              if (kp.pp.c11 != 0.0) {
#pragma unroll
                for (int c = 0; c < M; ++c) fh[c] += kp.pp.c11 * nn * (ui[c] - uo[c]);
              }
            }
          }
#pragma unroll
        for (int c = 0; c < M; ++c) sFH[w * M + c] = fh[c];
      } else {
        const int v = w - n2p, lw = v / NQ, q = v - lw * NQ;
        le = lw / LPE;
        const int rem = lw - le * LPE;
        dir = rem / NL;
        line = rem - dir * NL;
        const double* mk = io.bMET(cur) + le * C::METP;
        const double* sul = io.pU(cur, le);
        const double* sql = io.pQ(cur, le);
        double uq[M], qq[C::SECOND ? MD : 1];
#pragma unroll
        for (int c = 0; c < M; ++c) uq[c] = 0.0;
        if (C::SECOND) {
#pragma unroll
          for (int c = 0; c < MD; ++c) qq[c] = 0.0;
        }
#pragma unroll
        for (int t = 0; t < NP; ++t) {
          const int nd = node_on_line<C>(dir, line, t);
          const double ph = sphi[t * NQ + q];
#pragma unroll
          for (int c = 0; c < M; ++c) uq[c] += ph * sul[nd * M + c];
          if (C::SECOND) {
#pragma unroll
            for (int c = 0; c < MD; ++c) qq[c] += ph * sql[nd * MD + c];
          }
        }
        double nv[D];
#pragma unroll
        for (int d = 0; d < D; ++d) nv[d] = mk[((dir * NL + line) * NQ + q) * D + d];
        double f[M];
#pragma unroll
        for (int c = 0; c < M; ++c) f[c] = 0.0;
        if (C::HAS_INV) euler_fn<D>(uq, nv, kp.pp.gamma, f, ok);
        if (C::SECOND) {
          double fv[M];
          visc_fn<D, C::PH, double, double, double>(uq, qq, nv, kp.pp, fv, ok);
#pragma unroll
          for (int c = 0; c < M; ++c) f[c] += fv[c];
        }
#pragma unroll
        for (int c = 0; c < M; ++c) sF[v * M + c] = f[c];
      }
      if (!ok) report_line<C>(kp, kp.order[k0 + le], dir, line, io.pU(cur, le));
    }
    __syncthreads();
    // ---- R3a: one item per (element, line, component): the line's NP
    // projections r_i = sum_q dq[i][q] F_q + mi[i][0] Fh_0 + mi[i][1] Fh_1 from
    // NQ + 2 loads, the coefficients compile-time constant-bank operands
    for (int w = tid; w < nb * LPE * M; w += nthr) {
      const int lw = w / M, c = w - lw * M;
      const int l = lw / LPE, rem = lw - l * LPE, dir = rem / NL, ln = rem - dir * NL;
      const double* fq = sF + lw * NQ * M + c;
      double f[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) f[q] = fq[q * M];
      const double fh0 = sFH[(lw * 2 + 0) * M + c], fh1 = sFH[(lw * 2 + 1) * M + c];
      double* acc = sacc + (l * D + dir) * NPE * M + c;
#pragma unroll
      for (int i = 0; i < NP; ++i) {
        double r = 0.0;
#pragma unroll
        for (int q = 0; q < NQ; ++q) r += kp.bt.dq[i][q] * f[q];
        r += kp.bt.mi[i][0] * fh0;
        r += kp.bt.mi[i][1] * fh1;
        acc[node_on_line<C>(dir, ln, i) * M] = r;
      }
    }
    __syncthreads();
    // ---- R3b: dU/dt = S - (1/J) sum_dir r
    // (even element blocks: two entries per thread, one 16-byte store)
    constexpr int EW = (NPE * M) % 2 == 0 ? 2 : 1;
    for (int idx = tid * EW; idx < nb * NPE * M; idx += nthr * EW) {
      const int l = idx / (NPE * M), off = idx - l * NPE * M;
      const size_t e = static_cast<size_t>(sord[l]);
      double val[EW];
#pragma unroll
      for (int x = 0; x < EW; ++x) {
        const int nd = (off + x) / M;
        const double* a = sacc + l * D * NPE * M + off + x;
        double sum = a[0];
#pragma unroll
        for (int d = 1; d < D; ++d) sum = sum + a[d * NPE * M];
        const double invJ = io.bMET(cur)[l * C::METP + C::MET_NV + C::MET_NE + nd];
        const double src = kp.source ? __ldg(kp.source + e * (NPE * M) + off + x) : 0.0;
        val[x] = src - invJ * sum;
      }
      double* out = R + e * (NPE * M) + off;
      if (EW == 2) *reinterpret_cast<double2*>(out) = make_double2(val[0], val[EW - 1]);
      else out[0] = val[0];
    }
    io.advance(kp, U, Q, batch, it, G, nbatch, tid, nthr);
  }
}

// ======================================== gradient, persistent + TMA, flattened
// Q = (1/J) sum_dir M^-1 [u_hat (x) n |ends - sum_q w phi' u_q (x) nvec_q]
// (PAPER.md:520-573).  Items per batch: G1 one per (element, line, component
// c) interpolates u_c along the line and accumulates the line's contribution
//   g[i][d] = sum_q dq[i][q] u_q nvec_q[d] + sum_side mi[i][side] uh n_side[d]
// in registers (u_hat the switch-selected trace: own where S = +1, neighbour
// where S = -1, g_D on boundaries), written per direction to shared memory;
// G2 one per (element, node, c*D+d) sums the directions, scales by 1/J and
// stores coalesced.
template <class C, int EPB>
struct GradF {
  using IO = BatchIO<C, EPB, false>;
  static constexpr int ACC = EPB * C::D * C::NPE * C::MD;
  static constexpr int TAB = IO::ev(2 * C::NP * C::NQ + 2 * C::NP);
  static constexpr int TOTAL = IO::SMEM + ACC + TAB;
  static constexpr int THREADS = 256;
  static constexpr long long bytes_per_elem() { return IO::bytes_per_elem() + 8LL * C::D * C::NPE * C::MD; }
};
template <class C>
struct GradFEpb {
  static constexpr long long per = GradF<C, 1>::bytes_per_elem();
  static constexpr int raw = static_cast<int>((LDG_RESF_BUDGET_KB * 1024LL) / per);
  static constexpr int value = raw < 1 ? 1 : (raw > 8 ? 8 : raw);
};

template <class C, int EPB>
__global__ void __launch_bounds__(GradF<C, EPB>::THREADS)
k_gradient_f(const KParams<C> kp, const double* __restrict__ U, double* __restrict__ Qo) {
  constexpr int NP = C::NP, NQ = C::NQ, NPE = C::NPE, NL = C::NL, M = C::M, D = C::D, MD = C::MD,
                LPE = C::LPE, P = C::P;
  using GP = GradF<C, EPB>;
  extern __shared__ __align__(16) double smem[];
  typename GP::IO io(smem);
  double* const sacc = smem + GP::IO::SMEM;  // [EPB][D][NPE][MD]
  double* const sphi = sacc + GP::ACC;
  double* const sdq = sphi + NP * NQ;
  double* const smi = sdq + NP * NQ;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int nbatch = (kp.E + EPB - 1) / EPB;
  const int G = gridDim.x;
  if (static_cast<int>(blockIdx.x) >= nbatch) return;
  io.init(tid);
  for (int i = tid; i < NP * NQ; i += nthr) {
    sphi[i] = (&kp.bt.phi[0][0])[i];
    sdq[i] = (&kp.bt.dq[0][0])[i];
  }
  for (int i = tid; i < 2 * NP; i += nthr) smi[i] = (&kp.bt.mi[0][0])[i];
  __syncthreads();
  io.start(kp, U, nullptr, blockIdx.x, G, nbatch, tid, nthr);
  for (int batch = blockIdx.x, it = 0; batch < nbatch; batch += G, ++it) {
    const int cur = it & 1;
    const int k0 = batch * EPB, nb = min(EPB, kp.E - k0);
    io.begin(kp, U, nullptr, batch, it, G, nbatch, tid, nthr);
    const int* sord = io.eid(cur);  // element ids of the batch (epilogue addresses)
    // ---- G1: one (line, component) per item
    for (int v = tid; v < nb * LPE * M; v += nthr) {
      const int lw = v / M, c = v - lw * M;
      const int l = lw / LPE, rem = lw - l * LPE;
      const int dir = rem / NL, line = rem - dir * NL;
      const double* mk = io.bMET(cur) + l * C::METP;
      const double* sul = io.pU(cur, l);
      const double* nvl = mk + (dir * NL + line) * NQ * D;
      double ul[NP];
#pragma unroll
      for (int t = 0; t < NP; ++t) ul[t] = sul[node_on_line<C>(dir, line, t) * M + c];
      double g[NP][D];
#pragma unroll
      for (int i = 0; i < NP; ++i)
#pragma unroll
        for (int d = 0; d < D; ++d) g[i][d] = 0.0;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        double uq = 0.0;
#pragma unroll
        for (int t = 0; t < NP; ++t) uq += sphi[t * NQ + q] * ul[t];
        double w[D];
#pragma unroll
        for (int d = 0; d < D; ++d) w[d] = uq * nvl[q * D + d];
#pragma unroll
        for (int i = 0; i < NP; ++i) {
          const double dqi = sdq[i * NQ + q];
#pragma unroll
          for (int d = 0; d < D; ++d) g[i][d] += dqi * w[d];
        }
      }
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        const int2 cn = io.bCONN(cur)[(l * D + dir) * 2 + side];
        double uh;
        if (cn.x < 0)  // boundary: g_D, the interior trace, or mixed (no-slip wall)
          uh = bnd_uhat(kp, -1 - cn.x, bnd_g(kp, -1 - cn.x, k0 + l, dir * 2 + side, line), c, ul[side ? P : 0]);
        else if (conn_sign(cn.y) > 0)
          uh = ul[side ? P : 0];  // S = +1
        else uh = io.bNB(cur)[((lw << 1) | side) * M + c];
        const double* nep = mk + C::MET_NV + ((dir * 2 + side) * NL + line) * D;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const double w = uh * nep[d];
#pragma unroll
          for (int i = 0; i < NP; ++i) g[i][d] += smi[i * 2 + side] * w;
        }
      }
      double* acc = sacc + (l * D + dir) * NPE * MD + c * D;
#pragma unroll
      for (int t = 0; t < NP; ++t) {
        const int nd = node_on_line<C>(dir, line, t);
#pragma unroll
        for (int d = 0; d < D; ++d) acc[nd * MD + d] = g[t][d];
      }
    }
    __syncthreads();
    // ---- G2: Q = (1/J) sum_dir d^(dir)
    // (even element blocks: two entries per thread, one 16-byte store)
    constexpr int EW = (NPE * MD) % 2 == 0 ? 2 : 1;
    for (int idx = tid * EW; idx < nb * NPE * MD; idx += nthr * EW) {
      const int l = idx / (NPE * MD), off = idx - l * NPE * MD;
      double val[EW];
#pragma unroll
      for (int x = 0; x < EW; ++x) {
        const int nd = (off + x) / MD;
        const double* a = sacc + l * D * NPE * MD + off + x;
        double s = a[0];
#pragma unroll
        for (int d = 1; d < D; ++d) s = s + a[d * NPE * MD];
        val[x] = io.bMET(cur)[l * C::METP + C::MET_NV + C::MET_NE + nd] * s;
      }
      double* out = Qo + static_cast<size_t>(sord[l]) * (NPE * MD) + off;
      if (EW == 2) *reinterpret_cast<double2*>(out) = make_double2(val[0], val[EW - 1]);
      else out[0] = val[0];
    }
    io.advance(kp, U, nullptr, batch, it, G, nbatch, tid, nthr);
  }
}

// ===================================================================== Jacobian
// Lines intersecting tile `s` of an element.
//   2-D: all D*NL lines, all rows on them in the tile ("full").
//   3-D slab tiles (x2 = s): dir-0 and dir-1 lines of the slab (full) and every
//     dir-2 line (only its row at position s).
//   3-D line tiles (dir-0 line s = j + NP k): that dir-0 line (full), the
//     dir-1 lines (i, k) (row at position j) and dir-2 lines (i, j) (row k).
// prow(): position on the line of the tile's single row for non-full lines.
template <class C>
struct TileLines {
  // work unit: 0 = element (all D*NL lines, full), 1 = slab, 2 = dir-0 line of rows
  static constexpr int NLT = C::WU == 0 ? C::D * C::NL : (C::WU == 1 ? 2 * C::NP + C::NP * C::NP : 1 + 2 * C::NP);
  __device__ static __forceinline__ void get(int tl, int s, int& dir, int& line) {
    constexpr int NP = C::NP;
    if (C::WU == 0) {
      dir = tl / C::NL;
      line = tl - dir * C::NL;
    } else if (C::WU == 1) {
      if (tl < 2 * NP) {
        dir = tl / NP;
        line = (tl - dir * NP) + NP * s;
      } else {
        dir = 2;
        line = tl - 2 * NP;
      }
    } else {
      const int j = s % NP, k = s / NP;
      if (tl == 0) {
        dir = 0;
        line = s;
      } else if (tl <= NP) {
        dir = 1;
        line = (tl - 1) + NP * k;
      } else {
        dir = 2;
        line = (tl - 1 - NP) + NP * j;
      }
    }
  }
  __device__ static __forceinline__ bool full(int dir) {
    return C::WU == 0 || (C::WU == 1 ? dir < 2 : dir == 0);
  }
  __device__ static __forceinline__ int prow(int dir, int s) {
    if (C::WU == 1) return s;
    return dir == 1 ? s % C::NP : s / C::NP;
  }
  // Row items of a slab / line unit: the full lines come first (NFULL of
  // them, every row), then one row of each transverse line; rr -> (tl, i).
  static constexpr int NFULL = C::WU == 1 ? 2 * C::NP : 1;
  static constexpr int NROWS = NFULL * C::NP + (NLT - NFULL);
  __device__ static __forceinline__ void row_item(int rr, int s, int& tl, int& i) {
    if (rr < NFULL * C::NP) {
      tl = rr / C::NP;
      i = rr - tl * C::NP;
    } else {
      tl = NFULL + rr - NFULL * C::NP;
      int dir, line;
      get(tl, s, dir, line);
      i = prow(dir, s);
    }
  }
};

// Endpoint flux Jacobians of every element line end, into a per-element
// scratch consumed by k_jacobian:
//   SE[k][gs][Ein (m*m) | Eout (m*m) | Eq (m*mD, second-order)]
//   gs = (dir*2 + side)*NL + line  (the order of the metric's endpoint normals)
// Ein = dFhat/du_in, Eout = dFhat/du_out (Riemann + LDG viscous + C11 terms,
// each element with its own normal), Eq = dFhat_vis/dq of the switch-selected
// side.  One thread per (line end, pass); SEEDS components are seeded per
// thread in sequence (forward mode, Dual<1>), sharing the primal.
template <class C>
struct EndJac {
  static constexpr int NPASS = C::SECOND ? 3 : 2;
  static constexpr int EQS = C::SECOND ? C::M * C::MD : 0;
  static constexpr int SLOT = 2 * C::B11 + EQS;               // doubles per line end
  static constexpr int NLE = 2 * C::D * C::NL;                // line ends per element
  // Scratch block of one element, entry-major: SE[off * LS + le], le =
  // (dir*2 + side)*NL + line.  k_endjac lanes run over consecutive line ends
  // (coalesced stores); LS is odd where that keeps PER_ELEM even (16-byte
  // TMA rows) so shared-memory reads of neighbouring entries spread over banks.
  static constexpr int LS = SLOT % 2 == 0 ? (NLE | 1) : NLE + (NLE & 1);
  static constexpr int PER_ELEM = SLOT * LS;                  // doubles per element
  // k_endjac items per line end with `seeds` u-seeds per thread: the in and
  // out passes, plus one closed-form dF_vis/dq item (second order)
  static constexpr int items(int seeds) { return 2 * ((C::M + seeds - 1) / seeds) + (C::SECOND ? 1 : 0); }
};

// Effective scratch layout of a configuration (defined after the assembly
// kernels' shared-memory plans): entry-major (above) or, for the 3-D
// line-streaming assembly, group-major -- the line ends of one group of lines
// contiguous, so that k_jac_s3 fetches a group with one bulk copy.
template <class C>
struct SeLay;

// Line-end index functors for jac_tile: whole-element scratch block (k_endjac
// layout, persistent kernel) and tile-line staging (k_jacobian).
template <class C>
struct SeFull {
  static constexpr int LS = EndJac<C>::LS;
  __device__ __forceinline__ int operator()(int, int dir, int line, int side) const {
    return (dir * 2 + side) * C::NL + line;
  }
};
template <class C>
struct SeTile {
  static constexpr int LS = (2 * TileLines<C>::NLT) | 1;
  __device__ __forceinline__ int operator()(int tl, int, int, int side) const { return tl * 2 + side; }
};

static constexpr int LDG_EJ_MINB = 3;  // k_endjac min CTAs per SM (register cap 65536 / (128 * minb)) measured: C2 Jacobian 0.244 -> 0.239 ms, C3 -1.3 %, C4 neutral
// BND = false: the chunk's owned faces (flist = kp.owned, or every face of
// the chunk when null) except slip-wall / Neumann boundary ends; BND = true:
// exactly those ends (flist = their list), with the general boundary kinds.
template <class C, int SEEDS, bool BND>
__global__ void __launch_bounds__(128, LDG_EJ_MINB)
k_endjac(const KParams<C> kp, const double* __restrict__ U, const double* __restrict__ Q,
         double* __restrict__ SE, int k_begin, int k_end, long long o_begin, long long o_end,
         const int32_t* __restrict__ flist) {
  constexpr int NP = C::NP, NPE = C::NPE, NL = C::NL, M = C::M, D = C::D, MD = C::MD, P = C::P,
                B11 = C::B11;
  using EJ = EndJac<C>;
  constexpr int NSP = (M + SEEDS - 1) / SEEDS;         // u-seed groups per pass
  constexpr int IPS = EJ::items(SEEDS);                 // items per line end
  // Items: (face, pass item, line), lines fastest.  A face is an element's
  // local face ds = 2 dir + side; with face sharing (kp.owned) only the faces
  // this chunk owns are visited and the result is also written, negated with
  // in/out swapped, into the partner's line end: the numerical flux is
  // conservative, Fh(u_o, u_i, -n) = -Fh(u_i, u_o, n) (Riemann, LDG switch
  // (S flips across a face) and penalty terms alike).
  using SL = SeLay<C>;
  constexpr int LS = SL::ES;
  // unroll factor of the dual-number seed loop: rolled for the 3-D
  // second-order operators (instruction-cache bound: C5 Jacobian -1 ms;
  // neutral for C2)
  constexpr int EJ_SU = (C::D == 3 && C::SECOND) ? 1 : SEEDS;
  // GMW (group-major scratch, all seeds per item): one warp per (face, pass
  // item), lanes over the face's NL line ends; a lane's B11 entries go through
  // a per-warp shared-memory stage and leave as one contiguous run per line
  // end, written by consecutive lanes (flush).
  constexpr bool GMW = SL::GM && !BND && SEEDS >= M;
  static_assert(!GMW || (NL <= 32 && B11 <= 32 && EJ::EQS % B11 == 0), "k_endjac: warp-per-face mapping");
  __shared__ double stage_all[GMW ? (128 / 32) * 32 * B11 : 1];
  const int lane = threadIdx.x & 31;
  double* const stg = stage_all + (GMW ? (threadIdx.x >> 5) * 32 * B11 : 0);
  int line, sub;
  int64_t fi;
  bool act = true;
  if (GMW) {
    const int64_t wg = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (wg >= (o_end - o_begin) * IPS) return;  // the whole warp
    sub = static_cast<int>(wg % IPS);
    fi = wg / IPS;
    act = lane < NL;
    line = act ? lane : 0;  // spare lanes shadow line end 0 (their results are not flushed)
  } else {
    const int64_t item = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (item >= (o_end - o_begin) * NL * IPS) return;
    line = static_cast<int>(item % NL);
    const int64_t rest = item / NL;
    sub = static_cast<int>(rest % IPS);
    fi = rest / IPS;
  }
  const int fc = flist ? __ldg(flist + o_begin + fi) : static_cast<int>(k_begin * 2 * D + fi);
  const int k = fc / (2 * D), ds = fc - k * 2 * D, dir = ds >> 1, side = ds & 1;
  const int gs = ds * NL + line;
  const size_t e = kp.order[k];
  const double* mk = kp.metric + static_cast<size_t>(k) * C::METP;
  const int2 cn = __ldg(&kp.conn[(static_cast<size_t>(k) * D + dir) * 2 + side]);
  const bool bd = cn.x < 0;
  const int S = conn_sign(cn.y);
  const int nd = node_on_line<C>(dir, line, side ? P : 0);
  double* slot = SE + static_cast<size_t>(k - k_begin) * SL::PER_ELEM + SL::base(dir, side, line);  // entry o at slot[o * LS]
  // partner line end (same chunk only): pass 0 <-> pass 1, all entries negated
  double* pslot = nullptr;
  int2 fp = make_int2(-1, 0);
  if (kp.owned && !bd) fp = __ldg(&kp.fpart[static_cast<size_t>(k) * 2 * D + ds]);
  const bool part = fp.x >= k_begin && fp.x < k_end;  // (false without face sharing / on boundaries: fp.x = -1)
  int poff = 0;  // the partner line end's offset in its element's scratch block
  if (part) {
    int pl, ppos;
    line_of<C>(fp.y >> 1, conn_node(cn.y, line, NP), pl, ppos);
    poff = SL::base(fp.y >> 1, fp.y & 1, pl);
    pslot = SE + static_cast<size_t>(fp.x - k_begin) * SL::PER_ELEM + poff;
  }
  auto put = [&](int ps, int o, double v) {
    if (GMW) {
      stg[lane * B11 + o] = v;  // (passes 0 and 1; pass 2 stages its chunks itself)
      return;
    }
    slot[(ps * B11 + o) * LS] = v;
    if (pslot) pslot[((ps == 2 ? 2 : 1 - ps) * B11 + o) * LS] = -v;
  };
  // GMW: the warp's staged entries [lane][B11] -> entries off .. off + B11 of
  // pass ps of the face's NL line ends, and, negated with in/out swapped, of
  // the partner face's
  auto flush = [&](int ps, int off) {
    __syncwarp();
    const int ln = lane < B11 ? lane : 0;
    double* const own = SE + static_cast<size_t>(k - k_begin) * SL::PER_ELEM + ps * B11 + off + ln;
    double* const pel =
        part ? SE + static_cast<size_t>(fp.x - k_begin) * SL::PER_ELEM + (ps == 2 ? 2 : 1 - ps) * B11 + off + ln
             : nullptr;
#pragma unroll 5
    for (int it = 0; it < NL; ++it) {
      const int po = __shfl_sync(0xffffffffu, poff, it);
      const double v = stg[it * B11 + ln];
      if (lane < B11) {
        own[SL::base(dir, side, it)] = v;
        if (part) pel[po] = -v;
      }
    }
    __syncwarp();
  };
  int pass, g0;
  if (sub < NSP) {
    pass = 0;
    g0 = sub * SEEDS;
  } else if (sub < 2 * NSP) {
    pass = 1;
    g0 = (sub - NSP) * SEEDS;
  } else {
    pass = 2;
    g0 = (sub - 2 * NSP) * SEEDS;
  }
  double n[D];
#pragma unroll
  for (int d = 0; d < D; ++d) n[d] = __ldg(mk + C::MET_NV + (ds * NL + line) * D + d);
  double nn = n[0] * n[0];
#pragma unroll
  for (int d = 1; d < D; ++d) nn += n[d] * n[d];
  nn = sqrt(nn);
  const double* bcp = bd ? bnd_g(kp, -1 - cn.x, k, ds, line) : nullptr;
  const size_t own = e * NPE + nd;
  const size_t onb = bd ? 0 : static_cast<size_t>(cn.x) * NPE + conn_node(cn.y, line, NP);
  double uiv[M], uov[M];
  // boundary kind: Dirichlet / characteristic (ghost = g), slip wall (ghost =
  // mirrored u_in), Neumann (constant flux: no u dependence), see bnd_flux
  const int bkind = (BND && bd) ? __ldg(kp.bck + (-1 - cn.x)) : -1;
  const bool bneu = BND && bkind == BC_NEUMANN, bslip = BND && bkind == BC_SLIP_WALL,
             bnos = BND && bkind == BC_NO_SLIP;
#pragma unroll
  for (int c = 0; c < M; ++c) {
    uiv[c] = __ldg(U + own * M + c);
    if (!bd) uov[c] = __ldg(U + onb * M + c);
  }
  if (bd) bc_ghost<D, M>(bkind, bcp, uiv, n, uov);
  bool ok = true;
  using D1 = Dual<1>;
  if (pass < 2) {
    if (pass == 1 && bd) {
#pragma unroll
      for (int j = 0; j < SEEDS; ++j)
        if (g0 + j < M)
#pragma unroll
          for (int c = 0; c < M; ++c) slot[(B11 + c * M + g0 + j) * LS] = 0.0;  // boundary: no partner
      return;
    }
    double qiv[C::SECOND ? MD : 1], qov[C::SECOND ? MD : 1];
    if (C::SECOND) {
#pragma unroll
      for (int c = 0; c < MD; ++c) {
        qiv[c] = __ldg(Q + own * MD + c);
        qov[c] = bd ? 0.0 : __ldg(Q + onb * MD + c);
      }
    }
    // Closed-form parts (all seeds at once): the LLF inviscid Jacobian
    // (llf_jac) and, second order, the viscous flux of the switch-selected
    // side (visc_du) plus the C11 penalty; dual-number seeds carry the rest
    // (the Roe flux).
    constexpr bool LLFC = C::HAS_INV && C::RI != LDG_ROE && SEEDS >= M;
    constexpr bool VCF = C::SECOND && VISC_DU_CLOSED && SEEDS >= M;
    constexpr bool ALLC = (!C::HAS_INV || LLFC) && (!C::SECOND || VCF);
    double Jx[(LLFC || VCF) ? M * M : 1];
#pragma unroll
    for (int c = 0; c < ((LLFC || VCF) ? M * M : 1); ++c) Jx[c] = 0.0;
    if (LLFC) llf_jac<D>(uov, uiv, n, kp.pp.gamma, pass, Jx, ok);  // (LLFC: never a BND instantiation)
    if (VCF) {
      const bool sel_in = bd || S <= 0;  // the viscous flux is taken from u_in (else u_out)
      if ((pass == 0) == sel_in && !bneu) {
        double Jv[M * M];
        visc_du<D, C::PH>(sel_in ? uiv : uov, sel_in ? qiv : qov, n, kp.pp, Jv, ok);
#pragma unroll
        for (int c = 0; c < M * M; ++c) Jx[c] += Jv[c];
      }
      double pen = 0.0;
      if (bd) pen = (pass == 0 && !bneu && !bslip) ? (kp.pp.c11bd / (D == 2 ? nn : sqrt(nn))) * nn : 0.0;
      else if (kp.pp.c11 != 0.0) pen = pass == 0 ? kp.pp.c11 * nn : -(kp.pp.c11 * nn);
#pragma unroll
      for (int c = 0; c < M; ++c) Jx[c * M + c] += pen;
    }
static constexpr int LDG_EJ_DUALN = 0;  // all M seeds in one Dual<M> evaluation of the Riemann flux (first-order, not BND) measured slower: +18 us at 168 regs (spills), +6 us at 255
    constexpr bool DN = LDG_EJ_DUALN && !BND && !C::SECOND && C::HAS_INV && !LLFC && SEEDS == M;
    if (DN) {
      using DM = Dual<(DN ? M : 1)>;
      DM ui[M], uo[M], fh[M];
#pragma unroll
      for (int c = 0; c < M; ++c) {
        ui[c] = DM(uiv[c]);
        uo[c] = DM(uov[c]);
#pragma unroll
        for (int b = 0; b < (DN ? M : 1); ++b) {
          ui[c].d[b] = (pass == 0 && c == b) ? 1.0 : 0.0;
          uo[c].d[b] = (pass == 1 && c == b) ? 1.0 : 0.0;
        }
        fh[c] = DM(0.0);
      }
      if (C::RI == LDG_ROE) roe_fn<D>(uo, ui, n, kp.pp.gamma, fh, ok);
      else llf_fn<D>(uo, ui, n, kp.pp.gamma, fh, ok);
#pragma unroll
      for (int c = 0; c < M; ++c)
#pragma unroll
        for (int b = 0; b < (DN ? M : 1); ++b) put(pass, c * M + b, fh[c].d[b]);
    } else if (ALLC) {
#pragma unroll
      for (int c = 0; c < ((LLFC || VCF) ? M * M : 0); ++c) put(pass, c, Jx[c]);
    } else
#pragma unroll EJ_SU
    for (int j = 0; j < SEEDS; ++j) {
      const int b = (LLFC || VCF) ? j : g0 + j;
      if (b >= M) break;
      D1 ui[M], uo[M], fh[M];
#pragma unroll
      for (int c = 0; c < M; ++c) {
        ui[c] = D1(uiv[c]);
        uo[c] = D1(uov[c]);
        ui[c].d[0] = (pass == 0 && c == b) ? 1.0 : 0.0;
        uo[c].d[0] = (pass == 1 && c == b) ? 1.0 : 0.0;
        fh[c] = D1(0.0);
      }
      if (bslip || bnos) bc_ghost<D, M>(bkind, bcp, ui, n, uo);  // the ghost follows u_in (BND only)
      if (C::HAS_INV && !bneu) {
        if (C::RI == LDG_ROE) roe_fn<D>(uo, ui, n, kp.pp.gamma, fh, ok);
        else if (!LLFC) llf_fn<D>(uo, ui, n, kp.pp.gamma, fh, ok);
      }
      if (C::SECOND && !VCF) {
        D1 fv[M];
        if (bd) {
          if (bnos) {  // mixed wall: momentum penalty on m - 0, zero energy flux
            visc_fn<D, C::PH, D1, double, D1>(ui, qiv, n, kp.pp, fv, ok);
            const double c11 = kp.pp.c11bd / (D == 2 ? nn : sqrt(nn));
            fh[0] = fh[0] + fv[0];
#pragma unroll
            for (int c = 1; c < M - 1; ++c) fh[c] = fh[c] + fv[c] + (c11 * nn) * ui[c];
          } else if (!bneu) {
            visc_fn<D, C::PH, D1, double, D1>(ui, qiv, n, kp.pp, fv, ok);
            const double c11 = bslip ? 0.0 : kp.pp.c11bd / (D == 2 ? nn : sqrt(nn));
#pragma unroll
            for (int c = 0; c < M; ++c) fh[c] = fh[c] + fv[c] + (c11 * nn) * (ui[c] - __ldg(bcp + c));
          }
        } else {
          if (S > 0) visc_fn<D, C::PH, D1, double, D1>(uo, qov, n, kp.pp, fv, ok);
          else visc_fn<D, C::PH, D1, double, D1>(ui, qiv, n, kp.pp, fv, ok);
#pragma unroll
          for (int c = 0; c < M; ++c) fh[c] = fh[c] + fv[c];
          if (kp.pp.c11 != 0.0) {
#pragma unroll
            for (int c = 0; c < M; ++c) fh[c] = fh[c] + (kp.pp.c11 * nn) * (ui[c] - uo[c]);
          }
        }
      }
#pragma unroll
      for (int c = 0; c < M; ++c)
        put(pass, c * M + b, fh[c].d[0] + ((LLFC || VCF) ? Jx[(c * M + b) % ((LLFC || VCF) ? M * M : 1)] : 0.0));
    }
    if (GMW) flush(pass, 0);
  } else if (C::SECOND) {
    // dF_vis/dq of the switch-selected side, closed form (visc_dq)
    const bool out = !bd && S > 0;
    double usrc[M];
#pragma unroll
    for (int c = 0; c < M; ++c) usrc[c] = out ? uov[c] : uiv[c];
    double L[M * MD];
    visc_dq<D, C::PH>(usrc, n, kp.pp, L, ok);
    if (GMW) {
#pragma unroll
      for (int ch = 0; ch < (M * MD) / B11; ++ch) {
#pragma unroll
        for (int c = 0; c < B11; ++c)
          stg[lane * B11 + c] = (bneu || (bnos && (ch * B11 + c) / MD == M - 1)) ? 0.0 : L[ch * B11 + c];
        flush(2, ch * B11);
      }
    } else {
#pragma unroll
      for (int c = 0; c < M * MD; ++c) put(2, c, (bneu || (bnos && c / MD == M - 1)) ? 0.0 : L[c]);
    }
  }
  if (!ok && act) {
    // a non-physical state at this line end: report the offending nodal state
    double m2 = 0.0;
#pragma unroll
    for (int d = 0; d < D; ++d) m2 += uiv[1 + d] * uiv[1 + d];
    const bool own_bad =
        C::HAS_INV && (!(uiv[0] > 0.0) || !((kp.pp.gamma - 1.0) * (uiv[D + 1] - 0.5 * m2 / uiv[0]) > 0.0));
    double st[M];
#pragma unroll
    for (int c = 0; c < M; ++c) st[c] = (own_bad || bd) ? uiv[c] : uov[c];
    report_bad_state<double, M>(kp.err, own_bad || bd ? static_cast<int>(e) : cn.x,
                                own_bad || bd ? nd : conn_node(cn.y, line, NP), st);
  }
}

// K11 (+ K12 for second-order physics) of one row tile.  Store layout:
//   K11[((T*NS11 + slot)*B11 + a*M + b)*NT + r]       T = k*TPE + tile, r = row in tile
//   K12[((T*NS12 + slot)*B12 + a'*MD + b)*NT + r]     a' = stored row (NS: a-1)
// Jacobian CTA size (128 threads keeps 3 CTAs/SM within the register file).
// Jacobian store (block-contiguous line-structured BSR): row tiles of NT rows,
// blocks contiguous in row-major order:
//   K11[(((T*NS11 + slot)*m + a)*NT + r)*m + b]
//   K12[(((T*NS12 + slot)*R12 + a')*NT + r)*mD + b]      (NS: a' = a-1)
//   K21[((T*NS12 + slot)*NT + r)*D + d]                   (component-diagonal)
// i.e. per (slot, block row a) the rows of the tile are consecutive and each
// row's m entries contiguous.  The assembly writes straight from registers:
// one thread per (tile line, a, b) forms the line blocks of every row of its
// line, so each group of m lanes stores one full block row (32 B for m=4:
// whole sectors); an SpMV warp (32 rows of one block row a) reads one
// contiguous 1 KB run per slot.  The self (diagonal) block of a row collects the
// contributions of all D lines through it; the dir-0 thread adds the other
// directions' terms, so every entry is written exactly once (no atomics, no
// staging tile, no zero fill).
template <class C>
struct JacThreads {
  static constexpr bool big = C::D == 3 && C::WU == 0;  // 3-D element work unit: many lines
  static constexpr int rows = (C::NPE * C::M + 31) / 32 * 32;  // jac_k11_rows3 items
  // other work units: one phase-2 item (tile line, a, b) per thread when that
  // is 129..256 threads (no tail round behind the barrier), else 128
  static constexpr int p2 = (TileLines<C>::NLT * C::B11 + 31) / 32 * 32;
  // (measured: second-order tiles gain from it; the C2 Euler tile too since
  // the single-chunk endpoint scratch: 0.242 vs 0.252 ms at 160 vs 128 threads)
  static constexpr int small = p2 > 128 && p2 <= 256 ? p2 : 128;
  // 3-D slab / line work units (one CTA per unit, shared memory for one CTA
  // per SM): as many warps as the 128-register cap allows
  static constexpr bool unit3 = C::D == 3 && C::WU != 0;
  static constexpr int value = big ? (rows < 128 ? 128 : (rows > 640 ? 640 : rows)) : (unit3 ? 512 : small);
  static constexpr int min_blocks = big || unit3 ? 1 : (small > 128 ? 65536 / (small * 128) : 4);
};

template <class C>
struct JacSmem {
  static constexpr int NLT = TileLines<C>::NLT;
  static constexpr int U = C::NPE * C::M;
  static constexpr int Q = C::SECOND ? C::NPE * C::MD : 0;
  static constexpr int A = C::HAS_INV ? NLT * C::NQ * C::B11 : 0;  // dFinv/du . nvec at quad points
  static constexpr int AV = C::VIS_U ? NLT * C::NQ * C::B11 : 0;    // dFvis/du . nvec
  static constexpr int BQ = C::SECOND ? NLT * C::NQ * C::M * C::MD : 0;  // dFvis/dq . nvec
  static constexpr int SEC = ((2 * NLT) | 1) * EndJac<C>::SLOT;  // endpoint flux Jacobians (tile lines)
  static constexpr int TABD = (C::NP * C::NQ + 2 * C::NP + 1) / 2 * 2;  // cc diagonal + M^-1 columns
  // + full cc[i][t][q] + phi[t][q]: the assembly reads its basis coefficients
  // from shared memory (constant-bank operands are hoisted into registers by
  // the compiler and spill)
  static constexpr int NQ8 = (C::NQ + 1) / 2 * 2;
  static constexpr int CC8 = LDG_JAC_SMEMTAB == 2 ? C::NP * C::NP * NQ8 : 0;  // pair-padded cc (16-byte loads)
  static constexpr int TAB = TABD + (C::NP * C::NP * C::NQ + C::NP * C::NQ + 1) / 2 * 2 + CC8;
  static constexpr int ST11 = C::NS11 * C::B11 * C::NT;       // store doubles per tile
  static constexpr int ST12 = C::SECOND ? C::NS12 * C::B12 * C::NT : 0;
  static constexpr int WORK = A + AV + BQ + TAB;
  static constexpr int MET = (C::METP + 1) / 2 * 2;  // k_jacobian stages the element's metric
  static constexpr int TOTAL = U + Q + SEC + WORK + MET;
};

static constexpr int LDG_P2_UNROLL = 0;  // tuning knob: unroll of the phase-2 row loop (0 = full)
constexpr int P2_UNROLL_K = LDG_P2_UNROLL;
static constexpr int LDG_P2_ROWS = 0;  // tuning knob: 2-D phase 2 with one row per item (1) or one line per item (0); measured: per-line items are faster (C2 0.264 vs 0.297 ms)
constexpr bool P2_ROWS = LDG_P2_ROWS != 0;


template <class C>
__device__ __forceinline__ int tile_line_of(int dir, int line, int s) {
  constexpr int NP = C::NP;
  if (C::WU == 0) return dir * C::NL + line;
  if (C::WU == 1) return dir < 2 ? dir * NP + line % NP : 2 * NP + line;
  return dir == 0 ? 0 : (dir == 1 ? 1 + line % NP : 1 + NP + line % NP);
}

// 3-D element work unit, row-major K11 assembly: one thread per (slab s,
// row r, column b) forms column b of every K11 block of its row.  It walks the
// three lines through its node (dirs 2, 1, then 0), loading each line's
// flux-Jacobian column A[q][.][b] into registers once and reusing it for all
// NP blocks of that line; the self (diagonal) block accumulates in registers
// across the three lines and is stored with the dir-0 blocks.  For every
// slot the lanes of a warp run over consecutive (r, b), so each store
// instruction writes 256 contiguous bytes of one block row a.
template <class C, class EIdx>
__device__ __forceinline__ void jac_k11_rows3(const double* mk, const int2* scon, const double* sE, EIdx eidx,
                                              const double* sA, const double* sAv, const double* scc,
                                              const double* smi, double* __restrict__ K11e, const int tid,
                                              const int nthr) {
  constexpr int NP = C::NP, NQ = C::NQ, NL = C::NL, M = C::M, NT = C::NT, P = C::P, B11 = C::B11,
                TPE = C::TPE;
  using EJ = EndJac<C>;
  constexpr bool VOL11 = C::HAS_INV || C::VIS_U;
  constexpr int ST = JacSmem<C>::ST11;
  constexpr int RB = NT * M;  // (row, b) entries per (slab, slot, a)
  constexpr int LS = EIdx::LS;
  for (int w = tid; w < TPE * RB; w += nthr) {
    const int s = w / RB, rb = w - s * RB;
    const int r = rb / M, b = rb - r * M;
    const int x0 = r % NP, x1 = r / NP, x2 = s;
    const int nd = r + NT * s;
    const double sc = -mk[C::MET_NV + C::MET_NE + nd];
    double* out = K11e + static_cast<size_t>(s) * ST + rb;
    double vs[M];
#pragma unroll
    for (int a = 0; a < M; ++a) vs[a] = 0.0;
#pragma unroll
    for (int dd = 0; dd < 3; ++dd) {
      const int dir = 2 - dd;
      const int line = dir == 0 ? x1 + NP * x2 : (dir == 1 ? x0 + NP * x2 : x0 + NP * x1);
      const int i = dir == 0 ? x0 : (dir == 1 ? x1 : x2);
      const int tl = dir * NL + line;
      double av[VOL11 ? NQ : 1][M];
      if (VOL11) {
#pragma unroll
        for (int q = 0; q < NQ; ++q)
#pragma unroll
          for (int a = 0; a < M; ++a)
            av[q][a] = (C::HAS_INV ? sA[(tl * NQ + q) * B11 + a * M + b] : 0.0) +
                       (C::VIS_U ? sAv[(tl * NQ + q) * B11 + a * M + b] : 0.0);
      }
      const double* e0 = sE + eidx(tl, dir, line, 0);
      const double* e1 = sE + eidx(tl, dir, line, 1);
      const double mi0 = smi[i * 2 + 0], mi1 = smi[i * 2 + 1];
      // line block (i, t) column b
      auto blk = [&](const int t, double* v) {
#pragma unroll
        for (int a = 0; a < M; ++a) v[a] = 0.0;
        if (VOL11) {
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            const double cq = scc[(i * NP + t) * NQ + q];
#pragma unroll
            for (int a = 0; a < M; ++a) v[a] += cq * av[q][a];
          }
        }
        if (t == 0) {
#pragma unroll
          for (int a = 0; a < M; ++a) v[a] += mi0 * e0[(a * M + b) * LS];
        }
        if (t == P) {
#pragma unroll
          for (int a = 0; a < M; ++a) v[a] += mi1 * e1[(a * M + b) * LS];
        }
      };
      double v[M];
      if (dir != 0) {
        blk(i, v);
#pragma unroll
        for (int a = 0; a < M; ++a) vs[a] += v[a];
#pragma unroll
        for (int tp = 0; tp < P; ++tp) {
          blk(tp + (tp >= i ? 1 : 0), v);
          double* o = out + static_cast<size_t>(NP + (dir - 1) * P + tp) * B11 * NT;
#pragma unroll
          for (int a = 0; a < M; ++a) o[a * RB] = sc * v[a];
        }
      } else {
#pragma unroll
        for (int t = 0; t < NP; ++t) {
          blk(t, v);
          if (t == i) {
#pragma unroll
            for (int a = 0; a < M; ++a) v[a] += vs[a];
          }
          double* o = out + static_cast<size_t>(t) * B11 * NT;
#pragma unroll
          for (int a = 0; a < M; ++a) o[a * RB] = sc * v[a];
        }
      }
      // neighbour node-columns 2*dir + side
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        const bool nb = scon[dir * 2 + side].x >= 0;
        const double* eo = (side ? e1 : e0) + B11 * LS;
        const double mi = side ? mi1 : mi0;
        double* o = out + static_cast<size_t>(C::D * P + 1 + 2 * dir + side) * B11 * NT;
#pragma unroll
        for (int a = 0; a < M; ++a) o[a * RB] = nb ? sc * (mi * eo[(a * M + b) * LS]) : 0.0;
      }
    }
  }
}

// One Jacobian row tile.  su/sq element state and gradient, mk the element's
// metric (1/J included), sE the endpoint flux Jacobians of the tile lines
// indexed by eidx(tl, dir, line, side); stab = {cc[p][p][q], mi[p][s]}.
// PHS: bit 0 runs phase 1 (quadrature-point flux Jacobians into sA/sAv/sBq),
// bit 1 phases 2-3 (expansion and stores); 3 = both, with a barrier between.
template <class C, class EIdx, int PHS = 3>
__device__ __forceinline__ void jac_tile(const KParams<C>& kp, const int k, const int s, const size_t e,
                                         const double* su, const double* sq, const double* mk, const int2* scon,
                                         const double* sE, EIdx eidx, double* sA, double* sAv, double* sBq,
                                         const double* stab, double* __restrict__ K11t,
                                         double* __restrict__ K12t, const int tid, const int nthr) {
  constexpr int NP = C::NP, NQ = C::NQ, NL = C::NL, M = C::M, D = C::D, MD = C::MD, NT = C::NT, P = C::P,
                B11 = C::B11;
  using SM = JacSmem<C>;
  constexpr int NLT = SM::NLT, LS = EIdx::LS;
  // measured: second-order tiles (phase 3 follows, more live state) prefer
  // the rolled row loop, the Euler tile the unrolled one
  constexpr int P2_UNROLL = P2_UNROLL_K > 0 ? P2_UNROLL_K : (C::SECOND ? 1 : NP);
  const double* const tcc = stab + SM::TABD;                  // cc[i][t][q]
  const double* const tphi = tcc + NP * NP * NQ;               // phi[t][q]
  const double* const tmi = stab + NP * NQ;                    // mi[i][side]
  auto CC = [&](int i, int t, int q) { return JAC_SMEMTAB == 1 ? tcc[(i * NP + t) * NQ + q] : kp.bt.cc[i][t][q]; };
  // sum_q cc[i][t][q] f[q]: constant bank, or (JAC_SMEMTAB == 2) 16-byte
  // loads from the pair-padded shared table (f padded with zeros)
  constexpr int NQ8 = SM::NQ8;
  const double* const tcc8 = stab + SM::TAB - SM::CC8;
  auto ccdot = [&](int i, int t, const double* f) {
    double v = 0.0;
    if (JAC_SMEMTAB == 2) {
      const double2* c2 = reinterpret_cast<const double2*>(tcc8 + (i * NP + t) * NQ8);
#pragma unroll
      for (int h = 0; h < NQ8 / 2; ++h) {
        const double2 cv = c2[h];
        v += cv.x * f[2 * h];
        if (2 * h + 1 < NQ) v += cv.y * f[2 * h + 1];
      }
    } else if (JAC_CHAINS == 2) {
      // two independent partial sums (half the dependent DFMA chain)
      double v1 = 0.0;
#pragma unroll
      for (int q = 0; q < NQ; q += 2) v += CC(i, t, q) * f[q];
#pragma unroll
      for (int q = 1; q < NQ; q += 2) v1 += CC(i, t, q) * f[q];
      v += v1;
    } else {
#pragma unroll
      for (int q = 0; q < NQ; ++q) v += CC(i, t, q) * f[q];
    }
    return v;
  };
  auto MI = [&](int i, int sd) { return JAC_SMEMTAB ? tmi[i * 2 + sd] : kp.bt.mi[i][sd]; };
  auto PHI = [&](int t, int q) { return JAC_SMEMTAB ? tphi[t * NQ + q] : kp.bt.phi[t][q]; };
  // ---- phase 1a: inviscid A_q = d(F.nvec_q)/du at the quadrature points (closed form)
  constexpr bool VOL11 = C::HAS_INV || C::VIS_U;
  if ((PHS & 1) && C::HAS_INV) {
    for (int w = tid; w < NLT * NQ; w += nthr) {
      const int tl = w / NQ, q = w - tl * NQ;
      int dir, line;
      TileLines<C>::get(tl, s, dir, line);
      double nv[D], uq[M];
#pragma unroll
      for (int d = 0; d < D; ++d) nv[d] = mk[((dir * NL + line) * NQ + q) * D + d];
#pragma unroll
      for (int c = 0; c < M; ++c) uq[c] = 0.0;
#pragma unroll
      for (int t = 0; t < NP; ++t) {
        const int nd = node_on_line<C>(dir, line, t);
        const double ph = PHI(t, q);
#pragma unroll
        for (int c = 0; c < M; ++c) uq[c] += ph * su[nd * M + c];
      }
      bool ok = true;
      euler_jac_n<D>(uq, nv, kp.pp.gamma, sA + (tl * NQ + q) * B11, ok);
      if (!ok) report_line<C>(kp, static_cast<int>(e), dir, line, su);
    }
  }
  // ---- phase 1c (second-order): viscous flux derivatives at the quadrature
  // points: one item per u-seed (dual numbers) plus one closed-form dF/dq item
  if ((PHS & 1) && C::SECOND) {
    constexpr int NSU = C::VIS_U ? (VISC_DU_CLOSED ? 1 : M) : 0, NSEED = NSU + 1;
    for (int w = tid; w < NLT * NQ * NSEED; w += nthr) {
      const int sd = w % NSEED, tq = w / NSEED, tl = tq / NQ, q = tq - tl * NQ;
      int dir, line;
      TileLines<C>::get(tl, s, dir, line);
      double nv[D], uq[M], qq[MD];
#pragma unroll
      for (int d = 0; d < D; ++d) nv[d] = mk[((dir * NL + line) * NQ + q) * D + d];
#pragma unroll
      for (int c = 0; c < M; ++c) uq[c] = 0.0;
#pragma unroll
      for (int c = 0; c < MD; ++c) qq[c] = 0.0;
#pragma unroll
      for (int t = 0; t < NP; ++t) {
        const int nd = node_on_line<C>(dir, line, t);
        const double ph = PHI(t, q);
#pragma unroll
        for (int c = 0; c < M; ++c) uq[c] += ph * su[nd * M + c];
#pragma unroll
        for (int c = 0; c < MD; ++c) qq[c] += ph * sq[nd * MD + c];
      }
      bool ok = true;
      using D1 = Dual<1>;
      D1 fv[M];
      if (sd < NSU && VISC_DU_CLOSED) {
        double Jv[M * M];
        visc_du<D, C::PH>(uq, qq, nv, kp.pp, Jv, ok);
        double* a = sAv + (tl * NQ + q) * B11;
#pragma unroll
        for (int c = 0; c < M * M; ++c) a[c] = Jv[c];
      } else if (sd < NSU) {
        D1 du[M];
#pragma unroll
        for (int c = 0; c < M; ++c) {
          du[c] = D1(uq[c]);
          du[c].d[0] = c == sd ? 1.0 : 0.0;
        }
        visc_fn<D, C::PH, D1, double, D1>(du, qq, nv, kp.pp, fv, ok);
        double* a = sAv + (tl * NQ + q) * B11;
#pragma unroll
        for (int c = 0; c < M; ++c) a[c * M + sd] = fv[c].d[0];
      } else {
        double L[M * MD];
        visc_dq<D, C::PH>(uq, nv, kp.pp, L, ok);
        double* bqp = sBq + (tl * NQ + q) * M * MD;
#pragma unroll
        for (int c = 0; c < M * MD; ++c) bqp[c] = L[c];
      }
      if (!ok) report_line<C>(kp, static_cast<int>(e), dir, line, su);
    }
  }
  if (PHS == 3) __syncthreads();
  if (!(PHS & 2)) return;

  if (C::D == 3 && C::WU == 0)
    jac_k11_rows3<C>(mk, scon, sE, eidx, sA, sAv, stab + JacSmem<C>::TABD, stab + NP * NQ, K11t, tid, nthr);
  // ---- phase 2: K11 rows of every tile line, stored block row by block row
  const double* sccd = stab;            // cc[p][p][q]
  const double* smi = stab + NP * NQ;   // M^-1[p][0], M^-1[p][p]
  auto avq = [&](int tl, int q, int ab) {
    return (C::HAS_INV ? sA[(tl * NQ + q) * B11 + ab] : 0.0) + (C::VIS_U ? sAv[(tl * NQ + q) * B11 + ab] : 0.0);
  };
  // one (tile line, block entry ab): setup shared by the rows of the line,
  // then rows(body, full) runs body(i) for the rows this item owns
  auto line_item = [&](const int tl, const int ab, auto&& rows) {
    int dir, line;
    TileLines<C>::get(tl, s, dir, line);
    double av[NQ8];
#pragma unroll
    for (int q = 0; q < NQ8; ++q) av[q] = (VOL11 && q < NQ) ? avq(tl, q, ab) : 0.0;
    const double* e0 = sE + eidx(tl, dir, line, 0);
    const double* e1 = sE + eidx(tl, dir, line, 1);
    const double ein0 = e0[ab * LS], ein1 = e1[ab * LS];
    const double eo0 = e0[(B11 + ab) * LS], eo1 = e1[(B11 + ab) * LS];
    const int2 c0 = scon[dir * 2 + 0];
    const int2 c1 = scon[dir * 2 + 1];
    auto body = [&](const int i) {
      const int nd = node_on_line<C>(dir, line, i);
      const int r = nd % NT;
      const double sc = -mk[C::MET_NV + C::MET_NE + nd];
      double* rowp = K11t + static_cast<size_t>(nd / NT) * SM::ST11 + (static_cast<size_t>(ab / M) * NT + r) * M + ab % M;
#pragma unroll
      for (int t = 0; t < NP; ++t) {
        if (t == i && dir != 0) continue;  // the dir-0 thread owns the self block
        double v = VOL11 ? ccdot(i, t, av) : 0.0;
        if (t == 0) v += MI(i, 0) * ein0;
        if (t == P) v += MI(i, 1) * ein1;
        if (t == i) {
          // self block: add the lines of the other directions through this node
#pragma unroll
          for (int d2 = 1; d2 < D; ++d2) {
            int l2, p2;
            line_of<C>(d2, nd, l2, p2);
            const int tl2 = tile_line_of<C>(d2, l2, s);
            if (VOL11) {
#pragma unroll
              for (int q = 0; q < NQ; ++q) v += sccd[p2 * NQ + q] * avq(tl2, q, ab);
            }
            if (p2 == 0) v += smi[p2 * 2 + 0] * sE[eidx(tl2, d2, l2, 0) + ab * LS];
            if (p2 == P) v += smi[p2 * 2 + 1] * sE[eidx(tl2, d2, l2, 1) + ab * LS];
          }
        }
        rowp[static_cast<size_t>(inel_slot<C>(dir, i, t)) * NT * B11] = sc * v;
      }
      rowp[static_cast<size_t>(C::D * P + 1 + 2 * dir + 0) * NT * B11] = c0.x >= 0 ? sc * (MI(i, 0) * eo0) : 0.0;
      rowp[static_cast<size_t>(C::D * P + 1 + 2 * dir + 1) * NT * B11] = c1.x >= 0 ? sc * (MI(i, 1) * eo1) : 0.0;
    };
    rows(body, TileLines<C>::full(dir), dir);
  };
  if (C::D == 2 && P2_ROWS) {
    // 2-D (every line full): one item per (row position i, tile line, ab),
    // i outermost -- NP * NLT * B11 items balance over the CTA (the per-line
    // items leave a tail round), and i is warp-uniform when NLT * B11 is a
    // multiple of 32, so cc[i][t][q] stays a uniform constant-bank operand
    constexpr int NI = NLT * B11;
    for (int w = tid; w < NP * NI; w += nthr) {
      const int i = w / NI, rest = w - i * NI, tl = rest / B11, ab = rest - tl * B11;
      line_item(tl, ab, [&](auto& body, bool, int) { body(i); });
    }
  } else if (C::D == 3 && C::WU != 0) {
    // slab / line units: one row per item (the full lines' items would carry
    // NP rows against one for the transverse lines')
    using TL = TileLines<C>;
    for (int w = tid; w < TL::NROWS * B11; w += nthr) {
      const int rr = w / B11, ab = w - rr * B11;
      int tl, i;
      TL::row_item(rr, s, tl, i);
      line_item(tl, ab, [&](auto& body, bool, int) { body(i); });
    }
  } else {
    for (int w = (C::D == 3 && C::WU == 0) ? NLT * B11 : tid; w < NLT * B11; w += nthr) {
      const int tl = w / B11, ab = w - tl * B11;
      line_item(tl, ab, [&](auto& body, bool full, int dir) {
        if (full) {
#pragma unroll P2_UNROLL
          for (int i = 0; i < NP; ++i) body(i);
        } else {
          body(TileLines<C>::prow(dir, s));
        }
      });
    }
  }
  if (!C::SECOND) return;

  // ---- phase 3: K12 = dR/dQ (stored rows a' of each block)
  constexpr int B12 = C::B12, A0 = C::PH == PH_NS ? 1 : 0;
  auto k12_item = [&](const int tl, const int ab, auto&& rows) {
    const int a = ab / MD + A0, b = ab % MD;
    int dir, line;
    TileLines<C>::get(tl, s, dir, line);
    const bool full = TileLines<C>::full(dir);
    double bv[NQ8];
#pragma unroll
    for (int q = 0; q < NQ8; ++q) bv[q] = q < NQ ? sBq[(tl * NQ + q) * M * MD + a * MD + b] : 0.0;
    const double eq0 = sE[eidx(tl, dir, line, 0) + (2 * B11 + a * MD + b) * LS];
    const double eq1 = sE[eidx(tl, dir, line, 1) + (2 * B11 + a * MD + b) * LS];
    const int2 c0 = scon[dir * 2 + 0];
    const int2 c1 = scon[dir * 2 + 1];
    // own-end dependence when boundary or S <= 0; neighbour slot otherwise
    const bool own0 = c0.x < 0 || conn_sign(c0.y) <= 0;
    const bool own1 = c1.x < 0 || conn_sign(c1.y) <= 0;
    auto body = [&](const int i) {
      const int nd = node_on_line<C>(dir, line, i);
      const int r = nd % NT;
      const double sc = -mk[C::MET_NV + C::MET_NE + nd];
      double* rowp = K12t + static_cast<size_t>(nd / NT) * SM::ST12 + (static_cast<size_t>(ab / MD) * NT + r) * MD + ab % MD;
#pragma unroll
      for (int t = 0; t < NP; ++t) {
        if (t == i && dir != 0) continue;
        double v = ccdot(i, t, bv);
        if (t == 0 && own0) v += MI(i, 0) * eq0;
        if (t == P && own1) v += MI(i, 1) * eq1;
        if (t == i) {
#pragma unroll
          for (int d2 = 1; d2 < D; ++d2) {
            int l2, p2;
            line_of<C>(d2, nd, l2, p2);
            const int tl2 = tile_line_of<C>(d2, l2, s);
#pragma unroll
            for (int q = 0; q < NQ; ++q) v += sccd[p2 * NQ + q] * sBq[(tl2 * NQ + q) * M * MD + a * MD + b];
            if (p2 == 0 || p2 == P) {
              const int sd2 = p2 == 0 ? 0 : 1;
              const int2 cx = scon[d2 * 2 + sd2];
              if (cx.x < 0 || conn_sign(cx.y) <= 0)
                v += smi[p2 * 2 + sd2] * sE[eidx(tl2, d2, l2, sd2) + (2 * B11 + a * MD + b) * LS];
            }
          }
        }
        rowp[static_cast<size_t>(inel_slot<C>(dir, i, t)) * NT * B12] = sc * v;
      }
      double nbv = 0.0;
      if (!own0) nbv = sc * (MI(i, 0) * eq0);
      if (!own1) nbv = sc * (MI(i, 1) * eq1);
      rowp[static_cast<size_t>(C::D * P + 1 + dir) * NT * B12] = nbv;
    };
    rows(body, full, dir);
  };
  if (C::D == 3 && C::WU != 0) {
    using TL = TileLines<C>;
    for (int w = tid; w < TL::NROWS * B12; w += nthr) {
      const int rr = w / B12, ab = w - rr * B12;
      int tl, i;
      TL::row_item(rr, s, tl, i);
      k12_item(tl, ab, [&](auto& body, bool, int) { body(i); });
    }
  } else {
    for (int w = tid; w < NLT * B12; w += nthr) {
      const int tl = w / B12, ab = w - tl * B12;
      k12_item(tl, ab, [&](auto& body, bool full, int dir) {
        if (full) {
#pragma unroll
          for (int i = 0; i < NP; ++i) body(i);
        } else {
          body(TileLines<C>::prow(dir, s));
        }
      });
    }
  }
}

template <class C>
__device__ __forceinline__ void fill_tab(const KParams<C>& kp, double* stab, int tid, int nthr) {
  constexpr int NP = C::NP, NQ = C::NQ;
  for (int i = tid; i < NP * NQ; i += nthr) {
    const int p = i / NQ, q = i - p * NQ;
    stab[i] = kp.bt.cc[p][p][q];
  }
  for (int i = tid; i < 2 * NP; i += nthr) stab[NP * NQ + i] = (&kp.bt.mi[0][0])[i];
  for (int i = tid; i < NP * NP * NQ; i += nthr) stab[JacSmem<C>::TABD + i] = (&kp.bt.cc[0][0][0])[i];
  for (int i = tid; i < NP * NQ; i += nthr) stab[JacSmem<C>::TABD + NP * NP * NQ + i] = (&kp.bt.phi[0][0])[i];
  if (JacSmem<C>::CC8) {
    constexpr int NQ8 = JacSmem<C>::NQ8;
    double* cc8 = stab + JacSmem<C>::TAB - JacSmem<C>::CC8;
    for (int x = tid; x < NP * NP * NQ8; x += nthr) {
      const int it = x / NQ8, q = x - it * NQ8;
      cc8[x] = q < NQ ? (&kp.bt.cc[0][0][0])[it * NQ + q] : 0.0;
    }
  }
}

template <class C>
__global__ void __launch_bounds__(JacThreads<C>::value, JacThreads<C>::min_blocks)
k_jacobian(const KParams<C> kp, const double* __restrict__ U, const double* __restrict__ Q,
           const double* __restrict__ SE, double* __restrict__ K11, double* __restrict__ K12, int k_begin) {
  constexpr int NPE = C::NPE, NL = C::NL, M = C::M, MD = C::MD;
  using SM = JacSmem<C>;
  using EJ = EndJac<C>;
  constexpr int NLT = SM::NLT;
  extern __shared__ __align__(16) double smem[];
  double* su = smem;
  double* sq = su + SM::U;
  double* sE = sq + SM::Q;
  double* sA = sE + SM::SEC;
  double* sAv = sA + SM::A;
  double* sBq = sAv + SM::AV;
  double* stab = sBq + SM::BQ;
  double* smet = stab + SM::TAB;
  const int W = blockIdx.x + k_begin * C::UPE;  // work unit id
  const int k = W / C::UPE, s = W - k * C::UPE;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const size_t e = kp.order[k];
  const double* mk = smet;
  // element state (+ gradient), metric, endpoint flux Jacobians of the
  // tile's line ends (k_endjac scratch of this chunk) in tile-line order:
  // all as asynchronous 8-byte copies, so their latencies overlap
  {
    const double* ug = U + e * (NPE * M);
    for (int i = tid; i < NPE * M; i += nthr) cp_async8(su + i, ug + i);
    if (C::SECOND) {
      const double* qg = Q + e * (NPE * MD);
      for (int i = tid; i < NPE * MD; i += nthr) cp_async8(sq + i, qg + i);
    }
    const double* mg = kp.metric + static_cast<size_t>(k) * C::METP;
    for (int i = tid; i < C::METP; i += nthr) cp_async8(smet + i, mg + i);
    const double* se = SE + static_cast<size_t>(k - k_begin) * EJ::PER_ELEM;
    for (int w = tid; w < NLT * 2 * EJ::SLOT; w += nthr) {
      const int o = w / (2 * NLT), idx = w - o * (2 * NLT);
      const int tl = idx >> 1, side = idx & 1;
      int dir, line;
      TileLines<C>::get(tl, s, dir, line);
      cp_async8(sE + o * SeTile<C>::LS + idx, se + o * EJ::LS + (dir * 2 + side) * NL + line);
    }
    cp_async_commit();
  }
  fill_tab<C>(kp, stab, tid, nthr);
  cp_async_wait_all();
  __shared__ int2 sconn[2 * C::D];
  if (tid < 2 * C::D) sconn[tid] = __ldg(&kp.conn[static_cast<size_t>(k) * C::D * 2 + tid]);
  __syncthreads();
  jac_tile<C>(kp, k, s, e, su, sq, mk, sconn, sE, SeTile<C>(), sA, sAv, sBq, stab,
              K11 + static_cast<size_t>(k) * C::TPE * SM::ST11,
              C::SECOND ? K12 + static_cast<size_t>(k) * C::TPE * SM::ST12 : nullptr, tid, nthr);
}

// Fused endpoint phase (JacP::FE): gather the neighbour traces of the
// element's line ends (cp.async), then one item per (line end, pass) forms
// the closed-form LLF endpoint Jacobian dFh/du_in (pass 0) or dFh/du_out
// (pass 1) straight into the shared endpoint block in the k_endjac scratch
// layout (entry-major, stride LS).  Boundary ends (Dirichlet-type only: the
// host enables the fused path when no slip / Neumann / no-slip wall exists):
// ghost = the boundary data, no out-block.
template <class C>
__device__ __forceinline__ void endpoint_gather(const double* __restrict__ U, const int2* sc, double* snb, int tid,
                                                int nthr) {
  constexpr int D = C::D, NL = C::NL, M = C::M, NP = C::NP, NPE = C::NPE;
  for (int w = tid; w < 2 * D * NL; w += nthr) {
    const int ds = w / NL, line = w - ds * NL;
    const int2 cn = sc[ds];
    if (cn.x < 0) continue;
    const size_t nd = static_cast<size_t>(cn.x) * NPE + conn_node(cn.y, line, NP);
#pragma unroll
    for (int c = 0; c < M; ++c) cp_async8(snb + w * M + c, U + nd * M + c);
  }
  cp_async_commit();
}
// (the traces of this element were gathered by endpoint_gather one element
// ahead; wait for them, then form the blocks)
template <class C>
__device__ __forceinline__ void endpoint_phase(const KParams<C>& kp, int k, const double* su, const double* mk,
                                               const int2* sc, double* sE, const double* snb,
                                               const double* __restrict__ SEg, int tid, int nthr) {
  constexpr int D = C::D, NL = C::NL, M = C::M, NP = C::NP, P = C::P, B11 = C::B11;
  constexpr int NLE = 2 * D * NL, LS = EndJac<C>::LS;
  cp_async_wait_all();
  __syncthreads();
  for (int w = tid; w < 2 * NLE; w += nthr) {
    const int pass = w / NLE, le = w - pass * NLE;
    const int ds = le / NL, line = le - ds * NL, dir = ds >> 1, side = ds & 1;
    const int2 cn = sc[ds];
    const bool bd = cn.x < 0;
    double J[M * M];
    if (bd) {
      const int kind = __ldg(kp.bck + (-1 - cn.x));
      if (kind == BC_SLIP_WALL || kind == BC_NEUMANN || kind == BC_NO_SLIP) {
        // general boundary kinds: blocks from k_endjac<..., BND> (global scratch of the chunk)
#pragma unroll
        for (int o = 0; o < M * M; ++o) sE[(pass * B11 + o) * LS + le] = __ldg(SEg + (pass * B11 + o) * LS + le);
        continue;
      }
    }
    if (bd && pass == 1) {
#pragma unroll
      for (int o = 0; o < M * M; ++o) sE[(B11 + o) * LS + le] = 0.0;
      continue;
    }
    const int nd = node_on_line<C>(dir, line, side ? P : 0);
    double n[D], ui[M], uo[M];
#pragma unroll
    for (int d = 0; d < D; ++d) n[d] = mk[C::MET_NV + (ds * NL + line) * D + d];
    const double* g = bd ? bnd_g(kp, -1 - cn.x, k, ds, line) : nullptr;
#pragma unroll
    for (int c = 0; c < M; ++c) {
      ui[c] = su[nd * M + c];
      uo[c] = bd ? __ldg(g + c) : snb[le * M + c];
    }
    bool ok = true;
    llf_jac<D>(uo, ui, n, kp.pp.gamma, pass, J, ok);
#pragma unroll
    for (int o = 0; o < M * M; ++o) sE[(pass * B11 + o) * LS + le] = J[o];
    if (!ok) {
      double m2 = 0.0;
#pragma unroll
      for (int d = 0; d < D; ++d) m2 += ui[1 + d] * ui[1 + d];
      const bool own_bad = !(ui[0] > 0.0) || !((kp.pp.gamma - 1.0) * (ui[D + 1] - 0.5 * m2 / ui[0]) > 0.0);
      report_bad_state<double, M>(kp.err, own_bad || bd ? static_cast<int>(kp.order[k]) : cn.x,
                                  own_bad || bd ? nd : conn_node(cn.y, line, NP), own_bad || bd ? ui : uo);
    }
  }
  __syncthreads();
}

// Persistent, TMA-prefetching Jacobian assembly (2-D: one tile = one element):
// two input buffers {U, Q, metric, endpoint-Jacobian scratch} of consecutive
// elements; the next element's inputs land while the current one assembles.
template <class C>
struct JacP {
  static constexpr int ev(int x) { return (x + 1) / 2 * 2; }
  static constexpr int U = ev(C::NPE * C::M);
  static constexpr int Q = C::SECOND ? ev(C::NPE * C::MD) : 0;
  static constexpr int MET = C::METP;
  static constexpr int CONN = ev(2 * C::D);  // int2 entries (8 B each)
  static constexpr int SE = ev(EndJac<C>::PER_ELEM);
  // fused endpoint phase (3-D element units, first order, LLF: closed-form
  // endpoint Jacobians computed in the assembly from gathered neighbour
  // traces; no k_endjac launch and no scratch round trip through HBM)
  static constexpr bool FE = C::D == 3 && C::WU == 0 && !C::SECOND && C::HAS_INV &&
                             C::RI != LDG_ROE;
  static constexpr int NBV = FE ? ev(2 * C::D * C::NL * C::M) : 0;  // neighbour traces per line end
  // fused: the endpoint block is computed per element (one copy outside the
  // ring), only the neighbour traces ride the ring
  static constexpr int SER = FE ? 0 : SE;   // endpoint block per ring buffer
  static constexpr int SE1 = FE ? SE : 0;   // single endpoint block (fused)
  static constexpr int BUF = U + Q + MET + CONN + SER + NBV;
  using SM = JacSmem<C>;
  // 2-D: the element's K11 tile is formed in shared memory and leaves with one
  // TMA bulk store (sequential write stream, no per-entry global stores;
  // measured: a small gain for the Euler tile, a loss for second-order tiles
  // whose larger footprint costs occupancy)
  // (rejected after measurement: a 2-D software pipeline of phases 2-3 of
  // element k with phase 1 of element k+1 -- C2 0.267 vs 0.265 ms, a loss for
  // C3 through occupancy; a 3-deep ring for every configuration -- C2 -0.9 us)
  static constexpr bool STAGE = C::D == 2 && !C::SECOND && (SM::ST11 % 2 == 0) &&
                                8LL * SM::ST11 <= 64 * 1024;
  static constexpr int STG = STAGE ? SM::ST11 : 0;
  static constexpr long long bytes(int nb) { return 8LL * (4 + nb * BUF + SM::WORK + STG + SE1); }
  // prefetch ring depth: 3 for the one-CTA-per-SM 3-D element units (when it
  // fits), 2 where several CTAs share an SM
  static constexpr int NBUF = (JacThreads<C>::big && bytes(3) <= 200 * 1024) ? 3 : 2;
  static constexpr int TOTAL = 4 + NBUF * BUF + SM::WORK + STG + SE1;  // 4 doubles hold up to 3 mbarriers
  static constexpr bool OK = C::WU == 0 && (C::NPE * C::M) % 2 == 0 && (!C::SECOND || (C::NPE * C::MD) % 2 == 0) &&
                             (EndJac<C>::PER_ELEM % 2 == 0) && bytes(2) <= 200 * 1024;
};

template <class C>
__global__ void __launch_bounds__(JacThreads<C>::value, JacThreads<C>::min_blocks)
k_jacobian_p(const KParams<C> kp, const double* __restrict__ U, const double* __restrict__ Q,
             const double* __restrict__ SE, double* __restrict__ K11, double* __restrict__ K12, int k_begin,
             int k_end) {
  constexpr int NPE = C::NPE, NL = C::NL, M = C::M, MD = C::MD, NB = JacP<C>::NBUF;
  using JP = JacP<C>;
  using SM = JacSmem<C>;
  using EJ = EndJac<C>;
  extern __shared__ __align__(16) double smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  double* const bufs = smem + 4;
  double* const work = bufs + NB * JP::BUF;
  double* sA = work;
  double* sAv = sA + SM::A;
  double* sBq = sAv + SM::AV;
  double* stab = sBq + SM::BQ;
  double* sstage = work + SM::WORK;  // K11 tile staging (JP::STAGE)
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int G = gridDim.x;
  if (k_begin + static_cast<int>(blockIdx.x) >= k_end) return;
  auto bU = [&](int bi) { return bufs + bi * JP::BUF; };
  auto bQ = [&](int bi) { return bufs + bi * JP::BUF + JP::U; };
  auto bMET = [&](int bi) { return bufs + bi * JP::BUF + JP::U + JP::Q; };
  auto bCONN = [&](int bi) { return reinterpret_cast<int2*>(bufs + bi * JP::BUF + JP::U + JP::Q + JP::MET); };
  double* const se1 = work + SM::WORK + JP::STG;  // fused: the element's endpoint block
  auto bSE = [&](int bi) {
    return JP::FE ? se1 : bufs + bi * JP::BUF + JP::U + JP::Q + JP::MET + JP::CONN;
  };
  auto bNBV = [&](int bi) { return bufs + bi * JP::BUF + JP::U + JP::Q + JP::MET + JP::CONN + JP::SER; };
  constexpr bool fe = JP::FE;
  if (tid == 0) {
    for (int b = 0; b < NB; ++b) mbar_init(&bar[b], 1);
    mbar_fence_init();
  }
  fill_tab<C>(kp, stab, tid, nthr);
  __syncthreads();
  auto issue = [&](int k, int bi) {
    const size_t e = __ldg(kp.order + k);
    unsigned bytes = NPE * M * 8 + C::METP * 8 + 2 * C::D * 8 + (fe ? 0 : EJ::PER_ELEM * 8);
    if (C::SECOND) bytes += NPE * MD * 8;
    mbar_expect_tx(&bar[bi], bytes);
    tma_load_1d(bU(bi), U + e * (NPE * M), NPE * M * 8, &bar[bi]);
    if (C::SECOND) tma_load_1d(bQ(bi), Q + e * (NPE * MD), NPE * MD * 8, &bar[bi]);
    tma_load_1d(bMET(bi), kp.metric + static_cast<size_t>(k) * C::METP, C::METP * 8, &bar[bi]);
    tma_load_1d(bCONN(bi), kp.conn + static_cast<size_t>(k) * C::D * 2, 2 * C::D * 8, &bar[bi]);
    // (fused: the endpoint Jacobians are computed in the element loop; an L2
    // evict-first read of the scratch measured no gain: C2 +0.7 us, C3 +8 us)
    if (!fe)
      tma_load_1d(bSE(bi), SE + static_cast<size_t>(k - k_begin) * EJ::PER_ELEM, EJ::PER_ELEM * 8, &bar[bi]);
  };
  const int k0 = k_begin + blockIdx.x;
  if (tid == 0)
    for (int b = 0; b < NB; ++b)
      if (k0 + b * G < k_end) issue(k0 + b * G, b);
  for (int k = k0, it = 0; k < k_end; k += G, ++it) {
    const int cur = it % NB;
    mbar_wait(&bar[cur], (it / NB) & 1);
    if (JP::FE && fe) {
      if (it == 0) endpoint_gather<C>(U, bCONN(cur), bNBV(cur), tid, nthr);
      endpoint_phase<C>(kp, k, bU(cur), bMET(cur), bCONN(cur), bSE(cur), bNBV(cur),
                        SE + static_cast<size_t>(k - k_begin) * EJ::PER_ELEM, tid, nthr);
      // prefetch: the next element's neighbour traces land during this assembly
      if (k + G < k_end) {
        const int nx = (it + 1) % NB;
        mbar_wait(&bar[nx], ((it + 1) / NB) & 1);
        endpoint_gather<C>(U, bCONN(nx), bNBV(nx), tid, nthr);
      }
    }
    // staging free again: the previous tile's bulk store has read it (waited
    // here by its issuer; jac_tile's barrier before phase 2 publishes it)
    if (JP::STAGE && tid == 0 && it > 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    const size_t e = kp.order[k];
    double* const K11g = K11 + static_cast<size_t>(k) * C::TPE * SM::ST11;
    jac_tile<C>(kp, k, 0, e, bU(cur), bQ(cur), bMET(cur), bCONN(cur), bSE(cur), SeFull<C>(), sA, sAv, sBq, stab,
                JP::STAGE ? sstage : K11g,
                C::SECOND ? K12 + static_cast<size_t>(k) * C::TPE * SM::ST12 : nullptr, tid, nthr);
    if (JP::STAGE) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();  // all reads of buffer `cur` (and of sA/sAv/sBq) done; tile staged
    if (JP::STAGE && tid == 0) {
      // tile store with an L2 evict-last policy (measured C2: 0.3944 vs 0.3979 ms
      // per step without a hint -- the SpMV then reads more of K11 from L2)
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;\n" ::"l"(K11g),
                   "r"(smem_u32(sstage)), "r"(static_cast<unsigned>(SM::ST11 * 8)), "l"(pol)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
    if (tid == 0 && k + NB * G < k_end) issue(k + NB * G, cur);
  }
  if (JP::STAGE && tid == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

// ============================================ 3-D line-streaming assembly
// For 3-D operators whose element flux-Jacobian working set does not fit
// shared memory (p = 4 Navier-Stokes, p = 4 Euler): one persistent CTA per
// element at a time.  The element's lines are streamed in groups of NP lines
// of one direction (dirs 2, 1, then 0; NL/NP groups per direction):
//   phase P  the group's quadrature-point flux Jacobians (A = dF_inv/du closed
//            form, Av = dF_vis/du closed form, Bq = dF_vis/dq closed form)
//   phase X  one item per (line, row, block entry) expands them into the line
//            blocks of that row (+ lifted endpoint blocks) and stores K11/K12
// with phase P of group g+1 (and its endpoint-scratch gather) running in the
// same barrier interval as phase X of group g (double-buffered).  No line is
// evaluated twice.  The self (diagonal) blocks accumulate in shared memory
// over the dir-2 and dir-1 passes; the dir-0 pass completes and stores them.
template <class C>
struct JacS3 {
  static constexpr int ev(int x) { return (x + 1) / 2 * 2; }
  static constexpr int NP = C::NP, NQ = C::NQ, M = C::M, MD = C::MD, B11 = C::B11;
  // lines per group: NP (one slab of a direction) for second-order physics,
  // a whole direction otherwise (no K12, small per-point footprint)
  static constexpr int GL = C::SECOND ? NP : C::NL;
  static constexpr int NG = C::NL / GL;                // groups per direction
  static constexpr int NPT = GL * NQ;                  // quadrature points per group
  // inviscid + viscous d/du Jacobians of a point are summed by the one
  // phase-P item that computes both (MERGE): one buffer, one load per point
  // and entry in phase X
  static constexpr bool MERGE = C::HAS_INV && C::VIS_U;
  static constexpr int A = C::HAS_INV ? NPT * B11 : 0;
  static constexpr int AV = (C::VIS_U && !MERGE) ? NPT * B11 : 0;
  static constexpr int BQ = C::SECOND ? NPT * M * MD : 0;
  static constexpr int PTS = ev(A + AV + BQ);          // one buffer
  static constexpr int SLS = 2 * GL;                   // line ends of a group (two sides)
  static constexpr int SEG = ev(SLS * EndJac<C>::SLOT); // one buffer: [side * GL + j][entry]
  static constexpr int U = ev(C::NPE * M);
  static constexpr int Q = C::SECOND ? ev(C::NPE * MD) : 0;
  static constexpr int MET = ev(C::METP);
  static constexpr int S11 = ev(C::NPE * B11);  // even sizes keep every buffer 16-byte aligned
  static constexpr int S12 = C::SECOND ? ev(C::NPE * C::B12) : 0;
  static constexpr int TAB = JacSmem<C>::TABD;         // cc[p][p][q], mi[p][side]
  static constexpr int NQ8 = (NQ + 1) / 2 * 2;          // cc rows padded to pairs (16-byte loads)
  static constexpr int CC8 = NP * NP * NQ8;
  static constexpr int IJ = ev(C::NPE + 2);             // 1/J buffer (aligned enclosing range)
  static constexpr int TOTAL = U + Q + MET + S11 + S12 + 2 * PTS + 2 * SEG + TAB + CC8 + 2 * IJ;
  static constexpr int THREADS = 512;
  static constexpr bool OK = C::D == 3 && 8LL * TOTAL <= 220 * 1024;
};

template <class C>
struct SeLay {
  using EJ = EndJac<C>;
  using S3 = JacS3<C>;
  // group-major for the configurations k_jac_s3 assembles (Launch::JAC_KIND == 1)
  static constexpr bool GM = !JacP<C>::OK && C::D == 3 && C::WU != 0 && S3::OK;
  static constexpr int GBLK = S3::SEG;  // one group: [side * GL + j][entry], a line end's entries contiguous
  static constexpr int PER_ELEM = GM ? C::D * S3::NG * GBLK : EJ::PER_ELEM;
  static constexpr int ES = GM ? 1 : EJ::LS;  // stride between the entries of a line end
  __host__ __device__ static constexpr int base(int dir, int side, int line) {
    return GM ? (dir * S3::NG + line / S3::GL) * GBLK + (side * S3::GL + line % S3::GL) * EJ::SLOT
              : (dir * 2 + side) * C::NL + line;
  }
};

template <class C>
__global__ void __launch_bounds__(JacS3<C>::THREADS, 1)
k_jac_s3(const KParams<C> kp, const double* __restrict__ U, const double* __restrict__ Q,
         const double* __restrict__ SE, double* __restrict__ K11, double* __restrict__ K12, int k_begin,
         int k_end) {
  using S3 = JacS3<C>;
  using EJ = EndJac<C>;
  using SM = JacSmem<C>;
  constexpr int NP = C::NP, NQ = C::NQ, NL = C::NL, NPE = C::NPE, M = C::M, MD = C::MD, D = C::D, P = C::P,
                NT = C::NT, B11 = C::B11, B12 = C::B12, GL = S3::GL, NG = S3::NG, SLS = S3::SLS;
  constexpr int A0 = C::PH == PH_NS ? 1 : 0;
  constexpr bool VOL11 = C::HAS_INV || C::VIS_U;
  extern __shared__ __align__(16) double smem[];
  double* const su = smem;
  double* const sq = su + S3::U;
  double* const mk = sq + S3::Q;
  double* const self11 = mk + S3::MET;
  double* const self12 = self11 + S3::S11;
  double* const pts0 = self12 + S3::S12;
  double* const seg0 = pts0 + 2 * S3::PTS;
  double* const stab = seg0 + 2 * S3::SEG;
  double* const cc8 = stab + S3::TAB;   // cc[i][t][q], rows padded to NQ8 (zeros)
  double* const sij0 = cc8 + S3::CC8;   // 1/J of the element's nodes, two buffers (element parity)
  const int tid = threadIdx.x, nthr = blockDim.x;
  const double* sccd = stab;            // cc[p][p][q]
  const double* smi = stab + NP * NQ;   // mi[p][side]
  constexpr int NQ8 = S3::NQ8;
  for (int x = tid; x < NP * NQ; x += nthr) stab[x] = kp.bt.cc[x / NQ][x / NQ][x % NQ];
  for (int x = tid; x < 2 * NP; x += nthr) stab[NP * NQ + x] = (&kp.bt.mi[0][0])[x];
  for (int x = tid; x < S3::CC8; x += nthr) {
    const int it = x / NQ8, q = x - it * NQ8;
    cc8[x] = q < NQ ? (&kp.bt.cc[0][0][0])[it * NQ + q] : 0.0;
  }
  // Factored line-block coefficients (cc[i][t][q] = dq[i][q] phi[t][q]): the
  // item scales its quadrature-point values by dq[i][.] once per line, then
  // sum_q phi[t][q] g[q] takes phi as compile-time-indexed constant-bank
  // operands (no shared-memory coefficient loads in the inner loop).
  constexpr bool FACT = true;
  auto phidot = [&](auto TC, const double* g) {
    constexpr int t = decltype(TC)::value;
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) v += kp.bt.phi[t][q] * g[q];
    return v;
  };
  // sum_q cc[i][t][q] f[q] with 16-byte coefficient loads
  auto ccdot = [&](int i, int t, const double* f) {
    const double2* c2 = reinterpret_cast<const double2*>(cc8 + (i * NP + t) * NQ8);
    double v = 0.0;
#pragma unroll
    for (int h = 0; h < NQ8 / 2; ++h) {
      const double2 cv = c2[h];
      v += cv.x * f[2 * h];
      if (2 * h + 1 < NQ) v += cv.y * f[2 * h + 1];
    }
    return v;
  };
  __shared__ int2 scon2[2][2 * D];           // connectivity, element parity
  __shared__ __align__(8) uint64_t ibar;     // element inputs
  unsigned iph = 0;
  if (tid == 0) mbar_init(&ibar, 1);
  __shared__ __align__(8) uint64_t sbar[2];  // one per scratch buffer
  unsigned sph = 0;                          // their phase parities (bit per buffer)
  if (tid == 0) {
    mbar_init(&sbar[0], 1);
    mbar_init(&sbar[1], 1);
    mbar_fence_init();
  }
  // group gi = (pass dd, group g): direction 2 - dd, lines g*GL + j
  auto gdir = [](int gi) { return 2 - gi / NG; };
  auto gline = [](int gi, int j) { return (gi % NG) * GL + j; };
  // Element inputs by bulk copy on one mbarrier (thread 0): the state and
  // gradient blocks (odd-sized blocks: the enclosing 16-byte-aligned range, data
  // at slot offset e & 1, as in BatchIO), the quadrature-point normals and the
  // 1/J table.  States, gradients and normals are read by phase P only, so the
  // next element's are fetched during the current element's last group (which
  // runs no phase P); 1/J and the connectivity, read by phase X, alternate
  // between two buffers.
  constexpr bool ODDU = ((NPE * M) & 1) != 0, ODDQ = C::SECOND && ((NPE * MD) & 1) != 0;
  constexpr int NVC = (C::MET_NV + 1) / 2 * 2;               // normals (rounded up to 16 bytes)
  constexpr int IJ0 = (C::MET_NV + C::MET_NE) / 2 * 2;       // aligned start of the 1/J range
  constexpr int IJN = C::METP - IJ0, IJO = C::MET_NV + C::MET_NE - IJ0;
  static_assert(IJN <= S3::IJ && NVC <= S3::MET, "k_jac_s3 input buffers");
  auto blk = [&](double* dst, const double* base, size_t ee, int N, bool odd, bool dry) -> unsigned {
    const double* src = base + ee * N;
    if (!odd) {
      if (!dry) tma_load_1d(dst, src, N * 8, &ibar);
      return N * 8;
    }
    const int par = static_cast<int>(ee & 1);
    if (par == 0 && ee + 1 == static_cast<size_t>(kp.E)) {  // no double behind the array's last block
      if (!dry) {
        tma_load_1d(dst, src, (N - 1) * 8, &ibar);
        dst[N - 1] = __ldg(src + N - 1);
      }
      return (N - 1) * 8;
    }
    if (!dry) tma_load_1d(dst, src - par, (N + 1) * 8, &ibar);
    return (N + 1) * 8;
  };
  // (issued by the lanes of warp t0 / 32: the last warp, which has no phase-X
  // items, when called from inside the group loop)
  auto load_inputs = [&](int kk, int eb, int t0) {
    const int lt = tid - t0;
    if (lt >= 0 && lt < 2 * D) scon2[eb][lt] = __ldg(&kp.conn[static_cast<size_t>(kk) * D * 2 + lt]);
    if (lt != 0) return;
    const size_t ee = kp.order[kk];
    const double* mg = kp.metric + static_cast<size_t>(kk) * C::METP;
    unsigned bytes = blk(nullptr, U, ee, NPE * M, ODDU, true) + (NVC + IJN) * 8;
    if (C::SECOND) bytes += blk(nullptr, Q, ee, NPE * MD, ODDQ, true);
    mbar_expect_tx(&ibar, bytes);
    blk(su, U, ee, NPE * M, ODDU, false);
    if (C::SECOND) blk(sq, Q, ee, NPE * MD, ODDQ, false);
    tma_load_1d(mk, mg, NVC * 8, &ibar);
    tma_load_1d(sij0 + eb * S3::IJ, mg + IJ0, IJN * 8, &ibar);
  };
  mbar_fence_init();
  __syncthreads();  // barriers initialised, tables written
  if (k_begin + static_cast<int>(blockIdx.x) < k_end) load_inputs(k_begin + blockIdx.x, 0, 0);
  int ebuf = 0;
  for (int k = k_begin + blockIdx.x; k < k_end; k += gridDim.x, ebuf ^= 1) {
    const size_t e = kp.order[k];
    const double* const suk = su + (ODDU ? static_cast<int>(e & 1) : 0);
    const double* const sqk = sq + (ODDQ ? static_cast<int>(e & 1) : 0);
    const double* const sij = sij0 + ebuf * S3::IJ + IJO;
    const int2* const scon = scon2[ebuf];
    const double* seel = SE + static_cast<size_t>(k - k_begin) * SeLay<C>::PER_ELEM;
    // endpoint scratch of group gi -> buffer bi: [off][side*GL + j] (stride
    // SLS), one bulk copy of the group's contiguous scratch block
    auto gather = [&](int gi, int bi) {
      if (tid == 0) {
        mbar_expect_tx(&sbar[bi], S3::SEG * 8);
        tma_load_1d(seg0 + bi * S3::SEG, seel + static_cast<size_t>(gdir(gi) * NG + gi % NG) * S3::SEG, S3::SEG * 8,
                    &sbar[bi]);
      }
    };
    // every thread waits for the group's block (acquires the async-proxy writes)
    auto gwait = [&](int bi) {
      mbar_wait(&sbar[bi], (sph >> bi) & 1u);
      sph ^= 1u << bi;
    };
    // phase P of group gi -> buffer
    auto phaseP = [&](int gi, double* pb) {
      const int dir = gdir(gi);
      double* pA = pb;
      double* pAv = pA + S3::A;
      double* pBq = pAv + S3::AV;
      // item kinds present: A (inviscid), Av (viscous d/du), Bq (viscous d/dq)
      constexpr bool MG = S3::MERGE;
      constexpr int KA = C::HAS_INV ? 1 : 0, KV = (C::VIS_U && !MG) ? 1 : 0, KB = C::SECOND ? 1 : 0;
      constexpr int KINDS = KA + KV + KB;
      // on the highest thread ids: phase X leaves them one item fewer
      for (int w = nthr - 1 - tid; w < GL * NQ * KINDS; w += nthr) {
        const int kind = w / (GL * NQ), pt = w - kind * (GL * NQ), j = pt / NQ, q = pt - j * NQ;
        const bool isA = KA && kind == 0, isV = MG ? isA : (KV && kind == KA);
        const int line = gline(gi, j);
        double nv[D], uq[M], qq[C::SECOND ? MD : 1];
#pragma unroll
        for (int d = 0; d < D; ++d) nv[d] = mk[((dir * NL + line) * NQ + q) * D + d];
#pragma unroll
        for (int c = 0; c < M; ++c) uq[c] = 0.0;
        if (C::SECOND) {
#pragma unroll
          for (int c = 0; c < MD; ++c) qq[c] = 0.0;
        }
#pragma unroll
        for (int t = 0; t < NP; ++t) {
          const int nd = node_on_line<C>(dir, line, t);
          const double ph = kp.bt.phi[t][q];
#pragma unroll
          for (int c = 0; c < M; ++c) uq[c] += ph * suk[nd * M + c];
          if (C::SECOND && isV) {
#pragma unroll
            for (int c = 0; c < MD; ++c) qq[c] += ph * sqk[nd * MD + c];
          }
        }
        bool ok = true;
        if (MG && isA) {
          euler_jac_n<D>(uq, nv, kp.pp.gamma, pA + pt * B11, ok);
          double Jv[M * M];
          visc_du<D, C::PH>(uq, qq, nv, kp.pp, Jv, ok);
#pragma unroll
          for (int c = 0; c < M * M; ++c) pA[pt * B11 + c] += Jv[c];
        } else if (isA) {
          if (C::HAS_INV) euler_jac_n<D>(uq, nv, kp.pp.gamma, pA + pt * B11, ok);
        } else if (isV) {
          double Jv[M * M];
          visc_du<D, C::PH>(uq, qq, nv, kp.pp, Jv, ok);
#pragma unroll
          for (int c = 0; c < M * M; ++c) pAv[pt * B11 + c] = Jv[c];
        } else if (C::SECOND) {
          double L[M * MD];
          visc_dq<D, C::PH>(uq, nv, kp.pp, L, ok);
#pragma unroll
          for (int c = 0; c < M * MD; ++c) pBq[pt * M * MD + c] = L[c];
        }
        if (!ok) report_line<C>(kp, static_cast<int>(e), dir, line, suk);
      }
    };
    auto avq = [&](const double* pA, const double* pAv, int j, int q, int ab) {
      if (S3::MERGE) return pA[(j * NQ + q) * B11 + ab];
      return (C::HAS_INV ? pA[(j * NQ + q) * B11 + ab] : 0.0) + (C::VIS_U ? pAv[(j * NQ + q) * B11 + ab] : 0.0);
    };
    // phase X of group gi from buffers pb (quadrature points) and sg (scratch).
    // The direction is a compile-time constant (DIRC) so the line/slot index
    // maps fold; one thread owns a (row position i, block entry) pair and walks
    // the group's GL lines (its index decomposition and slot offsets are
    // computed once per group).
    auto phaseX = [&](auto DIRC, int gi, const double* pb, const double* sg) {
      constexpr int dir = decltype(DIRC)::value;
      const double* pA = pb;
      const double* pAv = pA + S3::A;
      const double* pBq = pAv + S3::AV;
      const int2 c0 = scon[dir * 2 + 0], c1 = scon[dir * 2 + 1];
      const int g0 = (gi % NG) * GL;  // first line of the group
      constexpr int N11 = NP * B11;
      constexpr int N12 = C::SECOND ? NP * B12 : 0;
      double* const K11e = K11 + static_cast<size_t>(k) * C::TPE * SM::ST11;
      double* const K12e = C::SECOND ? K12 + static_cast<size_t>(k) * C::TPE * SM::ST12 : nullptr;
      for (int w = tid; w < N11 + N12; w += nthr) {
        if (w < N11) {
          // ---- K11: row position i, entry ab = a*M + b, all GL lines of the group
          // lanes run over (a, i, b): for dir 0 the NP rows of a line are
          // consecutive rows of one tile, so a (slot, a) run of NP * M
          // doubles is written by consecutive lanes
          const int a_ = w / (NP * M), r_ = w - a_ * (NP * M), i = r_ / M, ab = a_ * M + (r_ - i * M);
          const double li0 = smi[i * 2 + 0], li1 = smi[i * 2 + 1];
          const size_t eoff = (static_cast<size_t>(ab / M) * NT) * M + ab % M;
          double dqi[FACT ? NQ : 1];
          if (FACT) {
#pragma unroll
            for (int q = 0; q < NQ; ++q) dqi[q] = kp.bt.dq[i][q];
          }
#pragma unroll 1
          for (int j = 0; j < GL; ++j) {
            const int nd = node_on_line<C>(dir, g0 + j, i);
            const double sc = -sij[nd];
            const double e0 = sg[(j) * EJ::SLOT + ab], e1 = sg[(GL + j) * EJ::SLOT + ab];
            double av[NQ8];
#pragma unroll
            for (int q = 0; q < NQ8; ++q) {
              av[q] = (VOL11 && q < NQ) ? avq(pA, pAv, j, q, ab) : 0.0;
              if (FACT && q < NQ) av[q] *= dqi[q];
            }
            double* rowp = K11e + static_cast<size_t>(nd / NT) * SM::ST11 + eoff + static_cast<size_t>(nd % NT) * M;
            static_for<NP>([&](auto TC) {
              constexpr int t = decltype(TC)::value;
              double v = !VOL11 ? 0.0 : (FACT ? phidot(TC, av) : ccdot(i, t, av));
              if (t == 0) v += li0 * e0;
              if (t == P) v += li1 * e1;
              if (t == i) {
                // self block: dir 2 starts it, dir 1 adds, dir 0 completes and stores
                double* sp = self11 + nd * B11 + ab;
                if (dir == 2) *sp = v;
                else if (dir == 1) *sp += v;
                else rowp[static_cast<size_t>(t) * NT * B11] = sc * (v + *sp);
                return;
              }
              const int slot = dir == 0 ? t : NP + (dir - 1) * P + (t < i ? t : t - 1);
              rowp[static_cast<size_t>(slot) * NT * B11] = sc * v;
            });
            rowp[static_cast<size_t>(D * P + 1 + 2 * dir + 0) * NT * B11] =
                c0.x >= 0 ? sc * (li0 * sg[(j) * EJ::SLOT + (B11 + ab)]) : 0.0;
            rowp[static_cast<size_t>(D * P + 1 + 2 * dir + 1) * NT * B11] =
                c1.x >= 0 ? sc * (li1 * sg[(GL + j) * EJ::SLOT + (B11 + ab)]) : 0.0;
          }
        } else if (C::SECOND) {
          // ---- K12: row position i, stored entry ab = a' * MD + b, all GL lines
          const int v12 = w - N11;
          const int a_ = v12 / (NP * MD), r_ = v12 - a_ * (NP * MD), i = r_ / MD, ab = a_ * MD + (r_ - i * MD);
          const int a = ab / MD + A0, b = ab % MD;
          const double li0 = smi[i * 2 + 0], li1 = smi[i * 2 + 1];
          const bool own0 = c0.x < 0 || conn_sign(c0.y) <= 0;
          const bool own1 = c1.x < 0 || conn_sign(c1.y) <= 0;
          const size_t eoff = (static_cast<size_t>(ab / MD) * NT) * MD + ab % MD;
          double dqi[FACT ? NQ : 1];
          if (FACT) {
#pragma unroll
            for (int q = 0; q < NQ; ++q) dqi[q] = kp.bt.dq[i][q];
          }
#pragma unroll 1
          for (int j = 0; j < GL; ++j) {
            const int nd = node_on_line<C>(dir, g0 + j, i);
            const double sc = -sij[nd];
            double bv[NQ8];
#pragma unroll
            for (int q = 0; q < NQ8; ++q) {
              bv[q] = q < NQ ? pBq[(j * NQ + q) * M * MD + a * MD + b] : 0.0;
              if (FACT && q < NQ) bv[q] *= dqi[q];
            }
            const double eq0 = sg[(j) * EJ::SLOT + (2 * B11 + a * MD + b)];
            const double eq1 = sg[(GL + j) * EJ::SLOT + (2 * B11 + a * MD + b)];
            double* rowp = K12e + static_cast<size_t>(nd / NT) * SM::ST12 + eoff + static_cast<size_t>(nd % NT) * MD;
            static_for<NP>([&](auto TC) {
              constexpr int t = decltype(TC)::value;
              double v = FACT ? phidot(TC, bv) : ccdot(i, t, bv);
              if (t == 0 && own0) v += li0 * eq0;
              if (t == P && own1) v += li1 * eq1;
              if (t == i) {
                double* sp = self12 + nd * B12 + ab;
                if (dir == 2) *sp = v;
                else if (dir == 1) *sp += v;
                else rowp[static_cast<size_t>(t) * NT * B12] = sc * (v + *sp);
                return;
              }
              const int slot = dir == 0 ? t : NP + (dir - 1) * P + (t < i ? t : t - 1);
              rowp[static_cast<size_t>(slot) * NT * B12] = sc * v;
            });
            double nbv = 0.0;
            if (!own0) nbv = sc * (li0 * eq0);
            if (!own1) nbv = sc * (li1 * eq1);
            rowp[static_cast<size_t>(D * P + 1 + dir) * NT * B12] = nbv;
          }
        }
      }
    };
    // phase X for directions 1 and 2: the NP rows of a line lie in NP
    // different tiles, but the lines of a group are consecutive rows of each
    // of them.  One thread owns a (line j of the group, block entry) pair with
    // lanes running over (a, j, b) -- consecutive lanes write a contiguous
    // (slot, a) run -- and walks the line's NP row positions: the line's
    // quadrature-point values and endpoint entries are loaded once.
    auto phaseXL = [&](auto DIRC, int gi, const double* pb, const double* sg) {
      constexpr int dir = decltype(DIRC)::value;
      static_assert(dir == 1 || dir == 2, "phaseXL: directions 1 and 2");
      const double* pA = pb;
      const double* pAv = pA + S3::A;
      const double* pBq = pAv + S3::AV;
      const int2 c0 = scon[dir * 2 + 0], c1 = scon[dir * 2 + 1];
      const int g0 = (gi % NG) * GL;  // first line of the group
      constexpr int N11 = GL * B11;
      constexpr int N12 = C::SECOND ? GL * B12 : 0;
      constexpr bool TLINE = NT == NP;  // store tile: a dir-0 line of rows, else an x2 slab
      constexpr int NDS = dir == 1 ? NP : NP * NP;  // node stride along the line
      constexpr size_t RS11 = TLINE ? (dir == 1 ? size_t(SM::ST11) : size_t(NP) * SM::ST11)
                                    : (dir == 1 ? size_t(NP) * M : size_t(SM::ST11));
      constexpr size_t RS12 = TLINE ? (dir == 1 ? size_t(SM::ST12) : size_t(NP) * SM::ST12)
                                    : (dir == 1 ? size_t(NP) * MD : size_t(SM::ST12));
      double* const K11e = K11 + static_cast<size_t>(k) * C::TPE * SM::ST11;
      double* const K12e = C::SECOND ? K12 + static_cast<size_t>(k) * C::TPE * SM::ST12 : nullptr;
      for (int w = tid; w < N11 + N12; w += nthr) {
        if (w < N11) {
          const int jh = w / (NP * B11), r1 = w - jh * (NP * B11), a = r1 / (NP * M), r2 = r1 - a * (NP * M),
                    jl = r2 / M, b = r2 - jl * M;
          const int j = jh * NP + jl, ab = a * M + b;
          const int line = g0 + j, l1 = line % NP, l2 = line / NP;
          const int nd0 = dir == 1 ? l1 + NP * NP * l2 : l1 + NP * l2;
          const int t0 = TLINE ? (dir == 1 ? NP * l2 : l2) : (dir == 2 ? 0 : l2);
          const int r0 = TLINE ? l1 : (dir == 1 ? l1 : l1 + NP * l2);
          double* rowp = K11e + static_cast<size_t>(t0) * SM::ST11 + (static_cast<size_t>(a) * NT + r0) * M + b;
          const double* mks = sij + nd0;
          double* sp = self11 + nd0 * B11 + ab;
          double av[NQ];
#pragma unroll
          for (int q = 0; q < NQ; ++q) av[q] = VOL11 ? avq(pA, pAv, j, q, ab) : 0.0;
          const double e0 = sg[(j) * EJ::SLOT + ab], e1 = sg[(GL + j) * EJ::SLOT + ab];
          const double eo0 = sg[(j) * EJ::SLOT + (B11 + ab)], eo1 = sg[(GL + j) * EJ::SLOT + (B11 + ab)];
#pragma unroll 1
          for (int i = 0; i < NP; ++i, rowp += RS11, sp += NDS * B11) {
            const double sc = -mks[i * NDS];
            const double li0 = smi[i * 2 + 0], li1 = smi[i * 2 + 1];
            double g[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) g[q] = av[q] * kp.bt.dq[i][q];
            static_for<NP>([&](auto TC) {
              constexpr int t = decltype(TC)::value;
              double v = VOL11 ? phidot(TC, g) : 0.0;
              if (t == 0) v += li0 * e0;
              if (t == P) v += li1 * e1;
              if (t == i) {
                // self block: dir 2 starts it, dir 1 adds (dir 0 completes and stores)
                if (dir == 2) *sp = v;
                else *sp += v;
                return;
              }
              const int slot = NP + (dir - 1) * P + (t < i ? t : t - 1);
              rowp[static_cast<size_t>(slot) * NT * B11] = sc * v;
            });
            rowp[static_cast<size_t>(D * P + 1 + 2 * dir + 0) * NT * B11] = c0.x >= 0 ? sc * (li0 * eo0) : 0.0;
            rowp[static_cast<size_t>(D * P + 1 + 2 * dir + 1) * NT * B11] = c1.x >= 0 ? sc * (li1 * eo1) : 0.0;
          }
        } else if (C::SECOND) {
          const int v12 = w - N11;
          const int jh = v12 / (NP * B12), r1 = v12 - jh * (NP * B12), a_ = r1 / (NP * MD),
                    r2 = r1 - a_ * (NP * MD), jl = r2 / MD, b = r2 - jl * MD;
          const int j = jh * NP + jl, ab = a_ * MD + b, a = a_ + A0;
          const int line = g0 + j, l1 = line % NP, l2 = line / NP;
          const int nd0 = dir == 1 ? l1 + NP * NP * l2 : l1 + NP * l2;
          const int t0 = TLINE ? (dir == 1 ? NP * l2 : l2) : (dir == 2 ? 0 : l2);
          const int r0 = TLINE ? l1 : (dir == 1 ? l1 : l1 + NP * l2);
          double* rowp = K12e + static_cast<size_t>(t0) * SM::ST12 + (static_cast<size_t>(a_) * NT + r0) * MD + b;
          const double* mks = sij + nd0;
          double* sp = self12 + nd0 * B12 + ab;
          const bool own0 = c0.x < 0 || conn_sign(c0.y) <= 0;
          const bool own1 = c1.x < 0 || conn_sign(c1.y) <= 0;
          double bv[NQ];
#pragma unroll
          for (int q = 0; q < NQ; ++q) bv[q] = pBq[(j * NQ + q) * M * MD + a * MD + b];
          const double eq0 = sg[(j) * EJ::SLOT + (2 * B11 + a * MD + b)];
          const double eq1 = sg[(GL + j) * EJ::SLOT + (2 * B11 + a * MD + b)];
#pragma unroll 1
          for (int i = 0; i < NP; ++i, rowp += RS12, sp += NDS * B12) {
            const double sc = -mks[i * NDS];
            const double li0 = smi[i * 2 + 0], li1 = smi[i * 2 + 1];
            double g[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) g[q] = bv[q] * kp.bt.dq[i][q];
            static_for<NP>([&](auto TC) {
              constexpr int t = decltype(TC)::value;
              double v = phidot(TC, g);
              if (t == 0 && own0) v += li0 * eq0;
              if (t == P && own1) v += li1 * eq1;
              if (t == i) {
                if (dir == 2) *sp = v;
                else *sp += v;
                return;
              }
              const int slot = NP + (dir - 1) * P + (t < i ? t : t - 1);
              rowp[static_cast<size_t>(slot) * NT * B12] = sc * v;
            });
            double nbv = 0.0;
            if (!own0) nbv = sc * (li0 * eq0);
            if (!own1) nbv = sc * (li1 * eq1);
            rowp[static_cast<size_t>(D * P + 1 + dir) * NT * B12] = nbv;
          }
        }
      }
    };
    (void)sccd;
    // ---- pipeline over the 3*NG groups
    mbar_wait(&ibar, iph);
    iph ^= 1u;
    __syncthreads();  // element inputs (bulk data, connectivity)
    gather(0, 0);
    phaseP(0, pts0);
    gwait(0);
    __syncthreads();
    constexpr int NGT = 3 * NG;
    for (int gi = 0; gi < NGT - 1; ++gi) {
      const int cb = gi & 1, nb = cb ^ 1;
      gather(gi + 1, nb);
      {
        const double* pb = pts0 + cb * S3::PTS;
        const double* sgb = seg0 + cb * S3::SEG;
        // (an fp64 tensor-core (DMMA m8n8k4) phase X was measured parity-green
        // but slower -- C5 127.0 vs 92.8 ms: the per-entry epilogue, not the
        // contraction, bounds this phase; commit 101d93b)
        switch (gdir(gi)) {
          case 0: phaseX(std::integral_constant<int, 0>{}, gi, pb, sgb); break;
          case 1: phaseXL(std::integral_constant<int, 1>{}, gi, pb, sgb); break;
          default: phaseXL(std::integral_constant<int, 2>{}, gi, pb, sgb); break;
        }
      }
      phaseP(gi + 1, pts0 + nb * S3::PTS);
      gwait(nb);
      __syncthreads();
    }
    {
      // last group (direction 0, no phase P): the next element's inputs are
      // fetched behind it (kept out of the loop above: a call inside it costs
      // the loop's code quality more than the overlap gains, measured)
      constexpr int gi = NGT - 1, cb = gi & 1;
      if (k + static_cast<int>(gridDim.x) < k_end) load_inputs(k + gridDim.x, ebuf ^ 1, nthr - 32);
      phaseX(std::integral_constant<int, 0>{}, gi, pts0 + cb * S3::PTS, seg0 + cb * S3::SEG);
      __syncthreads();
    }
  }
}

// K21 = dQ/dU (U-independent; D scalars per node pair), same tiles/rows.
// K21 wall terms of row node nd of element k (processing index): at a
// no-slip-wall end the gradient trace of density and energy is the own trace
// (zero momentum), so K21 gains (1/J) M^-1[pos][side] n_d for those two
// components only -- kept out of the component-uniform K21 store and applied
// by its consumers (k_spmv21, k_pc_build, the export).  f(end_node, coef[D]).
template <class C, class F>
__device__ __forceinline__ void k21_wall_terms(const KParams<C>& kp, int k, int nd, F&& f) {
  constexpr int D = C::D, NL = C::NL, P = C::P;
  const double* mk = kp.metric + static_cast<size_t>(k) * C::METP;
  const double invJ = __ldg(mk + C::MET_NV + C::MET_NE + nd);
#pragma unroll
  for (int dir = 0; dir < D; ++dir)
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const int2 cx = __ldg(&kp.conn[(static_cast<size_t>(k) * D + dir) * 2 + side]);
      if (cx.x >= 0 || __ldg(kp.bck + (-1 - cx.x)) != BC_NO_SLIP) continue;
      int line, pos;
      line_of<C>(dir, nd, line, pos);
      const double mi = kp.bt.mi[pos][side];
      double cf[D];
#pragma unroll
      for (int d = 0; d < D; ++d) cf[d] = invJ * (mi * __ldg(mk + C::MET_NV + ((dir * 2 + side) * NL + line) * D + d));
      f(node_on_line<C>(dir, line, side ? P : 0), cf);
    }
}

template <class C>
__global__ void __launch_bounds__(128) k_k21(const KParams<C> kp, double* __restrict__ K21) {
  constexpr int NP = C::NP, NQ = C::NQ, NL = C::NL, D = C::D, NT = C::NT, P = C::P;
  constexpr int NLT = TileLines<C>::NLT;
  constexpr int ST = C::NS12 * D * NT;
  const int W = blockIdx.x;  // work unit
  const int k = W / C::UPE, s = W - k * C::UPE;
  const double* mk = kp.metric + static_cast<size_t>(k) * C::METP;
  double* Kt = K21 + static_cast<size_t>(k) * C::TPE * ST;
  auto coef = [&](int dir, int line, int p, int t, int d, int2 c0, int2 c1) {
    // line block entry (row position p, column position t) of direction d
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) v += kp.bt.cc[p][t][q] * __ldg(mk + ((dir * NL + line) * NQ + q) * D + d);
    // u_hat = own trace where S = +1, neighbour where S = -1; on boundaries
    // g_D (Dirichlet-type: no u dependence) or the own trace (Neumann / slip wall)
    auto own_uh = [&](int2 cx) { return cx.x >= 0 ? conn_sign(cx.y) > 0 : bnd_uhat_inner(kp, -1 - cx.x); };
    if (t == 0 && own_uh(c0))
      v += kp.bt.mi[p][0] * __ldg(mk + C::MET_NV + ((dir * 2 + 0) * NL + line) * D + d);
    if (t == P && own_uh(c1))
      v += kp.bt.mi[p][1] * __ldg(mk + C::MET_NV + ((dir * 2 + 1) * NL + line) * D + d);
    return v;
  };
  for (int w = threadIdx.x; w < NLT * D; w += blockDim.x) {
    const int tl = w / D, d = w - tl * D;
    int dir, line;
    TileLines<C>::get(tl, s, dir, line);
    const bool full = TileLines<C>::full(dir);
    const int2 c0 = __ldg(&kp.conn[(static_cast<size_t>(k) * D + dir) * 2 + 0]);
    const int2 c1 = __ldg(&kp.conn[(static_cast<size_t>(k) * D + dir) * 2 + 1]);
    const bool nbr0 = c0.x >= 0 && conn_sign(c0.y) <= 0;
    const bool nbr1 = c1.x >= 0 && conn_sign(c1.y) <= 0;
    const double n0 = __ldg(mk + C::MET_NV + ((dir * 2 + 0) * NL + line) * D + d);
    const double n1 = __ldg(mk + C::MET_NV + ((dir * 2 + 1) * NL + line) * D + d);
    auto body = [&](const int i) {
      const int nd = node_on_line<C>(dir, line, i);
      const int r = nd % NT;
      const double sc = __ldg(mk + C::MET_NV + C::MET_NE + nd);
      double* rowp = Kt + static_cast<size_t>(nd / NT) * ST + static_cast<size_t>(r) * D + d;
#pragma unroll
      for (int t = 0; t < NP; ++t) {
        if (t == i && dir != 0) continue;
        double v = coef(dir, line, i, t, d, c0, c1);
        if (t == i) {
#pragma unroll
          for (int d2 = 1; d2 < D; ++d2) {
            int l2, p2;
            line_of<C>(d2, nd, l2, p2);
            const int2 x0 = __ldg(&kp.conn[(static_cast<size_t>(k) * D + d2) * 2 + 0]);
            const int2 x1 = __ldg(&kp.conn[(static_cast<size_t>(k) * D + d2) * 2 + 1]);
            v += coef(d2, l2, p2, p2, d, x0, x1);
          }
        }
        rowp[static_cast<size_t>(inel_slot<C>(dir, i, t)) * NT * D] = sc * v;
      }
      double nbv = 0.0;
      if (nbr0) nbv = sc * (kp.bt.mi[i][0] * n0);
      if (nbr1) nbv = sc * (kp.bt.mi[i][1] * n1);
      rowp[static_cast<size_t>(C::D * P + 1 + dir) * NT * D] = nbv;
    };
    if (full) {
#pragma unroll
      for (int i = 0; i < NP; ++i) body(i);
    } else {
      body(TileLines<C>::prow(dir, s));
    }
  }
}

// ===================================================================== SpMV
// Column node of `slot` for the row at node nd of element e (reference id).
// NBR = number of neighbour slots per direction (2 for K11, 1 for K12/K21
// where `nsel` picks the side by the switch).
template <class C, int NSIN>
__device__ __forceinline__ int64_t slot_col(const KParams<C>& kp, int k, size_t e, int nd, int slot,
                                            int kind /*0: K11, 1: K12, 2: K21*/) {
  constexpr int NP = C::NP, D = C::D, P = C::P, NPE = C::NPE;
  const int x[3] = {nd % NP, (nd / NP) % NP, nd / (NP * NP)};
  const int st[3] = {1, NP, NP * NP};
  if (slot < NSIN) {
    int dir, t;
    if (slot < NP) {
      dir = 0;
      t = slot;
    } else {
      const int z = slot - NP;
      dir = 1 + z / P;
      t = z % P;
      if (t >= x[dir]) ++t;
    }
    return static_cast<int64_t>(e) * NPE + nd + (t - x[dir]) * st[dir];
  }
  int dir, side;
  const int z = slot - NSIN;
  if (kind == 0) {
    dir = z >> 1;
    side = z & 1;
  } else {
    dir = z;
    const int2 cs = __ldg(&kp.conn[(static_cast<size_t>(k) * D + dir) * 2 + 1]);
    // K12: the side whose switch is +1; K21: the side whose switch is -1.
    const bool plus1 = conn_sign(cs.y) > 0;
    side = kind == 1 ? (plus1 ? 1 : 0) : (plus1 ? 0 : 1);
  }
  const int2 cn = __ldg(&kp.conn[(static_cast<size_t>(k) * D + dir) * 2 + side]);
  if (cn.x < 0) return -1;
  int line, pos;
  line_of<C>(dir, nd, line, pos);
  return static_cast<int64_t>(cn.x) * NPE + conn_node(cn.y, line, NP);
}

// slot_col with the element's 2D connectivity entries already at hand (cn).
template <class C, int NSIN>
__device__ __forceinline__ int64_t slot_col_c(const int2* cn, size_t e, int nd, int slot, int kind) {
  constexpr int NP = C::NP, P = C::P, NPE = C::NPE;
  const int x[3] = {nd % NP, (nd / NP) % NP, nd / (NP * NP)};
  const int st[3] = {1, NP, NP * NP};
  if (slot < NSIN) {
    int dir, t;
    if (slot < NP) {
      dir = 0;
      t = slot;
    } else {
      const int z = slot - NP;
      dir = 1 + z / P;
      t = z % P;
      if (t >= x[dir]) ++t;
    }
    return static_cast<int64_t>(e) * NPE + nd + (t - x[dir]) * st[dir];
  }
  int dir, side;
  const int z = slot - NSIN;
  if (kind == 0) {
    dir = z >> 1;
    side = z & 1;
  } else {
    dir = z;
    const bool plus1 = conn_sign(cn[dir * 2 + 1].y) > 0;
    side = kind == 1 ? (plus1 ? 1 : 0) : (plus1 ? 0 : 1);
  }
  const int2 c = cn[dir * 2 + side];
  if (c.x < 0) return -1;
  int line, pos;
  line_of<C>(dir, nd, line, pos);
  return static_cast<int64_t>(c.x) * NPE + conn_node(c.y, line, NP);
}

// y = K11 x  (SPLIT: y = v - adt (K11 v + K12 w), the split matvec).
// One thread per (row, output component a); a warp covers 32 consecutive
// rows of one a.  Block row a of a slot is m contiguous doubles (16-byte
// loads when m is even); the x entries of a column are shared by the m
// threads of a row through L1.
// Jacobian value stream of the SpMV (read once): 0 ld.global.nc, 1 streaming
// (ld.global.cs), 2 ld.global.nc.L1::no_allocate
static constexpr int LDG_SPMV_STREAM = 1;  // measured: C2 SpMV 120.3 -> 115.4 us (ld.global.cs), C4 neutral
__device__ __forceinline__ double2 ld_stream2(const double* p) {
  if (LDG_SPMV_STREAM == 1) return __ldcs(reinterpret_cast<const double2*>(p));
  if (LDG_SPMV_STREAM == 2) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
  }
  return __ldg(reinterpret_cast<const double2*>(p));
}
__device__ __forceinline__ double ld_stream1(const double* p) { return LDG_SPMV_STREAM == 1 ? __ldcs(p) : __ldg(p); }
template <class C, bool SPLIT, bool ZC = false>
__global__ void __launch_bounds__(128)
k_spmv11(const KParams<C> kp, const double* __restrict__ V11, const double* __restrict__ V12,
         const double* __restrict__ x, const double* __restrict__ w, double adt, double* __restrict__ y, int rev) {
  constexpr int M = C::M, NT = C::NT, NPE = C::NPE, MD = C::MD, B11 = C::B11;
  // rev: blocks walk the rows from the end -- the Jacobian assembly writes the
  // store in increasing tile order, so its last ~L2-size of tiles is still
  // cached when the first matvec after an assembly starts (a gain where that
  // is a noticeable share of the store: the launcher sets rev for stores <= 1 GB)
  const int64_t gid = static_cast<int64_t>(rev ? gridDim.x - 1 - blockIdx.x : blockIdx.x) * blockDim.x +
                      threadIdx.x;
  const int64_t nrows = static_cast<int64_t>(kp.E) * NPE;
  const int lane = static_cast<int>(gid & 31);
  const int64_t wg = gid >> 5;
  const int a = static_cast<int>(wg % M);
  const int64_t row = (wg / M) * 32 + lane;
  // ZC (y is mapped pinned host memory, ldg_bsr_spmv_host), M = 4: the CTA's
  // four warps are the four components of the same 32 rows; the results leave
  // through shared memory so that every warp store writes whole node rows
  // (contiguous 256-byte runs over PCIe).  (Device y: direct stores, measured
  // 7 us faster on C2.)
  constexpr bool STG = ZC && !SPLIT && M == 4;
  __shared__ double sy[STG ? 4 * 32 : 1];
  if (!STG && row >= nrows) return;
  if (row < nrows) {
  const int64_t T = row / NT;
  const int r = static_cast<int>(row - T * NT);
  const int k = static_cast<int>(T / C::TPE);
  const int s = static_cast<int>(T - static_cast<int64_t>(k) * C::TPE);
  const int nd = s * NT + r;
  const size_t e = __ldg(kp.order + k);
  double acc = 0.0;
  const double* vb = V11 + T * C::NS11 * NT * B11 + (static_cast<size_t>(a) * NT + r) * M;
#pragma unroll
  for (int slot = 0; slot < C::NS11; ++slot) {
    const int64_t col = slot_col<C, C::D * C::P + 1>(kp, k, e, nd, slot, 0);
    if (col < 0) continue;
    const double* vp = vb + static_cast<size_t>(slot) * NT * B11;
    const double* xp = x + col * M;
    if (M % 2 == 0) {
#pragma unroll
      for (int b = 0; b < M; b += 2) {
        // (streaming loads where the store is small enough that its tail is
        // still in L2 -- the same condition as rev; measured C2 -5 us, C3 +6 us)
        const double2 kv = rev ? ld_stream2(vp + b) : __ldg(reinterpret_cast<const double2*>(vp + b));
        const double2 xv = __ldg(reinterpret_cast<const double2*>(xp + b));
        acc += kv.x * xv.x;
        acc += kv.y * xv.y;
      }
    } else {
#pragma unroll
      for (int b = 0; b < M; ++b) acc += (rev ? ld_stream1(vp + b) : __ldg(vp + b)) * __ldg(xp + b);
    }
  }
  if (SPLIT && C::SECOND) {
    constexpr int A0 = C::PH == PH_NS ? 1 : 0;
    if (a >= A0) {
      const double* vq = V12 + T * C::NS12 * NT * C::B12 + (static_cast<size_t>(a - A0) * NT + r) * MD;
#pragma unroll
      for (int slot = 0; slot < C::NS12; ++slot) {
        const int64_t col = slot_col<C, C::D * C::P + 1>(kp, k, e, nd, slot, 1);
        if (col < 0) continue;
        const double* vp = vq + static_cast<size_t>(slot) * NT * C::B12;
#pragma unroll
        for (int b = 0; b < MD; ++b) acc += __ldg(vp + b) * __ldg(w + col * MD + b);
      }
    }
  }
  if (STG) {
    sy[lane * 4 + a] = acc;
  } else {
    const size_t yo = (e * NPE + nd) * M + a;
    if (SPLIT) y[yo] = __ldg(x + yo) - adt * acc;
    else y[yo] = acc;
  }
  }
  if (STG) {
    __syncthreads();  // (reached by every thread of the CTA)
    // thread t writes component t % 4 of row (block rows) + t / 4
    const int t = threadIdx.x;
    const int64_t r2 = (wg / M) * 32 + (t >> 2);
    if (r2 < nrows) {
      const int64_t T2 = r2 / NT;
      const int k2 = static_cast<int>(T2 / C::TPE);
      const int nd2 = static_cast<int>(T2 - static_cast<int64_t>(k2) * C::TPE) * NT + static_cast<int>(r2 - T2 * NT);
      const size_t e2 = __ldg(kp.order + k2);
      y[(e2 * NPE + nd2) * M + (t & 3)] = sy[t];
    }
  }
}

// Split matvec y = v - adt (K11 v + K12 w) for second-order physics, streamed
// tile by tile (k_mv_tiles).  The store keeps each row tile's K11 and K12
// values contiguous (19 KB + 38 KB per dir-0 line tile of C5), so a
// persistent CTA per SM pulls whole tiles into shared memory with 1-D TMA
// bulk copies (cp.async.bulk, completion on an mbarrier) on an NSTAGE-deep
// ring: the HBM stream is a sequence of large bulk reads instead of
// per-thread strided 8-byte loads (the K12 rows are m*D = 15 doubles per lane
// in the row-per-thread kernel).  The v / w entries of every (slot, row)
// column node of tile i+1 are gathered into shared memory with cp.async while
// tile i computes (L1/L2 hits: a CTA walks consecutive tiles of the same
// elements; the tile's connectivity is fetched two tiles ahead).  Within a
// tile one item per (slot group, output component, row) forms a partial dot
// product from shared memory only; the partials land in shared memory and the
// (row, component) owner sums them in a fixed order (deterministic, no
// atomics) and writes y.  The gathers run on the threads with one item fewer.
template <class C>
struct MvT {
  static constexpr int ev(int x) { return (x + 1) / 2 * 2; }
  static constexpr int NT = C::NT, M = C::M, MD = C::MD, R12 = C::R12;
  static constexpr int ST11 = C::NS11 * C::B11 * NT;   // doubles per tile
  static constexpr int ST12 = C::NS12 * C::B12 * NT;
  static constexpr int BUF11 = ev(ST11 + 1);          // +1: an odd tile offset is loaded from 8 B earlier
  static constexpr int BUF12 = ev(ST12 + 1);
  static constexpr int BUF = BUF11 + BUF12;
  static constexpr int GX = C::NS11 * NT * M;          // gathered v per tile [slot][row][c]
  static constexpr int GW = C::NS12 * NT * MD;         // gathered w per tile [slot][row][c]
  static constexpr int GBUF = ev(GX + GW);
  // slots per item: K11 items take SG11 slots, K12 items SG12, so that every
  // item is about m*D multiply-adds long (C5: 15 each, 495 items, one round)
  static constexpr int SG11 = (MD + M - 1) / M, SG12 = 1;
  static constexpr int SG = SG11;
  static constexpr int G11 = (C::NS11 + SG11 - 1) / SG11, G12 = (C::NS12 + SG12 - 1) / SG12;
  static constexpr int NPART = G11 + G12;
  static constexpr int NOUT = NT * M;
  static constexpr int PART = ev(NOUT * NPART);
  // (C5 needs 880 role threads; 896 measured 0.6 % faster than 1024 in the
  // sustained matvec loop: four fewer idle warps at every tile barrier)
  static constexpr int THREADS = 896;
  static constexpr int I11 = G11 * M * NT, I12 = G12 * R12 * NT;  // items per tile
  // gather units: one per (K11 slot, row) and per (K12 slot, row, M-component group)
  static constexpr int NG = C::NS11 * NT + C::NS12 * NT * (MD / M);
  // gathers run GA tiles ahead (GA + 1 gather buffers): their first touch of
  // an element is an HBM miss, longer than one tile's compute.  Measured (C5):
  // one tile ahead 36.4 ms, two 30.8, three / four 30.8; ring of 2 or 3
  // tiles alike.
  static constexpr int GA = 2, NGB = GA + 1;
  static constexpr long long bytes(int ns) { return 8LL * (ns * BUF + NGB * GBUF + 2 * PART) + 64; }
  static constexpr int NSTAGE = bytes(3) <= 225 * 1024 ? 3 : 2;
  static constexpr int TOTAL = NSTAGE * BUF + NGB * GBUF + 2 * PART;
  // thread roles: items, owners (one warp per 32 outputs), issuer, gathers
  static constexpr int ROLES = (I11 + I12 + 31) / 32 * 32 + (NOUT + 31) / 32 * 32 + 1 + NG;
  static constexpr bool OK = C::SECOND && MD % M == 0 && SG12 == 1 && ROLES <= THREADS && bytes(2) <= 220 * 1024;
};

template <class C>
__global__ void __launch_bounds__(MvT<C>::THREADS, 1)
k_mv_tiles(const KParams<C> kp, const double* __restrict__ V11, const double* __restrict__ V12,
           const double* __restrict__ v, const double* __restrict__ w, double adt, double* __restrict__ y) {
  using MT = MvT<C>;
  constexpr int NT = C::NT, M = C::M, MD = C::MD, NPE = C::NPE, TPE = C::TPE, NS11 = C::NS11, NS12 = C::NS12,
                R12 = C::R12, SG = MT::SG, G11 = MT::G11, G12 = MT::G12, NPART = MT::NPART, NS = MT::NSTAGE;
  constexpr int NSIN = C::D * C::P + 1;
  constexpr int A0 = C::PH == PH_NS ? 1 : 0;
  // thread roles (one CTA barrier per tile): items of tile i on the lowest
  // ids, the owners of tile i-1 (fixed-order partial sums, y) and the TMA
  // issuer next, the gathers of tile i+1 on the highest ids
  constexpr int NITEM = MT::I11 + MT::I12;
  constexpr int OWN0 = (NITEM + 31) / 32 * 32, ISSUER = OWN0 + (MT::NOUT + 31) / 32 * 32;
  extern __shared__ __align__(16) double smem[];
  __shared__ __align__(8) uint64_t bar[NS];
  double* const ring = smem;
  double* const gath = smem + NS * MT::BUF;
  double* const part = gath + MT::NGB * MT::GBUF;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int64_t ntiles = static_cast<int64_t>(kp.E) * TPE;
  const int64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * per;
  const int64_t t1 = t0 + per < ntiles ? t0 + per : ntiles;
  const int n = t1 > t0 ? static_cast<int>(t1 - t0) : 0;
  // connectivity + element id of tile i, fetched 2 GA tiles ahead (cp.async)
  constexpr int GA = MT::GA, CR = 2 * GA + 1;
  __shared__ __align__(16) int2 sconn[CR][2 * C::D];
  __shared__ int sel[CR];
  __shared__ int gel[MT::GA + 2];  // element id of tile i, for its owners one iteration later
  auto fetch_conn = [&](int i) {  // by threads 0 .. 2D
    if (i >= n) return;
    const int64_t T = t0 + i;
    const int k = static_cast<int>(T / TPE);
    if (tid < 2 * C::D) cp_async8(&sconn[i % CR][tid], kp.conn + static_cast<size_t>(k) * 2 * C::D + tid);
    if (tid == 2 * C::D)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(&sel[i % CR])), "l"(kp.order + k)
                   : "memory");
  };
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&bar[i], 1);
    mbar_fence_init();
  }
  __syncthreads();
  // the issuer streams tile i into ring slot i % NS
  auto issue = [&](int i) {
    const int64_t T = t0 + i;
    double* b = ring + (i % NS) * MT::BUF;
    const int64_t o11 = T * MT::ST11, o12 = T * MT::ST12;
    const unsigned by11 = static_cast<unsigned>(8 * ((MT::ST11 + (o11 & 1) + 1) & ~1));
    const unsigned by12 = static_cast<unsigned>(8 * ((MT::ST12 + (o12 & 1) + 1) & ~1));
    mbar_expect_tx(&bar[i % NS], by11 + by12);
    tma_load_1d_once(b, V11 + (o11 & ~int64_t(1)), by11, &bar[i % NS]);
    tma_load_1d_once(b + MT::BUF11, V12 + (o12 & ~int64_t(1)), by12, &bar[i % NS]);
  };
  // v / w of every (slot, row) column node of tile i -> gather buffer i % NGB
  // (its connectivity is in sconn[i % CR] already); highest thread ids
  auto gather = [&](int i) {
    if (i >= n) return;
    const int64_t T = t0 + i;
    const int k = static_cast<int>(T / TPE), s = static_cast<int>(T - static_cast<int64_t>(k) * TPE);
    const int2* cn = sconn[i % CR];
    const size_t e = static_cast<size_t>(sel[i % CR]);
    double* gb = gath + (i % MT::NGB) * MT::GBUF;
    if (tid == nthr - 1) gel[i % (MT::GA + 2)] = static_cast<int>(e);
    for (int u = nthr - 1 - tid; u < MT::NG; u += nthr) {
      const bool is11 = u < NS11 * NT;
      const int u2 = is11 ? u : u - NS11 * NT;
      const int bg = is11 ? 0 : u2 % (MD / M);
      const int sr = is11 ? u2 : u2 / (MD / M);
      const int slot = sr / NT, r = sr - slot * NT;
      const int64_t col = slot_col_c<C, NSIN>(cn, e, s * NT + r, slot, is11 ? 0 : 1);
      double* dst = is11 ? gb + (slot * NT + r) * M : gb + MT::GX + (slot * NT + r) * MD + bg * M;
      if (col < 0) {
#pragma unroll
        for (int c = 0; c < M; ++c) dst[c] = 0.0;
      } else {
        const double* src = is11 ? v + col * M : w + col * MD + bg * M;
#pragma unroll
        for (int c = 0; c < M; ++c) cp_async8(dst + c, src + c);
      }
    }
  };
  // owners of tile i: fixed-order sums of its partials, y = v - adt (K11 v + K12 w)
  auto owners = [&](int i) {
    const int o = tid - OWN0;
    const int64_t T = t0 + i;
    const int k = static_cast<int>(T / TPE), s = static_cast<int>(T - static_cast<int64_t>(k) * TPE);
    const int a = o % M;
    const double* q = part + (i & 1) * MT::PART + o * NPART;
    double acc = 0.0;
#pragma unroll
    for (int g = 0; g < G11; ++g) acc += q[g];
    if (a >= A0) {
#pragma unroll
      for (int g = 0; g < G12; ++g) acc += q[G11 + g];
    }
    const size_t yo = (static_cast<size_t>(gel[i % (MT::GA + 2)]) * NPE + s * NT) * M + o;
    y[yo] = __ldg(v + yo) - adt * acc;
  };
  if (tid == ISSUER)
    for (int i = 0; i < NS && i < n; ++i) issue(i);
  // prologue: connectivity of tiles 0 .. 2GA-1, gathers of tiles 0 .. GA-1
  // (one cp.async group each; gather j's group fetches the connectivity of j + 2GA)
  for (int j = 0; j < 2 * GA; ++j) fetch_conn(j);
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  for (int j = 0; j < GA; ++j) {
    gather(j);
    fetch_conn(j + 2 * GA);
    cp_async_commit();
  }
  for (int i = 0; i < n; ++i) {
    const int64_t T = t0 + i;
    asm volatile("cp.async.wait_group %0;\n" ::"n"(GA - 1) : "memory");  // gather(i)'s group is complete
    __syncthreads();  // gathers of tile i visible; items and owners of the previous iteration done
    if (tid < NITEM) {
      const double* b11 = ring + (i % NS) * MT::BUF + ((T * MT::ST11) & 1);
      const double* b12 = ring + (i % NS) * MT::BUF + MT::BUF11 + ((T * MT::ST12) & 1);
      const double* gx = gath + (i % MT::NGB) * MT::GBUF;
      const double* gw = gx + MT::GX;
      double* pp = part + (i & 1) * MT::PART;
      mbar_wait(&bar[i % NS], (i / NS) & 1);
      const int it = tid;
      if (it < MT::I11) {
        // K11 item (slot group g, component a, row r)
        const int r = it % NT, a = (it / NT) % M, g = it / (NT * M);
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < SG; ++j) {
          const int slot = g * SG + j;
          if (slot >= NS11) break;
          const double* kv = b11 + ((slot * M + a) * NT + r) * M;
          const double* xv = gx + (slot * NT + r) * M;
#pragma unroll
          for (int c = 0; c < M; ++c) acc += kv[c] * xv[c];
        }
        pp[(r * M + a) * NPART + g] = acc;
      } else {
        // K12 item (slot g, stored row a', row r)
        const int i2 = it - MT::I11;
        const int r = i2 % NT, ap = (i2 / NT) % R12, g = i2 / (NT * R12);
        double acc = 0.0;
        const double* kv = b12 + ((g * R12 + ap) * NT + r) * MD;
        const double* wv = gw + (g * NT + r) * MD;
#pragma unroll
        for (int c = 0; c < MD; ++c) acc += kv[c] * wv[c];
        pp[(r * M + ap + A0) * NPART + G11 + g] = acc;
      }
    } else if (tid >= OWN0 && tid < OWN0 + MT::NOUT) {
      if (i > 0) owners(i - 1);
    } else if (tid == ISSUER) {
      // ring slot (i - 1) % NS was consumed before this iteration's barrier
      if (i > 0 && i - 1 + NS < n) issue(i - 1 + NS);
    }
    gather(i + GA);  // in flight while tiles i .. i+GA-1 compute
    fetch_conn(i + 3 * GA);
    cp_async_commit();
  }
  __syncthreads();
  if (n > 0 && tid >= OWN0 && tid < OWN0 + MT::NOUT) owners(n - 1);
}

// y = K12 w  (w: m*D per node); one thread per (row, stored row a')
template <class C>
__global__ void __launch_bounds__(128)
k_spmv12(const KParams<C> kp, const double* __restrict__ V12, const double* __restrict__ w,
         double* __restrict__ y) {
  constexpr int M = C::M, NT = C::NT, NPE = C::NPE, MD = C::MD, R12 = C::R12;
  constexpr int A0 = C::PH == PH_NS ? 1 : 0;
  const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nrows = static_cast<int64_t>(kp.E) * NPE;
  const int lane = static_cast<int>(gid & 31);
  const int64_t wg = gid >> 5;
  const int a = static_cast<int>(wg % M);
  const int64_t row = (wg / M) * 32 + lane;
  if (row >= nrows) return;
  const int64_t T = row / NT;
  const int r = static_cast<int>(row - T * NT);
  const int k = static_cast<int>(T / C::TPE);
  const int s = static_cast<int>(T - static_cast<int64_t>(k) * C::TPE);
  const int nd = s * NT + r;
  const size_t e = __ldg(kp.order + k);
  double acc = 0.0;
  if (a >= A0) {
    const double* vq = V12 + T * C::NS12 * NT * C::B12 + (static_cast<size_t>(a - A0) * NT + r) * MD;
#pragma unroll
    for (int slot = 0; slot < C::NS12; ++slot) {
      const int64_t col = slot_col<C, C::D * C::P + 1>(kp, k, e, nd, slot, 1);
      if (col < 0) continue;
      const double* vp = vq + static_cast<size_t>(slot) * NT * C::B12;
#pragma unroll
      for (int b = 0; b < MD; ++b) acc += __ldg(vp + b) * __ldg(w + col * MD + b);
    }
  }
  (void)R12;
  y[(e * NPE + nd) * M + a] = acc;
}

// w = K21 v  (w[(node*M + c)*D + d] = sum_slot K21[slot][d] v[col][c]); one thread per row
template <class C>
__global__ void __launch_bounds__(128)
k_spmv21(const KParams<C> kp, const double* __restrict__ V21, const double* __restrict__ v,
         double* __restrict__ w) {
  constexpr int M = C::M, NT = C::NT, NPE = C::NPE, D = C::D;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nrows = static_cast<int64_t>(kp.E) * NPE;
  if (row >= nrows) return;
  const int64_t T = row / NT;
  const int r = static_cast<int>(row - T * NT);
  const int k = static_cast<int>(T / C::TPE);
  const int s = static_cast<int>(T - static_cast<int64_t>(k) * C::TPE);
  const int nd = s * NT + r;
  const size_t e = __ldg(kp.order + k);
  double acc[M][D];
#pragma unroll
  for (int c = 0; c < M; ++c)
#pragma unroll
    for (int d = 0; d < D; ++d) acc[c][d] = 0.0;
  const double* vb = V21 + (T * C::NS12 * NT + r) * D;
#pragma unroll
  for (int slot = 0; slot < C::NS12; ++slot) {
    const int64_t col = slot_col<C, C::D * C::P + 1>(kp, k, e, nd, slot, 2);
    if (col < 0) continue;
    double kv[D];
#pragma unroll
    for (int d = 0; d < D; ++d) kv[d] = __ldg(vb + static_cast<size_t>(slot) * NT * D + d);
#pragma unroll
    for (int c = 0; c < M; ++c) {
      const double xv = __ldg(v + col * M + c);
#pragma unroll
      for (int d = 0; d < D; ++d) acc[c][d] += kv[d] * xv;
    }
  }
  if (C::HAS_INV && kp.noslip)
    k21_wall_terms<C>(kp, k, nd, [&](int end, const double* cf) {
      const double x0 = __ldg(v + (e * NPE + end) * M), x1 = __ldg(v + (e * NPE + end) * M + M - 1);
#pragma unroll
      for (int d = 0; d < D; ++d) {
        acc[0][d] += cf[d] * x0;
        acc[M - 1][d] += cf[d] * x1;
      }
    });
  const size_t wo = (e * NPE + nd) * M * D;
#pragma unroll
  for (int c = 0; c < M; ++c)
#pragma unroll
    for (int d = 0; d < D; ++d) w[wo + c * D + d] = acc[c][d];
}

// ===================================================== block-Jacobi preconditioner
// (PAPER.md:725-740).  A~ equals A = K11 + K12 K21
// on the block-diagonal Line-DG pattern (row and column node in the same
// element and on a common coordinate line), zero elsewhere; the product's
// entries that land on the pattern are summed over every middle node,
// neighbour elements included.  One CTA per element: the element block of
// I - alpha_dt A~ is gathered from the block-row store into shared memory,
// LU-factorised with partial pivoting (the oracle's pivot rule: the first
// largest |a_ik|), and written column-major with its pivots.
// INV (runtime mode ldg_set_precond_mode): the build also forms the explicit
// block inverse from the LU factors, so the apply is a dense, dependency-free
// block matvec streaming the factors at HBM rate instead of 2 NE dependent
// solve steps (measured C2: apply 0.49 -> 0.22 ms, build 11 -> 43 ms).
template <class C, bool INV_ = false>
struct PcCfg {
  static constexpr int NE = C::NPE * C::M;  // unknowns per element
  static constexpr int LDM = NE | 1;        // odd row stride (shared-memory banks)
  static constexpr bool OK = NE <= 128;
  static constexpr bool INV = INV_;
  static constexpr int LDX = NE | 1;        // inverse columns in shared memory (odd stride)
  static constexpr int THREADS = 256;
  static constexpr size_t smem() { return sizeof(double) * (NE * LDM + (INV ? NE * LDX : 0)) + sizeof(int) * NE; }
};

template <class C>
__device__ __forceinline__ bool pc_on_line(int a, int b) {
  int same = 0;
#pragma unroll
  for (int d = 0; d < C::D; ++d) {
    same += (a % C::NP) == (b % C::NP);
    a /= C::NP;
    b /= C::NP;
  }
  return same >= C::D - 1;
}

template <class C, bool INV>
__global__ void __launch_bounds__(PcCfg<C>::THREADS)
k_pc_build(const KParams<C> kp, const double* __restrict__ K11, const double* __restrict__ K12,
           const double* __restrict__ K21, double adt, double* __restrict__ LUc, int32_t* __restrict__ piv,
           int* __restrict__ bad) {
  using PC = PcCfg<C, INV>;
  constexpr int NE = PC::NE, LDM = PC::LDM, M = C::M, NPE = C::NPE, NT = C::NT, D = C::D, MD = C::MD,
                NS11 = C::NS11, NS12 = C::NS12, R12 = C::R12, NSIN = C::D * C::P + 1;
  constexpr int A0 = C::PH == PH_NS ? 1 : 0;
  extern __shared__ __align__(16) double Ms[];
  int* const spv = reinterpret_cast<int*>(Ms + NE * LDM + (PC::INV ? NE * PC::LDX : 0));  // pivot sequence
  __shared__ int spiv;
  __shared__ int sbad;
  const int k = blockIdx.x, tid = threadIdx.x, nthr = blockDim.x;
  const size_t e = kp.order[k];
  for (int x = tid; x < NE * LDM; x += nthr) Ms[x] = 0.0;
  if (tid == 0) sbad = 0;
  __syncthreads();
  // K11: the in-element line slots (each (row, column) node pair once)
  for (int w = tid; w < NPE * NSIN * M * M; w += nthr) {
    const int b = w % M, a = (w / M) % M, rest = w / (M * M), slot = rest % NSIN, nd = rest / NSIN;
    const int64_t col = slot_col<C, NSIN>(kp, k, e, nd, slot, 0);
    const int cl = static_cast<int>(col - static_cast<int64_t>(e) * NPE);
    const size_t T = static_cast<size_t>(k) * C::TPE + nd / NT;
    const double v = K11[(((T * NS11 + slot) * M + a) * NT + nd % NT) * M + b];
    Ms[(nd * M + a) * LDM + cl * M + b] = v;
  }
  __syncthreads();
  if (C::SECOND) {
    // K12 K21 on the pattern: every (row, K12 slot) path through its middle
    // node.  One owner thread per (row node, row component, column component):
    // it walks the paths in a fixed order and is the only writer of its
    // entries, so the sums are deterministic (no atomics).
    for (int w = tid; w < NPE * R12 * M; w += nthr) {
      const int b = w % M, ap = (w / M) % R12, nd = w / (M * R12);
      const size_t T12 = static_cast<size_t>(k) * C::TPE + nd / NT;
      for (int s12 = 0; s12 < NS12; ++s12) {
        const int64_t mid = slot_col<C, NSIN>(kp, k, e, nd, s12, 1);
        if (mid < 0) continue;
        const int em = static_cast<int>(mid / NPE), ndm = static_cast<int>(mid - static_cast<int64_t>(em) * NPE);
        const int km = __ldg(kp.inv_order + em);
        const size_t T21 = static_cast<size_t>(km) * C::TPE + ndm / NT;
        double k12[D];
#pragma unroll
        for (int d = 0; d < D; ++d)
          k12[d] = __ldg(K12 + (((T12 * NS12 + s12) * R12 + ap) * NT + nd % NT) * MD + b * D + d);
        for (int s21 = 0; s21 < NS12; ++s21) {
          const int64_t col = slot_col<C, NSIN>(kp, km, static_cast<size_t>(em), ndm, s21, 2);
          if (col < 0 || col / NPE != static_cast<int64_t>(e)) continue;
          const int cl = static_cast<int>(col - static_cast<int64_t>(e) * NPE);
          if (!pc_on_line<C>(nd, cl)) continue;
          double sum = 0.0;
#pragma unroll
          for (int d = 0; d < D; ++d) sum += k12[d] * __ldg(K21 + ((T21 * NS12 + s21) * NT + ndm % NT) * D + d);
          Ms[(nd * M + ap + A0) * LDM + cl * M + b] += sum;
        }
        if (C::HAS_INV && kp.noslip && em == static_cast<int>(e) && (b == 0 || b == M - 1))
          k21_wall_terms<C>(kp, km, ndm, [&](int end, const double* cf) {  // density and energy columns
            if (!pc_on_line<C>(nd, end)) return;
            double sum = 0.0;
#pragma unroll
            for (int d = 0; d < D; ++d) sum += k12[d] * cf[d];
            Ms[(nd * M + ap + A0) * LDM + end * M + b] += sum;
          });
      }
    }
    __syncthreads();
  }
  for (int x = tid; x < NE * NE; x += nthr) {
    const int i = x / NE, j = x - i * NE;
    Ms[i * LDM + j] = (i == j ? 1.0 : 0.0) - adt * Ms[i * LDM + j];
  }
  __syncthreads();
  // LU with partial pivoting
  for (int kk = 0; kk < NE; ++kk) {
    if (tid < 32) {
      double best = -1.0;
      int bi = kk;
      for (int i = kk + tid; i < NE; i += 32) {
        const double v = fabs(Ms[i * LDM + kk]);
        if (v > best) {
          best = v;
          bi = i;
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double ob = __shfl_down_sync(0xffffffffu, best, off);
        const int oi = __shfl_down_sync(0xffffffffu, bi, off);
        if (ob > best || (ob == best && oi < bi)) {
          best = ob;
          bi = oi;
        }
      }
      if (tid == 0) {
        spiv = bi;
        piv[static_cast<size_t>(k) * NE + kk] = bi;
        spv[kk] = bi;
        if (!(best > 0.0)) sbad = 1;
      }
    }
    __syncthreads();
    const int pr = spiv;
    if (pr != kk)
      for (int j = tid; j < NE; j += nthr) {
        const double t = Ms[kk * LDM + j];
        Ms[kk * LDM + j] = Ms[pr * LDM + j];
        Ms[pr * LDM + j] = t;
      }
    __syncthreads();
    const double ip = 1.0 / Ms[kk * LDM + kk];
    for (int i = kk + 1 + tid; i < NE; i += nthr) Ms[i * LDM + kk] *= ip;
    __syncthreads();
    // trailing update: warps over rows, lanes over columns (no per-entry
    // integer division; the row multiplier stays in a register)
    {
      const int ty = tid >> 5, tx = tid & 31, TY = nthr >> 5;
      for (int i = kk + 1 + ty; i < NE; i += TY) {
        const double lik = Ms[i * LDM + kk];
        for (int j = kk + 1 + tx; j < NE; j += 32) Ms[i * LDM + j] -= lik * Ms[kk * LDM + j];
      }
    }
    __syncthreads();
  }
  if (tid == 0 && sbad) atomicCAS(bad, -1, static_cast<int>(e));
  double* out = LUc + static_cast<size_t>(k) * NE * NE;
  if (PC::INV) {
    // X = A^-1 from P A = L U: X = U^-1 L^-1 P, all columns at once (row-major
    // X[i][j]); per column the operation order is that of a forward / back
    // substitution of P e_j (the oracle's lo_precond_build does the same)
    double* X = Ms + NE * LDM;
    __shared__ int sperm[128];
    if (tid == 0) {
      for (int i = 0; i < NE; ++i) sperm[i] = i;
      for (int kk = 0; kk < NE; ++kk) {
        const int p = spv[kk];
        const int t = sperm[kk];
        sperm[kk] = sperm[p];
        sperm[p] = t;
      }
    }
    __syncthreads();
    for (int x = tid; x < NE * NE; x += nthr) {
      const int i = x / NE, j = x - i * NE;
      X[i * PC::LDX + j] = sperm[i] == j ? 1.0 : 0.0;
    }
    __syncthreads();
    for (int kk = 0; kk < NE - 1; ++kk) {  // unit lower
      const int rem = NE - kk - 1;
      for (int x = tid; x < rem * NE; x += nthr) {
        const int i = kk + 1 + x / NE, j = x % NE;
        X[i * PC::LDX + j] -= Ms[i * LDM + kk] * X[kk * PC::LDX + j];
      }
      __syncthreads();
    }
    for (int kk = NE - 1; kk >= 0; --kk) {  // upper
      for (int j = tid; j < NE; j += nthr) X[kk * PC::LDX + j] = X[kk * PC::LDX + j] / Ms[kk * LDM + kk];
      __syncthreads();
      for (int x = tid; x < kk * NE; x += nthr) {
        const int i = x / NE, j = x % NE;
        X[i * PC::LDX + j] -= Ms[i * LDM + kk] * X[kk * PC::LDX + j];
      }
      __syncthreads();
    }
    for (int x = tid; x < NE * NE; x += nthr) {
      const int j = x / NE, i = x - j * NE;
      out[x] = X[i * PC::LDX + j];  // column-major inverse
    }
    return;
  }
  for (int x = tid; x < NE * NE; x += nthr) {
    const int j = x / NE, i = x - j * NE;
    out[x] = Ms[i * LDM + j];  // column-major
  }
}

// z = (I - alpha_dt A~)^-1 r, one warp per element: row interchanges, then
// column-oriented unit-lower and upper triangular solves on coalesced column
// loads of the element's LU factors.
template <class C, bool INV>
__global__ void __launch_bounds__(128)
k_pc_apply(const KParams<C> kp, const double* __restrict__ LUc, const int32_t* __restrict__ piv,
           const double* __restrict__ r, double* __restrict__ z) {
  using PC = PcCfg<C, INV>;
  constexpr int NE = PC::NE;
  __shared__ double zs[4][NE];
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = blockIdx.x * 4 + wl;
  if (k >= kp.E) return;
  const size_t e = __ldg(kp.order + k);
  double* zw = zs[wl];
  const double* re = r + e * NE;
  for (int i = lane; i < NE; i += 32) zw[i] = re[i];
  __syncwarp();
  if (PC::INV) {
    // z = A^-1 r: lanes over rows, columns streamed (coalesced column loads)
    constexpr int RPL = (NE + 31) / 32;
    double acc[RPL];
#pragma unroll
    for (int q = 0; q < RPL; ++q) acc[q] = 0.0;
    const double* Xc = LUc + static_cast<size_t>(k) * NE * NE;
    for (int j = 0; j < NE; ++j) {
      const double rj = zw[j];
#pragma unroll
      for (int q = 0; q < RPL; ++q) {
        const int i = lane + 32 * q;
        if (i < NE) acc[q] += __ldcs(Xc + j * NE + i) * rj;
      }
    }
    double* ze = z + e * NE;
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
      const int i = lane + 32 * q;
      if (i < NE) ze[i] = acc[q];
    }
    return;
  }
  (void)zw;
  (void)re;
  (void)e;
}

// LU apply: EPW elements per warp (32 / EPW lanes each), so every dependent
// column-load step of the substitutions serves EPW independent chains -- the
// solve is bound by that load latency, not by bandwidth.  Same operations in
// the same order per element as the single-element form.
static constexpr int LDG_PC_EPW = 2;  // measured (C2 apply): 1 -> 0.486 ms, 2 -> 0.407 ms
template <class C>
__global__ void __launch_bounds__(128)
k_pc_apply_lu2(const KParams<C> kp, const double* __restrict__ LUc, const int32_t* __restrict__ piv,
               const double* __restrict__ r, double* __restrict__ z) {
  using PC = PcCfg<C, false>;
  constexpr int NE = PC::NE, EPW = LDG_PC_EPW, LW = 32 / EPW;
  __shared__ double zs[4 * EPW][PC::OK ? NE : 1];  // (unused instantiations stay small)
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31, hl = lane / LW, sl = lane % LW;
  const int kk = (blockIdx.x * 4 + wl) * EPW + hl;
  if ((blockIdx.x * 4 + wl) * EPW >= kp.E) return;  // (whole warp)
  const bool valid = kk < kp.E;
  const int k = valid ? kk : kp.E - 1;  // an idle group shadows the last element (no store)
  const size_t e = __ldg(kp.order + k);
  double* zw = zs[wl * EPW + hl];
  const double* re = r + e * NE;
  for (int i = sl; i < NE; i += LW) zw[i] = re[i];
  __syncwarp();
  if (sl == 0) {
    const int32_t* pv = piv + static_cast<size_t>(k) * NE;
    for (int i = 0; i < NE; ++i) {
      const int p = pv[i];
      const double t = zw[i];
      zw[i] = zw[p];
      zw[p] = t;
    }
  }
  __syncwarp();
  const double* L = LUc + static_cast<size_t>(k) * NE * NE;
  for (int j = 0; j < NE - 1; ++j) {
    const double zj = zw[j];
    for (int i = j + 1 + sl; i < NE; i += LW) zw[i] -= L[j * NE + i] * zj;
    __syncwarp();
  }
  for (int j = NE - 1; j >= 0; --j) {
    if (sl == 0) zw[j] /= L[j * NE + j];
    __syncwarp();
    const double zj = zw[j];
    for (int i = sl; i < j; i += LW) zw[i] -= L[j * NE + i] * zj;
    __syncwarp();
  }
  if (valid) {
    double* ze = z + e * NE;
    for (int i = sl; i < NE; i += LW) ze[i] = zw[i];
  }
}

// ------------------------------------------------ line-ADI preconditioner
// Element blocks above 128 unknowns (3-D p >= 2) keep the line-based sparsity
// the paper calls for in 3-D: I - adt A~ is approximated by
// prod_d (I - adt A~_d), A~_d = the couplings of A~ along direction-d lines
// with the node-diagonal blocks split evenly over the D directions (oracle
// lo_precond_build, same definition).  Each factor is block diagonal over the
// d-lines: one dense NB = (p+1) m block per line, LU with partial pivoting,
// stored column-major [k][d][line][NB x NB] (+ pivots) in processing order.
template <class C>
struct PcLine {
  static constexpr int NB = C::NP * C::M;
  static constexpr int NBB = NB * NB;
  static constexpr int LDB = NB | 1;  // odd row stride in shared memory
  static constexpr int THREADS = 256;
  static constexpr size_t smem() { return sizeof(double) * C::NL * NB * LDB; }
  static constexpr bool OK = NB <= 32 && smem() <= 200 * 1024;
};

// One CTA per (element k, direction d): the d-line blocks of A~ in shared
// memory (K11 line slots; K12 K21 on the pattern by owner threads, fixed
// order), then I - adt A~_d and one warp per line factorises its block.
template <class C>
__global__ void __launch_bounds__(PcLine<C>::THREADS)
k_pc_line_build(const KParams<C> kp, const double* __restrict__ K11, const double* __restrict__ K12,
                const double* __restrict__ K21, double adt, double* __restrict__ LUc, int32_t* __restrict__ piv,
                int* __restrict__ bad) {
  using PL = PcLine<C>;
  constexpr int NB = PL::NB, LDB = PL::LDB, M = C::M, NP = C::NP, NPE = C::NPE, NT = C::NT, NL = C::NL, D = C::D,
                MD = C::MD, NS11 = C::NS11, NS12 = C::NS12, R12 = C::R12, NSIN = C::D * C::P + 1;
  constexpr int A0 = C::PH == PH_NS ? 1 : 0;
  extern __shared__ __align__(16) double B[];  // [line][NB][LDB]
  const int k = blockIdx.x, d = blockIdx.y, tid = threadIdx.x, nthr = blockDim.x;
  const size_t e = kp.order[k];
  for (int x = tid; x < NL * NB * LDB; x += nthr) B[x] = 0.0;
  __syncthreads();
  // K11: for every row node its d-line slots (self block shared by the D directions)
  for (int w = tid; w < NPE * NP * M * M; w += nthr) {
    const int b = w % M, a = (w / M) % M, t2 = (w / (M * M)) % NP, nd = w / (M * M * NP);
    int line, pos;
    line_of<C>(d, nd, line, pos);
    const int slot = t2 == pos ? nd % NP : inel_slot<C>(d, pos, t2);
    const size_t T = static_cast<size_t>(k) * C::TPE + nd / NT;
    double v = K11[(((T * NS11 + slot) * M + a) * NT + nd % NT) * M + b];
    if (t2 == pos) v = v / D;
    B[(line * NB + pos * M + a) * LDB + t2 * M + b] = v;
  }
  __syncthreads();
  if (C::SECOND) {
    // K12 K21 on the pattern (d-line pairs), one owner per (row, a', b)
    for (int w = tid; w < NPE * R12 * M; w += nthr) {
      const int b = w % M, ap = (w / M) % R12, nd = w / (M * R12);
      int line, pos;
      line_of<C>(d, nd, line, pos);
      const size_t T12 = static_cast<size_t>(k) * C::TPE + nd / NT;
      for (int s12 = 0; s12 < NS12; ++s12) {
        const int64_t mid = slot_col<C, NSIN>(kp, k, e, nd, s12, 1);
        if (mid < 0) continue;
        const int em = static_cast<int>(mid / NPE), ndm = static_cast<int>(mid - static_cast<int64_t>(em) * NPE);
        const int km = __ldg(kp.inv_order + em);
        const size_t T21 = static_cast<size_t>(km) * C::TPE + ndm / NT;
        double k12[D];
#pragma unroll
        for (int dd = 0; dd < D; ++dd)
          k12[dd] = __ldg(K12 + (((T12 * NS12 + s12) * R12 + ap) * NT + nd % NT) * MD + b * D + dd);
        auto add = [&](int cl, double sum) {
          int l2, p2;
          line_of<C>(d, cl, l2, p2);
          if (l2 != line) return;  // not on this row's d-line
          B[(line * NB + pos * M + ap + A0) * LDB + p2 * M + b] += cl == nd ? sum / D : sum;
        };
        for (int s21 = 0; s21 < NS12; ++s21) {
          const int64_t col = slot_col<C, NSIN>(kp, km, static_cast<size_t>(em), ndm, s21, 2);
          if (col < 0 || col / NPE != static_cast<int64_t>(e)) continue;
          double sum = 0.0;
#pragma unroll
          for (int dd = 0; dd < D; ++dd) sum += k12[dd] * __ldg(K21 + ((T21 * NS12 + s21) * NT + ndm % NT) * D + dd);
          add(static_cast<int>(col - static_cast<int64_t>(e) * NPE), sum);
        }
        if (C::HAS_INV && kp.noslip && em == static_cast<int>(e) && (b == 0 || b == M - 1))
          k21_wall_terms<C>(kp, km, ndm, [&](int end, const double* cf) {  // density and energy columns
            double sum = 0.0;
#pragma unroll
            for (int dd = 0; dd < D; ++dd) sum += k12[dd] * cf[dd];
            add(end, sum);
          });
      }
    }
    __syncthreads();
  }
  for (int x = tid; x < NL * NB * NB; x += nthr) {
    const int j = x % NB, i = (x / NB) % NB, l = x / (NB * NB);
    double* p = &B[(l * NB + i) * LDB + j];
    *p = (i == j ? 1.0 : 0.0) - adt * *p;
  }
  __syncthreads();
  // one warp per line block: LU with partial pivoting (first maximum, as the oracle)
  const int wid = tid >> 5, lane = tid & 31;
  for (int l = wid; l < NL; l += nthr / 32) {
    double* A = B + l * NB * LDB;
    int32_t* pv = piv + ((static_cast<size_t>(k) * D + d) * NL + l) * NB;
    for (int kk = 0; kk < NB; ++kk) {
      double best = -1.0;
      int bi = kk;
      for (int i = kk + lane; i < NB; i += 32) {
        const double v = fabs(A[i * LDB + kk]);
        if (v > best) {
          best = v;
          bi = i;
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double ob = __shfl_down_sync(0xffffffffu, best, off);
        const int oi = __shfl_down_sync(0xffffffffu, bi, off);
        if (ob > best || (ob == best && oi < bi)) {
          best = ob;
          bi = oi;
        }
      }
      bi = __shfl_sync(0xffffffffu, bi, 0);
      best = __shfl_sync(0xffffffffu, best, 0);
      if (lane == 0) pv[kk] = bi;
      if (!(best > 0.0)) {
        if (lane == 0) atomicCAS(bad, -1, static_cast<int>(e));
        break;
      }
      if (bi != kk)
        for (int j = lane; j < NB; j += 32) {
          const double t = A[kk * LDB + j];
          A[kk * LDB + j] = A[bi * LDB + j];
          A[bi * LDB + j] = t;
        }
      __syncwarp();
      const double ip = 1.0 / A[kk * LDB + kk];
      for (int i = kk + 1 + lane; i < NB; i += 32) A[i * LDB + kk] *= ip;
      __syncwarp();
      for (int x = lane; x < (NB - kk - 1) * (NB - kk - 1); x += 32) {
        const int i = kk + 1 + x / (NB - kk - 1), j = kk + 1 + x % (NB - kk - 1);
        A[i * LDB + j] -= A[i * LDB + kk] * A[kk * LDB + j];
      }
      __syncwarp();
    }
    // column-major store: lane i of a solve step reads column j contiguously
    double* out = LUc + ((static_cast<size_t>(k) * D + d) * NL + l) * PL::NBB;
    for (int x = lane; x < NB * NB; x += 32) {
      const int j = x / NB, i = x - j * NB;
      out[x] = A[i * LDB + j];
    }
  }
}

// z = (I - adt A~_{D-1})^-1 ... (I - adt A~_0)^-1 r: one CTA per element, the
// element's vector in shared memory, one warp per line solve (lane i holds
// entry i of the line vector; NB <= 32), directions in sequence.
template <class C>
__global__ void __launch_bounds__(256)
k_pc_line_apply(const KParams<C> kp, const double* __restrict__ LUc, const int32_t* __restrict__ piv,
                const double* __restrict__ r, double* __restrict__ z) {
  using PL = PcLine<C>;
  constexpr int NB = PL::NB, M = C::M, NPE = C::NPE, NL = C::NL, D = C::D, NE = NPE * M;
  __shared__ double zs[PL::OK ? NE : 1];
  const int k = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const size_t e = __ldg(kp.order + k);
  for (int i = tid; i < NE; i += blockDim.x) zs[i] = r[e * NE + i];
  __syncthreads();
  for (int d = 0; d < D; ++d) {
    for (int l = wid; l < NL; l += nw) {
      const size_t blk = (static_cast<size_t>(k) * D + d) * NL + l;
      const double* L = LUc + blk * PL::NBB;
      const int32_t* pv = piv + blk * NB;
      const int t = lane / M, a = lane - t * M;
      const int nd = lane < NB ? node_on_line<C>(d, l, t) : 0;
      double x = lane < NB ? zs[nd * M + a] : 0.0;
      // lane i holds row i of the factors (NB independent coalesced column
      // loads issued up front: the solve below is a register/shuffle chain)
      double row[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) row[j] = lane < NB ? __ldg(L + j * NB + lane) : 1.0;
      int pvl = lane < NB ? __ldg(pv + lane) : lane;
      // row interchanges in order
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        const int p = __shfl_sync(0xffffffffu, pvl, i);
        const double xi = __shfl_sync(0xffffffffu, x, i), xp = __shfl_sync(0xffffffffu, x, p);
        if (lane == i) x = xp;
        else if (lane == p) x = xi;
      }
      // forward (unit L), column-oriented
#pragma unroll
      for (int j = 0; j < NB - 1; ++j) {
        const double xj = __shfl_sync(0xffffffffu, x, j);
        if (lane > j && lane < NB) x -= row[j] * xj;
      }
      // backward (U)
#pragma unroll
      for (int j = NB - 1; j >= 0; --j) {
        if (lane == j) x = x / row[j];
        const double xj = __shfl_sync(0xffffffffu, x, j);
        if (lane < j) x -= row[j] * xj;
      }
      if (lane < NB) zs[nd * M + a] = x;
    }
    __syncthreads();
  }
  for (int i = tid; i < NE; i += blockDim.x) z[e * NE + i] = zs[i];
}

}  // namespace ldg
