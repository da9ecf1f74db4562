// A/B of the HBM data layout of the state U (and R) for the Line-DG
// residual's access pattern, on B200:
//   AoS  (current)  U[e][node][c]      -- reference GridFunction, field.hpp:8-9
//   SoA  (north_star "line-major structure-of-arrays") U[c][e][node]
// Element records are padded to 16-byte multiples in both layouts (TMA 1-D
// bulk copies need 16-byte sizes and addresses).  Per element the kernel stages the element's state in shared memory (1-D
// TMA bulk copies: one per element in AoS, one per component in SoA), gathers
// the neighbour traces of its 2D faces (one node record of m doubles per line
// end in AoS, m scattered 8-byte loads in SoA -- the neighbour is another,
// randomly numbered element), forms a per-node value from both and writes R in
// the same layout.  Persistent CTAs, two-stage mbarrier ring, random element
// numbering like the configs.  Reports GB/s of the algorithmic bytes
// (U + R + neighbour traces) for the C2 (2-D p=4 m=4) and C5 (3-D p=4 m=5) shapes.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bulk(void* s, const void* g, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   su32(s)), "l"(g), "r"(bytes), "r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void expect(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void waitp(uint64_t* bar, unsigned par) {
  asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(
                   su32(bar)), "r"(par) : "memory");
}

template <int NPE, int M, int NF, int NL, bool SOA>
struct Lay {
  static constexpr int SA = (NPE * M + 1) / 2 * 2;  // AoS element stride (doubles)
  static constexpr int SS = (NPE + 1) / 2 * 2;      // SoA per-component element stride
};
template <int NPE, int M, int NF, int NL, bool SOA>
__global__ void __launch_bounds__(256) k_layout(const double* __restrict__ U, double* __restrict__ R,
                                               const int* __restrict__ nbr, int E) {
  using L = Lay<NPE, M, NF, NL, SOA>;
  constexpr int SA = L::SA, SS = L::SS;
  __shared__ __align__(16) double su[2][SOA ? SS * M : SA];
  __shared__ double snb[NF * NL * M];
  __shared__ __align__(8) uint64_t bar[2];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int e, int b) {
    if (!SOA) {
      expect(&bar[b], SA * 8);
      bulk(su[b], U + (size_t)e * SA, SA * 8, &bar[b]);
    } else {
      expect(&bar[b], SS * M * 8);
      for (int c = 0; c < M; ++c) bulk(su[b] + c * SS, U + ((size_t)c * E + e) * SS, SS * 8, &bar[b]);
    }
  };
  int it = 0;
  if (tid == 0 && (int)blockIdx.x < E) issue(blockIdx.x, 0);
  for (int e = blockIdx.x; e < E; e += gridDim.x, ++it) {
    const int b = it & 1;
    const int en = e + gridDim.x;
    if (tid == 0 && en < E) issue(en, b ^ 1);
    // neighbour traces: NF faces x NL line ends x M components
    for (int w = tid; w < NF * NL * M; w += blockDim.x) {
      const int c = w % M, l = (w / M) % NL, f = w / (M * NL);
      const int ne = nbr[(size_t)e * NF + f];
      const int node = (l * 7 + f) % NPE;  // a face node of the neighbour
      snb[w] = SOA ? U[((size_t)c * E + ne) * SS + node] : U[(size_t)ne * SA + node * M + c];
    }
    waitp(&bar[b], (it >> 1) & 1);
    __syncthreads();
    for (int w = tid; w < NPE * M; w += blockDim.x) {
      const int nd = SOA ? w % NPE : w / M, c = SOA ? w / NPE : w % M;
      const double u = SOA ? su[b][c * SS + nd] : su[b][nd * M + c];
      const double t = snb[((nd % NF) * NL + nd % NL) * M + c];
      const size_t o = SOA ? ((size_t)c * E + e) * SS + nd : (size_t)e * SA + nd * M + c;
      R[o] = 0.5 * u + 0.25 * t;
    }
    __syncthreads();
  }
}

template <int NPE, int M, int NF, int NL>
void run(const char* name, int E) {
  const size_t n = (size_t)E * ((NPE + 1) / 2 * 2) * M + 16;  // the larger padded footprint
  double *U, *R;
  int* nbr;
  cudaMalloc(&U, n * 8);
  cudaMalloc(&R, n * 8);
  cudaMalloc(&nbr, (size_t)E * NF * 4);
  std::vector<int> h((size_t)E * NF);
  std::mt19937 rng(7);
  for (auto& x : h) x = rng() % E;
  cudaMemcpy(nbr, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(U, 0, n * 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 6;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms[2];
  for (int v = 0; v < 2; ++v) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      if (v == 0) k_layout<NPE, M, NF, NL, false><<<grid, 256>>>(U, R, nbr, E);
      else k_layout<NPE, M, NF, NL, true><<<grid, 256>>>(U, R, nbr, E);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms[v], a, b);
    }
  }
  const double bytes = 2.0 * E * NPE * M * 8 + (double)E * NF * NL * M * 8;  // algorithmic (unpadded)
  printf("{\"shape\": \"%s\", \"elements\": %d, \"aos_ms\": %.4f, \"soa_ms\": %.4f, \"aos_GBs\": %.1f, "
         "\"soa_GBs\": %.1f, \"err\": \"%s\"}\n",
         name, E, ms[0], ms[1], bytes / (ms[0] * 1e-3) / 1e9, bytes / (ms[1] * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(U);
  cudaFree(R);
  cudaFree(nbr);
}

int main() {
  run<25, 4, 4, 5>("C2 2-D Euler p=4 (npe 25, m 4)", 16384 * 16);
  run<125, 5, 6, 25>("C5 3-D NS p=4 (npe 125, m 5)", 110592);
  return 0;
}
