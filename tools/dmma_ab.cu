// A/B of the line-block contraction of the Jacobian assembly on B200:
//   O[(i,t)][ab] = sum_q cc[i][t][q] * A_q[ab]
// per coordinate line: M = (p+1)^2 = 25 (i,t) pairs (padded to 32), K = n_q = 7
// (padded to 8), N = 85 block entries (K11 25 + K12 60, padded to 88) -- the
// C5 (3-D Navier-Stokes p = 4) shape.  Variant 0: FFMA, one thread per output
// entry (the kernels' scheme).  Variant 1: DMMA, mma.sync.m8n8k4 f64 (the
// only fp64 tensor-core instruction on sm_100a; tcgen05 has no f64 kind).
// Inputs in shared memory, results folded into a per-thread checksum so the
// comparison isolates the contraction.  Output: one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int MR = 32, KQ = 8, NN = 88;

__global__ void __launch_bounds__(256) k_ffma(const double* __restrict__ cc, const double* __restrict__ A,
                                             double* __restrict__ out, int lines) {
  __shared__ double scc[MR * KQ];
  __shared__ double sA[8][KQ * NN];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < MR * KQ; i += blockDim.x) scc[i] = cc[i];
  for (int i = lane; i < KQ * NN; i += 32) sA[wid][i] = A[(blockIdx.x * 8 + wid) % 64 * KQ * NN + i];
  __syncthreads();
  double chk = 0.0;
  for (int l = 0; l < lines; ++l) {
    const double s = 1.0 + 1e-3 * l;
    for (int o = lane; o < 25 * 85; o += 32) {
      const int it = o / 85, ab = o - it * 85;
      double v = 0.0;
#pragma unroll
      for (int q = 0; q < 7; ++q) v += scc[it * KQ + q] * sA[wid][q * NN + ab];
      chk += s * v;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = chk;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256) k_dmma(const double* __restrict__ cc, const double* __restrict__ A,
                                             double* __restrict__ out, int lines) {
  __shared__ double scc[MR * KQ];
  __shared__ double sA[8][KQ * NN];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < MR * KQ; i += blockDim.x) scc[i] = cc[i];
  for (int i = lane; i < KQ * NN; i += 32) sA[wid][i] = A[(blockIdx.x * 8 + wid) % 64 * KQ * NN + i];
  __syncthreads();
  // fragments: A (8x4 row) lane -> [lane/4][lane%4]; B (4x8 col) lane -> [lane%4][lane/4];
  // C (8x8) lane -> [lane/4][2(lane%4) + {0,1}]
  double afr[4][2];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) afr[mt][ks] = scc[(mt * 8 + lane / 4) * KQ + ks * 4 + lane % 4];
  double chk = 0.0;
  for (int l = 0; l < lines; ++l) {
    const double s = 1.0 + 1e-3 * l;
#pragma unroll
    for (int nt = 0; nt < NN / 8; ++nt) {
      const double b0 = sA[wid][(lane % 4) * NN + nt * 8 + lane / 4];
      const double b1 = sA[wid][(4 + lane % 4) * NN + nt * 8 + lane / 4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        double d0 = 0.0, d1 = 0.0;
        dmma(d0, d1, afr[mt][0], b0);
        dmma(d0, d1, afr[mt][1], b1);
        chk += s * (d0 + d1);
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = chk;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 4, lines = 2000;
  double *cc, *A, *out;
  cudaMalloc(&cc, MR * KQ * 8);
  cudaMalloc(&A, 64 * KQ * NN * 8);
  cudaMalloc(&out, grid * 256 * 8);
  cudaMemset(cc, 0, MR * KQ * 8);
  cudaMemset(A, 0, 64 * KQ * NN * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double useful = 2.0 * 25 * 85 * 7;  // flops per line (unpadded)
  float ms[2];
  for (int v = 0; v < 2; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (v == 0) k_ffma<<<grid, 256>>>(cc, A, out, lines);
      else k_dmma<<<grid, 256>>>(cc, A, out, lines);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms[v], e0, e1);
    }
  }
  const double nl = double(grid) * 8 * lines;
  printf("{\"shape\": \"per line [25x7]x[7x85] (C5 K11+K12 block entries)\", \"lines\": %.0f, "
         "\"ffma_ms\": %.3f, \"dmma_ms\": %.3f, \"ffma_useful_tflops\": %.2f, \"dmma_useful_tflops\": %.2f, "
         "\"err\": \"%s\"}\n",
         nl, ms[0], ms[1], nl * useful / (ms[0] * 1e-3) / 1e12, nl * useful / (ms[1] * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
