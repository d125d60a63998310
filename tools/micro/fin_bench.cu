// Standalone microbenchmark: summing S slab partials [S][N] -> [N] (the
// narrow-grad finalize), three thread mappings.  nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 fin_bench.cu -o fin_bench
#include <cstdio>
#include <cuda_runtime.h>

__global__ void a_groups(const float* P, int S, long N, float* out) {  // 32 outputs x 8 slab groups
  __shared__ float part[8][33];
  int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  long e = (long)blockIdx.x * 32 + lane;
  float v = 0.f;
  if (e < N)
    for (int s0 = grp; s0 < S; s0 += 64) {
      float q[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) q[u] = s0 + 8 * u < S ? __ldcs(P + (long)(s0 + 8 * u) * N + e) : 0.f;
#pragma unroll
      for (int u = 0; u < 8; ++u) v += q[u];
    }
  part[grp][lane] = v;
  __syncthreads();
  if (grp || e >= N) return;
  float t = part[0][lane];
  for (int g = 1; g < 8; ++g) t += part[g][lane];
  out[e] = t;
}

__global__ void b_thread(const float* P, int S, long N, float* out) {  // one output per thread
  long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= N) return;
  float v = 0.f;
  int s = 0;
  for (; s + 8 <= S; s += 8) {
    float q[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) q[u] = __ldcs(P + (long)(s + u) * N + e);
#pragma unroll
    for (int u = 0; u < 8; ++u) v += q[u];
  }
  for (; s < S; ++s) v += P[(long)s * N + e];
  out[e] = v;
}

template <int SMAX>
__global__ void c_allin(const float* P, int S, long N, float* out) {  // all S loads issued, then summed
  long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= N) return;
  float q[SMAX];
#pragma unroll
  for (int s = 0; s < SMAX; ++s) q[s] = s < S ? P[(long)s * N + e] : 0.f;
  float v = 0.f;
#pragma unroll
  for (int s = 0; s < SMAX; ++s) v += q[s];
  out[e] = v;
}

int main() {
  const int S = 74;
  const long N = 4096 * 11;
  float *P, *o;
  cudaMalloc(&P, (size_t)S * N * 4);
  cudaMalloc(&o, N * 4);
  cudaMemset(P, 0, (size_t)S * N * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int variant = 0; variant < 3; ++variant) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      for (int i = 0; i < 20; ++i) {
        if (variant == 0) a_groups<<<(N + 31) / 32, 256>>>(P, S, N, o);
        if (variant == 1) b_thread<<<(N + 255) / 256, 256>>>(P, S, N, o);
        if (variant == 2) c_allin<80><<<(N + 127) / 128, 128>>>(P, S, N, o);
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("variant %d: %.2f us per launch (%.0f GB/s)\n", variant, ms * 1e3 / 20, S * N * 4 / (ms * 1e-3 / 20) / 1e9);
    }
  }
  return 0;
}
