// DMMA / DFMA dependent-issue latency on one warp (clock64 per instruction)
// for 1..8 independent accumulator chains: tells how many independent DMMA
// chains a warp needs in flight to keep the FP64 pipe busy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_latency tools/dmma_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int IT = 1024;

__device__ __forceinline__ void mma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int N>
__global__ void lat_dmma(double* out, long long* cyc, double a, double b) {
  double c[N][2];
#pragma unroll
  for (int i = 0; i < N; ++i) c[i][0] = c[i][1] = i;
  __syncwarp();
  long long t0 = clock64();
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < N; ++i) mma(c[i][0], c[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) s += c[i][0] + c[i][1];
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  if (s == 1.2345) out[0] = s;
}

template <int N>
__global__ void lat_dfma(double* out, long long* cyc, double a, double b) {
  double c[N];
#pragma unroll
  for (int i = 0; i < N; ++i) c[i] = i;
  long long t0 = clock64();
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < N; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) s += c[i];
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  if (s == 1.2345) out[0] = s;
}

template <int N>
void run(double* o, long long* c) {
  long long h;
  lat_dmma<N><<<1, 32>>>(o, c, 1.0000001, 1e-9);
  lat_dmma<N><<<1, 32>>>(o, c, 1.0000001, 1e-9);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("dmma chains=%d cycles/instr=%.2f  cycles/chain-step=%.2f\n", N, double(h) / (IT * N), double(h) / IT);
  lat_dfma<N><<<1, 32>>>(o, c, 1.0000001, 1e-9);
  lat_dfma<N><<<1, 32>>>(o, c, 1.0000001, 1e-9);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("dfma chains=%d cycles/instr=%.2f  cycles/chain-step=%.2f\n", N, double(h) / (IT * N), double(h) / IT);
}

int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 8);
  cudaMalloc(&c, 8);
  run<1>(o, c);
  run<2>(o, c);
  run<3>(o, c);
  run<4>(o, c);
  run<6>(o, c);
  run<8>(o, c);
  return 0;
}
