// FP64 peak microbenchmarks for B200 (sm_100a): DFMA, DMMA (mma.sync f64
// shapes), DFMA+DMMA co-issue, HBM store/copy bandwidth.  Prints one JSON
// object.  These are the roofline denominators for the fp64 assembly kernels
// (MEASURED_PEAKS.json has no fp64 figure).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peaks tools/fp64_peaks.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void dfma_kernel(double* out, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void mma_m8n8k4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma_m16n8k4(double* c, double a0, double a1, double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a0), "d"(a1), "d"(b));
}
__device__ __forceinline__ void mma_m16n8k16(double* c, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
               "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int NACC>
__global__ void dmma_m8n8k4_kernel(double* out, double a, double b) {
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = i; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) mma_m8n8k4(c[i][0], c[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int NACC>
__global__ void dmma_m16n8k4_kernel(double* out, double a, double b) {
  double c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) c[i][j] = j;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) mma_m16n8k4(c[i], a, b, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

template <int NACC>
__global__ void dmma_m16n8k16_kernel(double* out, double a, double b) {
  double c[NACC][4];
  double av[8], bv[4];
#pragma unroll
  for (int j = 0; j < 8; ++j) av[j] = a + j;
#pragma unroll
  for (int j = 0; j < 4; ++j) bv[j] = b + j;
#pragma unroll
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) c[i][j] = j;
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) mma_m16n8k16(c[i], av, bv);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

// DMMA and DFMA interleaved in the same warp: does the FMA pipe run beside DMMA?
__global__ void mixed_kernel(double* out, double a, double b) {
  double c[4][2];
  double x[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) { c[i][0] = 0; c[i][1] = i; }
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) mma_m8n8k4(c[i][0], c[i][1], a, b);
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void store_kernel(double2* dst, size_t n2) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n2; i += stride) dst[i] = make_double2((double)i, 1.0);
}
__global__ void copy_kernel(double2* dst, const double2* src, size_t n2) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n2; i += stride) dst[i] = src[i];
}

template <class F>
float time_ms(F launch, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(e0); cudaEventDestroy(e1);
  return best;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out; CK(cudaMalloc(&out, 64));
  const int threads = 256;
  const int blocks = sms * 8;
  const double nthr = (double)threads * blocks;
  const double nwarps = nthr / 32.0;
  printf("{\n  \"sms\": %d,\n", sms);

  float ms = time_ms([&] { dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7); }, 5);
  printf("  \"dfma_tflops\": %.3f,\n", nthr * ITERS * 8 * 2 / (ms * 1e-3) / 1e12);

  ms = time_ms([&] { dmma_m8n8k4_kernel<4><<<blocks, threads>>>(out, 1e-3, 1e-3); }, 5);
  printf("  \"dmma_m8n8k4_acc4_tflops\": %.3f,\n", nwarps * ITERS * 4 * 256 * 2 / (ms * 1e-3) / 1e12);
  ms = time_ms([&] { dmma_m8n8k4_kernel<8><<<blocks, threads>>>(out, 1e-3, 1e-3); }, 5);
  printf("  \"dmma_m8n8k4_acc8_tflops\": %.3f,\n", nwarps * ITERS * 8 * 256 * 2 / (ms * 1e-3) / 1e12);
  ms = time_ms([&] { dmma_m8n8k4_kernel<4><<<sms * 2, 128>>>(out, 1e-3, 1e-3); }, 5);
  printf("  \"dmma_m8n8k4_acc4_2warps_per_smsp_tflops\": %.3f,\n",
         (sms * 2 * 4.0) * ITERS * 4 * 256 * 2 / (ms * 1e-3) / 1e12);
  ms = time_ms([&] { dmma_m8n8k4_kernel<4><<<sms, 128>>>(out, 1e-3, 1e-3); }, 5);
  printf("  \"dmma_m8n8k4_acc4_1warp_per_smsp_tflops\": %.3f,\n",
         (sms * 4.0) * ITERS * 4 * 256 * 2 / (ms * 1e-3) / 1e12);
  ms = time_ms([&] { dmma_m16n8k4_kernel<4><<<blocks, threads>>>(out, 1e-3, 1e-3); }, 5);
  printf("  \"dmma_m16n8k4_acc4_tflops\": %.3f,\n", nwarps * ITERS * 4 * 512 * 2 / (ms * 1e-3) / 1e12);
  ms = time_ms([&] { dmma_m16n8k16_kernel<4><<<blocks, threads>>>(out, 1e-3, 1e-3); }, 5);
  printf("  \"dmma_m16n8k16_acc4_tflops\": %.3f,\n", nwarps * (ITERS / 4) * 4 * 2048 * 2 / (ms * 1e-3) / 1e12);
  ms = time_ms([&] { mixed_kernel<<<blocks, threads>>>(out, 1e-3, 1e-3); }, 5);
  {
    double fl_mma = nwarps * ITERS * 4 * 256 * 2, fl_fma = nthr * ITERS * 8 * 2;
    printf("  \"mixed_ms\": %.4f,\n  \"mixed_total_tflops\": %.3f,\n", ms, (fl_mma + fl_fma) / (ms * 1e-3) / 1e12);
  }

  size_t bytes = (size_t)8 << 30;
  double2 *a, *b;
  CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
  size_t n2 = bytes / sizeof(double2);
  ms = time_ms([&] { store_kernel<<<sms * 16, 512>>>(a, n2); }, 5);
  printf("  \"hbm_store_gbs\": %.1f,\n", bytes / (ms * 1e-3) / 1e9);
  ms = time_ms([&] { copy_kernel<<<sms * 16, 512>>>(b, a, n2); }, 5);
  printf("  \"hbm_copy_gbs\": %.1f,\n", 2.0 * bytes / (ms * 1e-3) / 1e9);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("  \"clock_khz_attr\": %d\n}\n", clk);
  return 0;
}
