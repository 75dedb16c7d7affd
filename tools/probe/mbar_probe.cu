// Minimal reproduction for compute-sanitizer synccheck: per-warp mbarrier
// initialised by lane 0 (inline PTX, as assemble_body.cuh), one bulk copy
// completing on it, all lanes waiting on the phase.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const double* src, double* out, int variant) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* buf = sm + w * 34;
  uint64_t* mb = reinterpret_cast<uint64_t*>(buf + 32);
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mb)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (variant == 1) __syncthreads(); else __syncwarp();
  if (lane == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)), "r"(256u) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(buf)), "l"(src + w * 32), "r"(256u), "r"(smem_u32(mb)) : "memory");
  }
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n"
               ::"r"(smem_u32(mb)), "r"(0) : "memory");
  out[blockIdx.x * blockDim.x + threadIdx.x] = buf[lane];
}
int main() {
  double *s, *o;
  cudaMalloc(&s, 1 << 16); cudaMalloc(&o, 1 << 16);
  cudaMemset(s, 0, 1 << 16);
  for (int v = 0; v < 2; ++v) {
    k<<<2, 128, 4 * 34 * 8>>>(s, o, v);
    printf("variant %d: %s\n", v, cudaGetErrorString(cudaDeviceSynchronize()));
  }
  return 0;
}
