// Multi-phase variant of mbar_probe.cu: the element-kernel pattern -- lane 0
// re-arms the warp's mbarrier once per element (fence.proxy.async, expect_tx,
// two bulk copies), all lanes wait on the alternating phase.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const double* src, double* out, int iters) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* buf = sm + w * 66;
  uint64_t* mb = reinterpret_cast<uint64_t*>(buf + 64);
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mb)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t phase = 0;
  double acc = 0.0;
  auto issue = [&](int it) {
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)), "r"(512u) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(buf)), "l"(src + (it % 8) * 64), "r"(256u), "r"(smem_u32(mb)) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(buf + 32)), "l"(src + (it % 8) * 64 + 32), "r"(256u), "r"(smem_u32(mb)) : "memory");
    }
  };
  issue(0);
  for (int it = 0; it < iters; ++it) {
    asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n"
                 ::"r"(smem_u32(mb)), "r"(phase) : "memory");
    phase ^= 1u;
    __syncwarp();
    acc += buf[lane] + buf[32 + lane];
    __syncwarp();
    if (it + 1 < iters) issue(it + 1);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  double *s, *o;
  cudaMalloc(&s, 1 << 16); cudaMalloc(&o, 1 << 16);
  cudaMemset(s, 0, 1 << 16);
  k<<<4, 128, 4 * 66 * 8>>>(s, o, 5);
  printf("multi-phase: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
