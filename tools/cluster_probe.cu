// Probe for the K1 cluster design: (1) how many clusters of CS CTAs (1 CTA per SM, ~200 KB
// shared memory) can be co-resident; (2) the aggregate DSMEM bandwidth of the all-to-all block
// exchange K1 would do (every CTA bulk-copies one block to every CTA of its cluster per step,
// cp.async.bulk.shared::cluster with mbarrier complete_tx, a cluster barrier per step).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_probe cluster_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa(unsigned a, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ unsigned cta_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

template <int CS>
__global__ void __launch_bounds__(416, 1) xchg(int iters, int blk, float* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm);
  unsigned char* src = sm + 128;
  unsigned char* dst = src + CS * blk;
  const unsigned me = cta_rank();
  for (int i = threadIdx.x; i < CS * blk; i += blockDim.x) src[i] = (unsigned char)(i + me);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  cluster_sync();
  for (int it = 0; it < iters; ++it) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(CS * blk)
                   : "memory");
    }
    cluster_sync();  // every receiver armed and its buffer free
    if (threadIdx.x < CS) {
      const unsigned d = (me + threadIdx.x) % CS;
      const unsigned rdst = mapa(smem_u32(dst + me * blk), d);
      const unsigned rbar = mapa(smem_u32(bar), d);
      asm volatile(
          "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(rdst),
          "r"(smem_u32(src + d * blk)), "r"(blk), "r"(rbar)
          : "memory");
    }
    mbar_wait(smem_u32(bar), it & 1);
    asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  if (threadIdx.x == 0 && dst[7] == 255 && dst[9] == 254) sink[0] = 1.f;
  cluster_sync();
}

template <int CS>
void run(int smem_extra) {
  auto k = xchg<CS>;
  const int blk = 3520;
  size_t smem = 128 + 2 * CS * blk + smem_extra;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (CS > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cfg.blockDim = dim3(416);
  cfg.dynamicSmemBytes = smem;
  cfg.gridDim = dim3(CS * 64);
  int ncl = 0;
  cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, k, &cfg);
  printf("CS=%d smem=%zu: max active clusters %d (%s) -> %d SMs\n", CS, smem, ncl, cudaGetErrorString(e), ncl * CS);
  if (ncl < 1) return;
  cfg.gridDim = dim3(CS * ncl);
  float* sink;
  cudaMalloc(&sink, 4);
  const int iters = 2000;
  cudaLaunchKernelEx(&cfg, k, 10, blk, sink);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaLaunchKernelEx(&cfg, k, iters, blk, sink);
  cudaEventRecord(b);
  e = cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double remote = (double)ncl * CS * (CS - 1) * blk * iters;
  printf("   %s: %d steps in %.3f ms = %.2f us/step; remote DSMEM %.1f GB/s aggregate, %.1f GB/s per SM\n",
         cudaGetErrorString(e), iters, ms, ms * 1e3 / iters, remote / (ms * 1e-3) / 1e9,
         remote / (ms * 1e-3) / 1e9 / (ncl * CS));
  cudaFree(sink);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  printf("%s, %d SMs, smem/block optin %zu\n", p.name, p.multiProcessorCount, p.sharedMemPerBlockOptin);
  run<8>(100000);
  run<16>(100000);
  run<16>(0);
  run<8>(0);
  run<4>(150000);
  return 0;
}
