// Microbenchmark: L2-resident read bandwidth and cluster DSMEM read bandwidth on sm_100a.
// Informs the K1 design choice (L2-resident workspace vs cluster-resident image).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membw_probe membw_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void l2_read(const float4* __restrict__ a, size_t n, int reps, float4* sink) {
  float4 acc = make_float4(0, 0, 0, 0);
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      float4 v = __ldcg(a + i);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  if (acc.x == 1234.5f) sink[0] = acc;
}

template <int CS>
__global__ void __cluster_dims__(CS, 1, 1) dsmem_read(int reps, float4* sink, int nbytes) {
  extern __shared__ float4 sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int n = nbytes / 16;
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = make_float4(i, 1, 2, 3);
  cl.sync();
  const int me = cl.block_rank();
  float4 acc = make_float4(0, 0, 0, 0);
  for (int r = 0; r < reps; ++r) {
    const int peer = (me + 1 + (r % (CS - 1))) % CS;
    const float4* rs = cl.map_shared_rank(sm, peer);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      float4 v = rs[i];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  cl.sync();
  if (acc.x == 1234.5f) sink[0] = acc;
}

__global__ void smem_read(int reps, float4* sink, int nbytes) {
  extern __shared__ float4 sm[];
  const int n = nbytes / 16;
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = make_float4(i, 1, 2, 3);
  __syncthreads();
  float4 acc = make_float4(0, 0, 0, 0);
  for (int r = 0; r < reps; ++r)
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      float4 v = sm[(i + r) % n];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  if (acc.x == 1234.5f) sink[0] = acc;
}

int main() {
  int dev = 0, nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  float4* sink;
  cudaMalloc(&sink, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (size_t mb : {16, 32, 48, 64, 96, 2048}) {
    size_t bytes = mb << 20, n = bytes / 16;
    float4* a;
    cudaMalloc(&a, bytes);
    cudaMemset(a, 0, bytes);
    int reps = (int)(8192 / mb) > 1 ? (int)(8192 / mb) : 1;
    l2_read<<<nsm * 8, 256>>>(a, n, 1, sink);
    cudaEventRecord(e0);
    l2_read<<<nsm * 8, 256>>>(a, n, reps, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"probe\":\"global_read\",\"MB\":%zu,\"GBps\":%.1f}\n", mb, (double)bytes * reps / ms / 1e6);
    cudaFree(a);
  }
  const int nb = 96 * 1024;
  cudaFuncSetAttribute(dsmem_read<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, nb);
  cudaFuncSetAttribute(dsmem_read<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, nb);
  cudaFuncSetAttribute(dsmem_read<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, nb);
  cudaFuncSetAttribute(smem_read, cudaFuncAttributeMaxDynamicSharedMemorySize, nb);
  const int reps = 200;
  for (int cs : {2, 4, 8}) {
    int grid = (nsm / cs) * cs * 2;
    auto launch = [&]() {
      if (cs == 2) dsmem_read<2><<<grid, 512, nb>>>(reps, sink, nb);
      if (cs == 4) dsmem_read<4><<<grid, 512, nb>>>(reps, sink, nb);
      if (cs == 8) dsmem_read<8><<<grid, 512, nb>>>(reps, sink, nb);
    };
    launch();
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    printf("{\"probe\":\"dsmem_read\",\"cluster\":%d,\"GBps\":%.1f,\"err\":\"%s\"}\n", cs,
           (double)grid * nb * reps / ms / 1e6, cudaGetErrorString(err));
  }
  {
    int grid = nsm * 2;
    smem_read<<<grid, 512, nb>>>(reps, sink, nb);
    cudaEventRecord(e0);
    smem_read<<<grid, 512, nb>>>(reps, sink, nb);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"probe\":\"smem_read\",\"GBps\":%.1f}\n", (double)grid * nb * reps / ms / 1e6);
  }
  return 0;
}
