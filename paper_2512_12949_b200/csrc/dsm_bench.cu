// DSM (distributed shared memory) bandwidth microbenchmark, the paper's
// Fig. 4/13 measurement redone on sm_100a: every CTA of a cluster pushes
// `chunk` bytes to its right ring neighbour `iters` times with
// cp.async.bulk shared::cta -> shared::cluster (mbarrier complete_tx),
// keeping `depth` transfers in flight.  Reports aggregate bytes/s.
// Used to calibrate dsm.bandwidth[n] of the B200 device profile.
#include <cuda_runtime.h>

#include <string>

#include "../../include/ff_dsm_bench.h"
#include "ptx.cuh"

namespace {

thread_local std::string g_err;

__global__ void __launch_bounds__(128, 1) dsm_push_kernel(int chunk, int depth, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  using namespace ff;
  const uint32_t base = smem_u32(smem);
  const uint32_t n = cluster_size();
  const uint32_t me = cluster_rank();
  const uint32_t right = (me + 1) % n, left = (me + n - 1) % n;
  // layout: [depth send slots][depth recv slots][depth full bars][depth free bars]
  const uint32_t send0 = base, recv0 = base + depth * chunk;
  const uint32_t full0 = recv0 + depth * chunk, free0 = full0 + 8 * depth;
  if (threadIdx.x == 0) {
    for (int i = 0; i < depth; ++i) {
      mbar_init(full0 + 8 * i, 1);
      mbar_init(free0 + 8 * i, 1);
    }
    fence_mbar_init();
    for (int i = 0; i < depth; ++i) {
      mbar_expect_tx(full0 + 8 * i, chunk);
      mbar_arrive(free0 + 8 * i);
    }
  }
  // touch the send buffer
  for (int i = threadIdx.x * 16; i < depth * chunk; i += blockDim.x * 16)
    st_shared_v4(send0 + i, i, i + 1, i + 2, i + 3);
  fence_proxy_async_smem();
  cluster_sync();
  if (threadIdx.x == 0) {
    // sender role: push i-th chunk into right's slot i % depth when credited
    for (int i = 0; i < iters; ++i) {
      const int s = i % depth;
      mbar_wait_cluster(free0 + 8 * s, (i / depth) & 1);
      dsm_bulk_push(mapa(recv0 + s * chunk, right), send0 + s * chunk, chunk, mapa(full0 + 8 * s, right));
    }
    bulk_commit();
    bulk_wait_read0();
  } else if (threadIdx.x == 32) {
    // receiver role: consume, re-arm, credit the left neighbour
    for (int i = 0; i < iters; ++i) {
      const int s = i % depth;
      mbar_wait_cluster(full0 + 8 * s, (i / depth) & 1);
      mbar_expect_tx(full0 + 8 * s, chunk);
      mbar_arrive_remote(mapa(free0 + 8 * s, left));
    }
  }
  __syncthreads();
  cluster_sync();
}

}  // namespace

extern "C" {

const char* ff_dsm_last_error(void) { return g_err.c_str(); }

int ff_dsm_push_bench(int cluster, int chunk_bytes, int depth, int iters, int num_clusters, float* ms_out) {
  const int smem = 2 * depth * chunk_bytes + 16 * depth + 64;
  if (smem > 232448) {
    g_err = "buffers exceed shared memory";
    return 5;
  }
  cudaError_t e = cudaFuncSetAttribute(dsm_push_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(dsm_push_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) {
    g_err = cudaGetErrorString(e);
    return 4;
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(cluster * num_clusters);
  lc.blockDim = dim3(128);
  lc.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  e = cudaLaunchKernelEx(&lc, dsm_push_kernel, chunk_bytes, depth, 4);  // warm-up
  cudaEventRecord(a);
  if (e == cudaSuccess) e = cudaLaunchKernelEx(&lc, dsm_push_kernel, chunk_bytes, depth, iters);
  cudaEventRecord(b);
  if (e == cudaSuccess) e = cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (e != cudaSuccess) {
    g_err = cudaGetErrorString(e);
    return 4;
  }
  *ms_out = ms;
  return 0;
}

int ff_max_active_clusters(int cluster, int smem_bytes, int* out) {
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(cluster);
  lc.blockDim = dim3(256);
  lc.dynamicSmemBytes = smem_bytes;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  cudaFuncSetAttribute(dsm_push_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  cudaFuncSetAttribute(dsm_push_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaError_t e = cudaOccupancyMaxActiveClusters(out, dsm_push_kernel, &lc);
  if (e != cudaSuccess) {
    g_err = cudaGetErrorString(e);
    return 4;
  }
  return 0;
}

}  // extern "C"
