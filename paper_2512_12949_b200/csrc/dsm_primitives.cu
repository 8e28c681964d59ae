// Test / microbenchmark driver of the DSM communication primitives
// (dsm_primitives.cuh): one fp32 tile per CTA, clusters of G CTAs.
#include <cuda.h>
#include <cuda_runtime.h>

#include <string>

#include "../../include/ff_dsm_bench.h"
#include "dsm_primitives.cuh"

namespace ff {
void dsm_set_error(const char* msg);  // dsm_bench.cu (ff_dsm_last_error)
}

namespace {

enum Op : int { OP_REDUCE_SCATTER = 0, OP_ALL_GATHER = 1, OP_ALL_EXCHANGE_ADD = 2, OP_ALL_EXCHANGE_MUL = 3, OP_SHUFFLE = 4 };

// bytes each CTA's barrier(s) expect per iteration: bar0 / bar1
__device__ __forceinline__ uint32_t expect0(int op, int N, int G) {
  switch (op) {
    case OP_REDUCE_SCATTER:
    case OP_ALL_EXCHANGE_ADD:
      return (uint32_t)((G - 1) * (N / G) * 4);
    case OP_ALL_GATHER:
      return (uint32_t)((G - 1) * (N / G) * 4);
    default:
      return (uint32_t)(N * 4);
  }
}

__global__ void __launch_bounds__(256, 1) dsm_primitive_kernel(int op, const float* in, float* out, int N, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  using namespace ff;
  const int G = (int)cluster_size(), rank = (int)cluster_rank();
  float* const tile_g = reinterpret_cast<float*>(smem);
  float* const recv_g = tile_g + N;
  const uint32_t tile = smem_u32(tile_g), recv = smem_u32(recv_g);
  const int recv_floats = (op == OP_REDUCE_SCATTER || op == OP_ALL_EXCHANGE_ADD) ? (G - 1) * (N / G) : N;
  const uint32_t bar0 = smem_u32(recv_g + recv_floats), bar1 = bar0 + 8;
  for (int i = threadIdx.x; i < N; i += blockDim.x) tile_g[i] = in[(size_t)blockIdx.x * N + i];
  if (threadIdx.x == 0) {
    mbar_init(bar0, 1);
    mbar_init(bar1, 1);
    fence_mbar_init();
    mbar_expect_tx(bar0, expect0(op, N, G));
    if (op == OP_ALL_EXCHANGE_ADD) mbar_expect_tx(bar1, (uint32_t)((G - 1) * (N / G) * 4));
  }
  __syncthreads();
  fence_proxy_async_smem();  // the tile (generic writes) is a bulk-copy source
  cluster_sync();            // every peer's barriers are armed before any push
  for (int it = 0; it < iters; ++it) {
    const uint32_t ph = (uint32_t)(it & 1);
    switch (op) {
      case OP_REDUCE_SCATTER:
        dsm::reduce_scatter_add(tile_g, recv_g, tile, recv, bar0, ph, N, G, rank);
        break;
      case OP_ALL_GATHER:
        dsm::all_gather(tile, bar0, ph, N, G, rank);
        break;
      case OP_ALL_EXCHANGE_ADD:
        dsm::reduce_scatter_add(tile_g, recv_g, tile, recv, bar0, ph, N, G, rank);
        dsm::all_gather(tile, bar1, ph, N, G, rank);
        break;
      case OP_ALL_EXCHANGE_MUL:
        dsm::all_exchange_mul(tile_g, recv_g, tile, recv, bar0, ph, N, rank);
        break;
      default:
        dsm::shuffle_hop(tile, recv, bar0, ph, N, G, rank);
        break;
    }
    if (threadIdx.x == 0 && it + 1 < iters) {  // re-arm before the barrier that precedes the next pushes
      mbar_expect_tx(bar0, expect0(op, N, G));
      if (op == OP_ALL_EXCHANGE_ADD) mbar_expect_tx(bar1, (uint32_t)((G - 1) * (N / G) * 4));
    }
    __syncthreads();
    fence_proxy_async_smem();
    cluster_sync();  // peers consumed their receive slots / tiles before the next pushes
  }
  const float* src = op == OP_SHUFFLE ? recv_g : tile_g;
  for (int i = threadIdx.x; i < N; i += blockDim.x) out[(size_t)blockIdx.x * N + i] = src[i];
}

}  // namespace

extern "C" int ff_dsm_primitive_run(int op, int cluster, int floats_per_cta, int clusters, const float* in, float* out,
                                    int iters, float* ms_out) {
  if (op < 0 || op > 4 || cluster < 1 || cluster > 16 || floats_per_cta <= 0 || clusters < 1 || iters < 1) {
    ff::dsm_set_error("bad arguments");
    return 5;
  }
  if (floats_per_cta % (4 * cluster) || (op == OP_ALL_EXCHANGE_MUL && cluster % 2)) {
    ff::dsm_set_error("floats_per_cta must be a multiple of 4 * cluster (mul: even cluster)");
    return 3;
  }
  const int recv_floats = (op == OP_REDUCE_SCATTER || op == OP_ALL_EXCHANGE_ADD)
                              ? (cluster - 1) * (floats_per_cta / cluster)
                              : floats_per_cta;
  const size_t smem = (size_t)(floats_per_cta + recv_floats) * 4 + 64;
  if (smem > 232448 - 1024) {
    ff::dsm_set_error("tile + receive slots exceed shared memory");
    return 3;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(dsm_primitive_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448 - 1024);
    cudaFuncSetAttribute(dsm_primitive_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(cluster * clusters, 1, 1);
  lc.blockDim = dim3(256, 1, 1);
  lc.dynamicSmemBytes = smem;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = cluster;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  lc.attrs = a;
  lc.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaError_t e = cudaLaunchKernelEx(&lc, dsm_primitive_kernel, op, in, out, floats_per_cta, iters);
  cudaEventRecord(e1);
  if (e == cudaSuccess) e = cudaEventSynchronize(e1);
  if (e == cudaSuccess && ms_out) cudaEventElapsedTime(ms_out, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (e != cudaSuccess) {
    ff::dsm_set_error(cudaGetErrorString(e));
    return 4;
  }
  return 0;
}
