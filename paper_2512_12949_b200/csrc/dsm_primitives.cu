// Test / microbenchmark driver of the DSM communication primitives
// (dsm_primitives.cuh): one fp32 tile per CTA, clusters of G CTAs.
#include <cuda.h>
#include <cuda_runtime.h>

#include <string>

#include "../../include/ff_dsm.h"
#include "dsm_primitives.cuh"

namespace ff {
namespace {
thread_local std::string g_dsm_err;
}
void dsm_set_error(const char* msg) { g_dsm_err = msg; }
}  // namespace ff

extern "C" const char* ff_dsm_last_error(void) { return ff::g_dsm_err.c_str(); }

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

// ---------------------------------------------------------------------------
// DSM fabric bandwidth (calibration of the device profile's dsm.bandwidth[n];
// the paper's Fig. 4 method): every CTA of a cluster of `cluster` CTAs moves data
// to its right neighbour, all co-resident clusters at once.
//   mode 0  bulk push: `issuers` warps each issue cp.async.bulk shared::cta ->
//           shared::cluster copies of `chunk` bytes into `depth` receive slots of
//           the neighbour (completion on the neighbour's per-slot mbarrier); one
//           recycler warp per issuer re-arms a landed slot and credits the sender
//           (remote red.add), so `issuers * depth * chunk` bytes stay in flight.
//   mode 1  pull: all 256 threads ld.shared::cluster.v4 the neighbour's buffer.
//   mode 2  remote store: all 256 threads st.shared::cluster.v4 into it.
// ---------------------------------------------------------------------------
namespace {

__device__ __forceinline__ uint4 ld_cluster_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void st_cluster_v4(uint32_t addr, uint4 v) {
  asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w) : "memory");
}

__global__ void __launch_bounds__(256, 1) dsm_bw_kernel(int mode, int chunk, int depth, int issuers, int iters,
                                                        uint32_t* sink) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (ff::smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t rank = ff::cluster_rank(), csize = ff::cluster_size();
  const uint32_t right = (rank + 1) % csize, left = (rank + csize - 1) % csize;
  const int warp = threadIdx.x / 32;
  if (mode != 0) {
    const int bytes = 128 * 1024;  // buffer of every CTA
    ff::cluster_sync();
    const uint32_t peer = ff::mapa(base, right);
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (int it = 0; it < iters; ++it) {
#pragma unroll 4
      for (int off = threadIdx.x * 16; off < bytes; off += 256 * 16) {
        if (mode == 1) {
          const uint4 v = ld_cluster_v4(peer + off);
          acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
        } else {
          st_cluster_v4(peer + off, make_uint4(it, off, rank, 0));
        }
      }
    }
    ff::cluster_sync();
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x9e3779b9u) sink[0] = 1;  // keep the loads
    return;
  }
  // mode 0: [src chunk][recv slots issuers x depth x chunk][barriers][credits]
  const uint32_t src = base;
  const uint32_t recv = base + chunk;
  const uint32_t bars = recv + issuers * depth * chunk;
  const uint32_t credits = bars + issuers * depth * 8;
  if (threadIdx.x == 0) {
    for (int i = 0; i < issuers * depth; ++i) ff::mbar_init(bars + 8 * i, 1);
    for (int i = 0; i < issuers; ++i) ff::st_shared_u32(credits + 4 * i, 0u);
    ff::fence_mbar_init();
    for (int i = 0; i < issuers * depth; ++i) ff::mbar_expect_tx(bars + 8 * i, (uint32_t)chunk);
  }
  ff::cluster_sync();
  if (warp < issuers && ff::elect_one()) {
    const int i = warp;
    for (int it = 0; it < iters; ++it) {
      const int s = it % depth;
      if (it >= depth) ff::credit_wait(credits + 4 * i, (uint32_t)(it - depth + 1));
      ff::dsm_bulk_push(ff::mapa(recv + (i * depth + s) * chunk, right), src, (uint32_t)chunk,
                        ff::mapa(bars + 8 * (i * depth + s), right));
    }
  } else if (warp >= 4 && warp - 4 < issuers && ff::elect_one()) {
    const int i = warp - 4;
    for (int it = 0; it < iters; ++it) {
      const int s = it % depth;
      ff::mbar_wait(bars + 8 * (i * depth + s), (uint32_t)((it / depth) & 1));
      if (it + depth < iters) ff::mbar_expect_tx(bars + 8 * (i * depth + s), (uint32_t)chunk);
      ff::credit_add_remote(ff::mapa(credits + 4 * i, left));
    }
  }
  ff::cluster_sync();
}

}  // namespace

extern "C" int ff_dsm_bandwidth(int mode, int cluster, int chunk_bytes, int depth, int issuers, int iters,
                                int* clusters_out, float* ms_out) {
  if (mode < 0 || mode > 2 || cluster < 2 || cluster > 16 || iters < 1 || issuers < 1 || issuers > 4 || depth < 1 ||
      chunk_bytes < 16 || chunk_bytes % 16) {
    ff::dsm_set_error("bad arguments");
    return 5;
  }
  const size_t smem = mode == 0 ? (size_t)chunk_bytes * (1 + issuers * depth) + issuers * depth * 8 + 64 + 1024
                                : (size_t)128 * 1024 + 1024;
  if (smem > 232448) {
    ff::dsm_set_error("slots exceed shared memory");
    return 3;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(dsm_bw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    cudaFuncSetAttribute(dsm_bw_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  cudaLaunchConfig_t lc = {};
  lc.blockDim = dim3(256, 1, 1);
  lc.dynamicSmemBytes = smem;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = cluster;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  lc.attrs = a;
  lc.numAttrs = 1;
  lc.gridDim = dim3(cluster, 1, 1);
  int active = 0;
  if (cudaOccupancyMaxActiveClusters(&active, dsm_bw_kernel, &lc) != cudaSuccess || active < 1) {
    ff::dsm_set_error("cluster shape cannot be resident");
    return 3;
  }
  lc.gridDim = dim3(cluster * active, 1, 1);
  uint32_t* sink = nullptr;
  cudaMalloc(&sink, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaError_t e = cudaLaunchKernelEx(&lc, dsm_bw_kernel, mode, chunk_bytes, depth, issuers, iters, sink);
  cudaEventRecord(e1);
  if (e == cudaSuccess) e = cudaEventSynchronize(e1);
  if (e == cudaSuccess && ms_out) cudaEventElapsedTime(ms_out, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  if (clusters_out) *clusters_out = active;
  if (e != cudaSuccess) {
    ff::dsm_set_error(cudaGetErrorString(e));
    return 4;
  }
  return 0;
}
