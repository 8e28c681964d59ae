// DSM (distributed shared memory) bandwidth microbenchmark, the paper's
// Fig. 4/13 measurement redone on sm_100a: every CTA of a cluster pushes
// `chunk` bytes to its right ring neighbour `iters` times with
// cp.async.bulk shared::cta -> shared::cluster (mbarrier complete_tx),
// keeping `depth` transfers in flight.  Reports aggregate bytes/s.
// Used to calibrate dsm.bandwidth[n] of the B200 device profile.
#include <cuda.h>
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

__global__ void stamp_kernel(unsigned long long* dst) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *dst = t;
}

// Launch-overhead probe: an otherwise empty kernel with the launch shape of
// the chain kernels (dynamic smem, cluster, TMEM alloc); stamps entry/exit.
__global__ void __launch_bounds__(256, 1) launch_probe_kernel(unsigned long long* stamps, int tmem) {
  extern __shared__ __align__(1024) uint8_t smem[];
  using namespace ff;
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    stamps[2 * blockIdx.x] = t;
  }
  if (tmem && threadIdx.x / 32 == 1) tmem_alloc<512>(smem_u32(smem));
  __syncthreads();
  if (tmem && threadIdx.x / 32 == 1) {
    tc_fence_after();
    tmem_dealloc<512>(*reinterpret_cast<volatile uint32_t*>(smem));
  }
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    stamps[2 * blockIdx.x + 1] = t;
  }
}

struct BigParams {
  unsigned long long pad[176];  // 1408 B, the size of PairMaps
};
__global__ void __launch_bounds__(256, 1) launch_probe_big_kernel(const __grid_constant__ BigParams bp,
                                                                  unsigned long long* stamps) {
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    stamps[2 * blockIdx.x] = t + (bp.pad[threadIdx.x + 100] & 1ull);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    stamps[2 * blockIdx.x + 1] = t;
  }
}

// launch-latency probe with a chain kernel's register footprint (~170 registers per thread)
__global__ void __launch_bounds__(256, 1) launch_probe_regs_kernel(unsigned long long* stamps, int n) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0) stamps[2 * blockIdx.x] = t;
  float v[160];
#pragma unroll
  for (int i = 0; i < 160; ++i) v[i] = (float)(i * n + threadIdx.x);
  float acc = 0.f;
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int i = 0; i < 160; ++i) acc = fmaf(acc, v[(i + r) % 160], v[i]);
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0) stamps[2 * blockIdx.x + 1] = t + (acc == 12345.f ? 1 : 0);
}

// launch-latency probe with eleven __grid_constant__ tensor maps (the pair kernel's params)
struct ElevenMaps {
  CUtensorMap m[11];
};
__global__ void __launch_bounds__(256, 1) launch_probe_tmap_kernel(const __grid_constant__ ElevenMaps maps,
                                                                   unsigned long long* stamps, int prefetch) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0) stamps[2 * blockIdx.x] = t;
  if (prefetch && threadIdx.x == 0)
    for (int i = 0; i < 11; ++i) ff::tma_prefetch_desc(&maps.m[i]);
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0) stamps[2 * blockIdx.x + 1] = t;
}

// launch-latency probe with ~100 KB of (never executed) code
__global__ void __launch_bounds__(256, 1) launch_probe_big_code_kernel(unsigned long long* stamps, int n, float* sink) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0) stamps[2 * blockIdx.x] = t;
  if (n == 12345) {  // never true at run time; the code is still in the binary
    float a = sink[threadIdx.x], b = sink[threadIdx.x + 1];
#pragma unroll
    for (int i = 0; i < 3000; ++i) {
      a = fmaf(a, b, (float)i);
      b = fmaf(b, a, (float)(i ^ 7));
      if ((i & 63) == 0) sink[threadIdx.x + i] = a;
    }
    sink[threadIdx.x] = a + b;
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0) stamps[2 * blockIdx.x + 1] = t;
}

__global__ void spin_kernel(long long cycles) {
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
}

}  // namespace

namespace ff {
// shared by the DSM primitive driver (dsm_primitives.cu): ff_dsm_last_error reports it
void dsm_set_error(const char* msg) { g_err = msg; }
}  // namespace ff

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

int ff_launch_probe(void* stamps, int ctas, int smem_bytes, int cluster, int tmem, void* stream) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(launch_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448 - 1024);
    cudaFuncSetAttribute(launch_probe_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(ctas, 1, 1);
  lc.blockDim = dim3(256, 1, 1);
  lc.dynamicSmemBytes = smem_bytes;
  lc.stream = reinterpret_cast<cudaStream_t>(stream);
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = cluster;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  lc.attrs = a;
  lc.numAttrs = cluster > 1 ? 1 : 0;
  cudaError_t e;
  if (tmem == 6) {
    static bool attr6 = false;
    if (!attr6) {
      cudaFuncSetAttribute(launch_probe_big_code_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448 - 1024);
      cudaFuncSetAttribute(launch_probe_big_code_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      attr6 = true;
    }
    e = cudaLaunchKernelEx(&lc, launch_probe_big_code_kernel, reinterpret_cast<unsigned long long*>(stamps), 0,
                           reinterpret_cast<float*>(stamps));
  } else if (tmem == 4 || tmem == 5) {
    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    ElevenMaps maps;
    cuuint64_t dims[2] = {64, 256}, str[1] = {128};
    cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    for (int i = 0; i < 11; ++i)
      reinterpret_cast<EncodeFn>(fp)(&maps.m[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, stamps, dims, str, box, es,
                                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    static bool attr4 = false;
    if (!attr4) {
      cudaFuncSetAttribute(launch_probe_tmap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448 - 1024);
      cudaFuncSetAttribute(launch_probe_tmap_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      attr4 = true;
    }
    e = cudaLaunchKernelEx(&lc, launch_probe_tmap_kernel, maps, reinterpret_cast<unsigned long long*>(stamps),
                           tmem == 5 ? 1 : 0);
  } else if (tmem == 3) {
    static bool attr3 = false;
    if (!attr3) {
      cudaFuncSetAttribute(launch_probe_regs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448 - 1024);
      cudaFuncSetAttribute(launch_probe_regs_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      attr3 = true;
    }
    e = cudaLaunchKernelEx(&lc, launch_probe_regs_kernel, reinterpret_cast<unsigned long long*>(stamps), 3);
  } else if (tmem == 2) {
    BigParams bp = {};
    lc.dynamicSmemBytes = 0;
    e = cudaLaunchKernelEx(&lc, launch_probe_big_kernel, bp, reinterpret_cast<unsigned long long*>(stamps));
  } else {
    e = cudaLaunchKernelEx(&lc, launch_probe_kernel, reinterpret_cast<unsigned long long*>(stamps), tmem);
  }
  if (e != cudaSuccess) {
    g_err = cudaGetErrorString(e);
    return 4;
  }
  return 0;
}

int ff_spin(long long cycles, int ctas, void* stream) {
  spin_kernel<<<ctas, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(cycles);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_err = cudaGetErrorString(e);
    return 4;
  }
  return 0;
}

int ff_stamp_globaltimer(void* dst, void* stream) {
  stamp_kernel<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(reinterpret_cast<unsigned long long*>(dst));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_err = cudaGetErrorString(e);
    return 4;
  }
  return 0;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// TMA streaming microbenchmark: each CTA streams `per_cta_kb` k-blocks of a
// row-major bf16 matrix [rows][cols] through a `stages`-deep ring of 32 KB
// stages (box = 64 cols x 64 rows MN-major, or 64 cols x 128 rows), the
// consumer only waits and releases.  Measures per-SM TMA ingress.
// ---------------------------------------------------------------------------
namespace {
// `producers` threads (one per warp) each own stages p, p+P, ... of a ring of
// `stages` x `stage_bytes` buffers; one consumer thread per producer.
__global__ void __launch_bounds__(256, 1) tma_stream_kernel(const __grid_constant__ CUtensorMap map, int rows,
                                                            int cols, int stages, int iters, int box_rows,
                                                            int producers, int stage_bytes) {
  using namespace ff;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const uint32_t full0 = base + stages * stage_bytes, empty0 = full0 + 8 * stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int box_blocks = box_rows >> 16;
  box_rows &= 0xffff;
  const int per_box = 64 * box_rows * 2 * (box_blocks ? box_blocks : 1);
  const int boxes = stage_bytes / per_box;
  const int col_tiles = cols / (64 * (box_blocks ? box_blocks : 1)), row_tiles = rows / box_rows;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int my_stages = stages / producers;
  if (lane == 0 && warp < producers) {
    int k = 0, phase = 0;
    for (int i = 0; i < iters; ++i) {
      const int stage = warp + k * producers;
      mbar_wait(empty0 + 8 * stage, phase ^ 1);
      mbar_expect_tx(full0 + 8 * stage, stage_bytes);
      for (int b = 0; b < boxes; ++b) {
        const long long lin = ((long long)(blockIdx.x * producers + warp) * 7919 + (long long)i * boxes + b);
        const int ct = (int)(lin % col_tiles), rt = (int)((lin / col_tiles) % row_tiles);
        if (box_blocks)
          tma_load_3d(base + stage * stage_bytes + b * per_box, &map, full0 + 8 * stage, 0, rt * box_rows,
                      ct * box_blocks);
        else
          tma_load_2d(base + stage * stage_bytes + b * per_box, &map, full0 + 8 * stage, ct * 64, rt * box_rows);
      }
      if (++k == my_stages) { k = 0; phase ^= 1; }
    }
  } else if (lane == 0 && warp >= 4 && warp - 4 < producers) {
    const int w = warp - 4;
    int k = 0, phase = 0;
    for (int i = 0; i < iters; ++i) {
      const int stage = w + k * producers;
      mbar_wait(full0 + 8 * stage, phase);
      mbar_arrive(empty0 + 8 * stage);
      if (++k == my_stages) { k = 0; phase ^= 1; }
    }
  }
  __syncthreads();
}
// Multicast variant: clusters of `csize` CTAs stream the same 3D tiles; CTA r
// of a cluster fetches slice r (box rows / csize) of every stage-sized tile
// and multicasts it to all CTAs, so each CTA receives `stage_bytes` per stage
// while issuing 1/csize of them.  Measures whether multicast lifts the per-SM
// operand feed above the single-CTA TMA ceiling.
__global__ void __launch_bounds__(256, 1) tma_mcast_kernel(const __grid_constant__ CUtensorMap map, int rows,
                                                           int cols, int stages, int iters, int box_rows,
                                                           int box_blocks, int stage_bytes, int flags) {
  using namespace ff;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const uint32_t full0 = base + stages * stage_bytes, empty0 = full0 + 8 * stages;
  const int csize = (int)cluster_size(), me = (int)cluster_rank();
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, csize);  // every CTA's consumer frees the stage cluster-wide
    }
    fence_mbar_init();
  }
  cluster_sync();
  const int slice_rows = box_rows / csize;
  const int slice_bytes = 64 * slice_rows * 2 * box_blocks;
  const int per_box = 64 * box_rows * 2 * box_blocks;
  const int boxes = stage_bytes / per_box;
  const int col_tiles = cols / (64 * box_blocks), row_tiles = rows / box_rows;
  const int cl = blockIdx.x / csize;
  const uint16_t mask = (uint16_t)((1u << csize) - 1u);
  const bool cta_wait = (flags & 2) != 0;    // csize == 1 only: producer waits with CTA scope
  const bool cta_arrive = (flags & 4) != 0;  // csize == 1 only: consumer arrives locally (no release.cluster)
  if (threadIdx.x == 0) {
    int stage = 0, phase = 0;
    for (int i = 0; i < iters; ++i) {
      if (cta_wait)
        mbar_wait(empty0 + 8 * stage, phase ^ 1);
      else
        mbar_wait_cluster(empty0 + 8 * stage, phase ^ 1);
      mbar_expect_tx(full0 + 8 * stage, stage_bytes);
      for (int b = 0; b < boxes; ++b) {
        const long long lin = (long long)cl * 7919 + (long long)i * boxes + b;
        const int ct = (int)(lin % col_tiles), rt = (int)((lin / col_tiles) % row_tiles);
        const uint32_t dst = base + stage * stage_bytes + b * per_box + me * slice_bytes;
        if (csize > 1)
          tma_load_3d_mcast(dst, &map, full0 + 8 * stage, 0, rt * box_rows + me * slice_rows, ct * box_blocks, mask);
        else
          tma_load_3d(dst, &map, full0 + 8 * stage, 0, rt * box_rows, ct * box_blocks);
      }
      if (++stage == stages) { stage = 0; phase ^= 1; }
    }
  } else if (threadIdx.x == 128) {
    int stage = 0, phase = 0;
    for (int i = 0; i < iters; ++i) {
      mbar_wait(full0 + 8 * stage, phase);
      if (cta_arrive)
        mbar_arrive(empty0 + 8 * stage);
      else if (flags & 8)  // relaxed remote arrives (no release fence)
        for (int r = 0; r < csize; ++r) mbar_arrive_remote_relaxed(mapa(empty0 + 8 * stage, r));
      else
        for (int r = 0; r < csize; ++r) mbar_arrive_remote(mapa(empty0 + 8 * stage, r));
      if (++stage == stages) { stage = 0; phase ^= 1; }
    }
  }
  __syncthreads();
  cluster_sync();
}
}  // namespace

extern "C" int ff_tma_stream_bench(const void* mat, int rows, int cols, int stages, int iters, int box_rows,
                                   int ctas, int producers, int stage_bytes, float* ms_out) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess) return 4;
  CUtensorMap map;
  const int bb = box_rows >> 16, br = box_rows & 0xffff;
  CUresult cr;
  if (bb) {
    cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)cols / 64};
    cuuint64_t strides[2] = {(cuuint64_t)cols * 2, 128};
    cuuint32_t box[3] = {64, (cuuint32_t)br, (cuuint32_t)bb};
    cuuint32_t estr[3] = {1, 1, 1};
    cr = reinterpret_cast<EncodeFn>(p)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(mat), dims, strides,
                                       box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)br};
    cuuint32_t estr[2] = {1, 1};
    cr = reinterpret_cast<EncodeFn>(p)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(mat), dims, strides,
                                       box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (cr != CUDA_SUCCESS) return 6;
  const int smem = stages * stage_bytes + 16 * stages + 2048;
  if (smem > 232448) return 5;
  cudaFuncSetAttribute(tma_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  tma_stream_kernel<<<ctas, 256, smem>>>(map, rows, cols, stages, 8, box_rows, producers, stage_bytes);
  cudaEventRecord(a);
  tma_stream_kernel<<<ctas, 256, smem>>>(map, rows, cols, stages, iters, box_rows, producers, stage_bytes);
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (e != cudaSuccess) return 4;
  *ms_out = ms;
  return 0;
}

extern "C" int ff_tma_mcast_bench(const void* mat, int rows, int cols, int stages, int iters, int box_rows,
                                  int box_blocks, int csize, int ctas, int stage_bytes, int flags, float* ms_out) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess) return 4;
  if (csize < 1 || box_rows % csize || ctas % csize) return 5;
  CUtensorMap map;
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)cols / 64};
  cuuint64_t strides[2] = {(cuuint64_t)cols * 2, 128};
  cuuint32_t box[3] = {64, (cuuint32_t)(box_rows / csize), (cuuint32_t)box_blocks};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult cr = reinterpret_cast<EncodeFn>(p)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(mat), dims,
                                              strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return 6;
  const int smem = stages * stage_bytes + 16 * stages + 2048;
  if (smem > 232448) return 5;
  cudaFuncSetAttribute(tma_mcast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(ctas, 1, 1);
  lc.blockDim = dim3(256, 1, 1);
  lc.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = (flags & 1) && csize == 1 ? 0 : 1;  // bit0: plain (non-cluster) launch
  if (csize > 1) flags &= ~6;  // bit3 (relaxed remote arrives) stays
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaLaunchKernelEx(&lc, tma_mcast_kernel, map, rows, cols, stages, 8, box_rows, box_blocks, stage_bytes, flags);
  cudaEventRecord(a);
  cudaLaunchKernelEx(&lc, tma_mcast_kernel, map, rows, cols, stages, iters, box_rows, box_blocks, stage_bytes, flags);
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
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
