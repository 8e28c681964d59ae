// FlashFuser's DSM communication primitives (paper SIII-B, dsm_comm; modeled
// by the reference analyzer.py:331-354) on sm_100a distributed shared memory.
//
// Every primitive works on one fp32 tile of N floats per CTA of a thread-block
// cluster of G CTAs (slice = N/G floats), moves data with
// cp.async.bulk.shared::cluster (a bulk copy from this CTA's shared memory into
// a peer's, completing bytes on the peer's mbarrier) and sums in cluster-rank
// order, so every result is deterministic:
//   reduce_scatter_add  CTA r ends with slice r of sum_g tile_g      (reduce-scatter)
//   all_gather          CTA r's slice r lands at slice r of every peer's tile
//   all_exchange_add    reduce_scatter_add + all_gather: every CTA ends with sum_g tile_g
//   all_exchange_mul    CTA pair (2i, 2i+1) holds SwiGLU's gate / up branch partials
//                       (spatial_split lowering): both end with silu(gate) * up
//   shuffle_hop         one ring hop: CTA r receives CTA r-1's tile (the shuffle the
//                       fused kernel iterates, ff_chain_kernel<kMode 0>)
// The receiving CTA arms its mbarrier with the bytes it expects before the
// cluster barrier that precedes the pushes; thread 0 issues the copies and
// the whole CTA waits on the barrier, then combines.
#pragma once
#include "ptx.cuh"

namespace ff {
namespace dsm {

// receive-slot index of sender `src` at receiver `dst` (G-1 slots, sender order)
__device__ __forceinline__ int slot_of(int src, int dst) { return src < dst ? src : src - 1; }

__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }

// Thread 0: push this CTA's part for every peer (peer d gets tile slice d) into
// the peer's receive slot; the peer's barrier `bar` completes when all G-1 arrive.
__device__ __forceinline__ void rs_push(uint32_t tile, uint32_t recv, uint32_t bar, int slice_bytes, int G, int rank) {
  if (threadIdx.x != 0) return;
  for (int d = 1; d < G; ++d) {
    const int dst = (rank + d) % G;
    dsm_bulk_push(mapa(recv + slot_of(rank, dst) * slice_bytes, dst), tile + dst * slice_bytes, slice_bytes,
                  mapa(bar, dst));
  }
}

// reduce-scatter (Add): after the barrier phase completes, slice `rank` of the
// tile holds the rank-ordered sum of every CTA's slice `rank`.
__device__ __forceinline__ void reduce_scatter_add(float* tile_g, const float* recv_g, uint32_t tile, uint32_t recv,
                                                   uint32_t bar, uint32_t phase, int N, int G, int rank) {
  const int slice = N / G;
  rs_push(tile, recv, bar, slice * 4, G, rank);
  mbar_wait_cluster(bar, phase);
  for (int i = threadIdx.x; i < slice; i += blockDim.x) {
    float acc = 0.f;
    for (int r = 0; r < G; ++r) {
      const float v = r == rank ? tile_g[rank * slice + i] : recv_g[slot_of(r, rank) * slice + i];
      acc = r == 0 ? v : acc + v;
    }
    tile_g[rank * slice + i] = acc;
  }
}

// all-gather: slice `rank` of this tile goes to the same place in every peer's tile.
__device__ __forceinline__ void all_gather(uint32_t tile, uint32_t bar, uint32_t phase, int N, int G, int rank) {
  const int slice_bytes = N / G * 4;
  __syncthreads();             // the slice is final (reduce step above)
  fence_proxy_async_smem();    // generic writes -> async-proxy bulk copy source
  __syncthreads();
  if (threadIdx.x == 0)
    for (int d = 1; d < G; ++d) {
      const int dst = (rank + d) % G;
      dsm_bulk_push(mapa(tile + rank * slice_bytes, dst), tile + rank * slice_bytes, slice_bytes, mapa(bar, dst));
    }
  mbar_wait_cluster(bar, phase);
}

// all_exchange (Mul) for a CTA pair: even rank holds the gate partial, odd the up partial.
__device__ __forceinline__ void all_exchange_mul(float* tile_g, const float* recv_g, uint32_t tile, uint32_t recv,
                                                 uint32_t bar, uint32_t phase, int N, int rank) {
  const int peer = rank ^ 1;
  if (threadIdx.x == 0) dsm_bulk_push(mapa(recv, peer), tile, N * 4, mapa(bar, peer));
  mbar_wait_cluster(bar, phase);
  // both CTAs must have pushed (read) their tile before either overwrites it
  cluster_sync();
  const bool gate_here = (rank & 1) == 0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const float mine = tile_g[i], other = recv_g[i];
    tile_g[i] = gate_here ? silu(mine) * other : silu(other) * mine;
  }
}

// one ring hop: recv <- tile of CTA rank-1
__device__ __forceinline__ void shuffle_hop(uint32_t tile, uint32_t recv, uint32_t bar, uint32_t phase, int N, int G,
                                            int rank) {
  if (threadIdx.x == 0) dsm_bulk_push(mapa(recv, (rank + 1) % G), tile, N * 4, mapa(bar, (rank + 1) % G));
  mbar_wait_cluster(bar, phase);
}

}  // namespace dsm
}  // namespace ff
