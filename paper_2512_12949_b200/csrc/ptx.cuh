// Thin inline-PTX layer for sm_100a: mbarriers, TMA, tcgen05 (UMMA + TMEM),
// and the cluster / distributed-shared-memory (DSM) transport used by the
// dsm_comm primitives.  Everything here is a single instruction (or a short
// fixed sequence); the dataflow lives in ff_chain.cu.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ff {

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t lane_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// ----------------------------------------------------------------------------
// cluster
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Map a local shared::cta address to the same offset in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}

// ----------------------------------------------------------------------------
// mbarrier
// ----------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
// Arrive on a barrier living in another CTA of the cluster (address from mapa).
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar)
               : "memory");
}
// Remote arrive without release semantics (the arriving thread publishes no
// data through it; e.g. "stage consumed" when the consumer is asynchronous).
__device__ __forceinline__ void mbar_arrive_remote_relaxed(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// Cluster-scope acquire variant: needed when the phase was completed by a
// remote arrive or a DSM bulk copy issued by another CTA.
__device__ __forceinline__ bool mbar_try_wait_cluster(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// Watchdog: a wait that never completes is a protocol bug; trap (the launch then
// fails with an error) instead of hanging the GPU.  try_wait suspends for a
// hardware-chosen interval per call, so 2^26 polls is several seconds.
#ifndef FF_WATCHDOG_POLLS
#define FF_WATCHDOG_POLLS (1u << 26)
#endif
__device__ __forceinline__ void watchdog_trap() { asm volatile("trap;"); }
// Diagnostic builds (-DFF_DIAG_WATCHDOG, never the shipped library): an expired wait records
// (source line, block, thread, info) in ff_diag and gives up instead of trapping, so the launch
// completes and the host can read which wait hung (ff_diag_read).
#ifdef FF_DIAG_WATCHDOG
// ff_diag[0] = expired waits; then up to 512 (key, info) records in expiry order
static __device__ unsigned long long ff_diag[1 + 2 * 512];
__device__ __forceinline__ void watchdog_record(unsigned line, unsigned long long info) {
  const unsigned long long key = ((unsigned long long)line << 40) | ((unsigned long long)blockIdx.x << 20) | threadIdx.x;
  const unsigned long long i = atomicAdd(&ff_diag[0], 1ull);
  if (i < 512) {
    ff_diag[1 + 2 * i] = key;
    ff_diag[2 + 2 * i] = info;
  }
}
#define FF_WD_EXPIRED(info) \
  {                         \
    watchdog_record(__LINE__, (unsigned long long)(info)); \
    break;                  \
  }
#else
#define FF_WD_EXPIRED(info) watchdog_trap()
#endif
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t polls = 0;
  while (!mbar_try_wait(bar, parity)) {
    if (++polls == FF_WATCHDOG_POLLS) FF_WD_EXPIRED(((unsigned long long)bar << 8) | parity);
  }
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  uint32_t polls = 0;
  while (!mbar_try_wait_cluster(bar, parity)) {
    if (++polls == FF_WATCHDOG_POLLS) FF_WD_EXPIRED(((unsigned long long)bar << 8) | 0x10 | parity);
  }
}

// Monotonic credit counters in shared memory (no phase aliasing, unlike an
// mbarrier that can be completed twice before the waiter looks).
// Remote credit / ack increment.  Relaxed: it publishes no data (the events it
// reports -- a landed push, a consumed receive buffer -- were observed through
// mbarriers before it is issued), and a release.cluster fence per hop costs
// ~1 us of latency on B200 (profiles/r01/tma_variants.log).
__device__ __forceinline__ void credit_add_remote(uint32_t cluster_addr) {
  asm volatile("red.relaxed.cluster.shared::cluster.add.u32 [%0], 1;" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_cluster_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.acquire.cluster.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void credit_wait(uint32_t addr, uint32_t target) {
  uint32_t polls = 0;
  while ((int)(ld_acquire_cluster_u32(addr) - target) < 0) {
    if (++polls == 16 * FF_WATCHDOG_POLLS) FF_WD_EXPIRED(((unsigned long long)addr << 32) | target);
  }
}

// gpu-scope release/acquire flags in global memory
__device__ __forceinline__ void st_release_gpu_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_gpu_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Invalidate one 128-byte L2 line without writing it back (scratch whose last reader is
// done: its dirty lines would otherwise cost a DRAM write-back after the kernel).
__device__ __forceinline__ void discard_l2_line(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// named barrier among `count` threads
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// ----------------------------------------------------------------------------
// fences
// ----------------------------------------------------------------------------
// Generic-proxy shared-memory writes -> visible to the async proxy (UMMA, bulk copies).
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ----------------------------------------------------------------------------
// TMA (global -> shared), bulk DSM copies (shared::cta -> shared::cluster)
// ----------------------------------------------------------------------------
// L2 prefetch of a tensor box (no shared-memory destination, no completion).
__device__ __forceinline__ void tma_prefetch_l2_3d(const void* desc, int32_t c0, int32_t c1, int32_t c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"(desc), "r"(c0), "r"(c1),
               "r"(c2)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_l2_4d(const void* desc, int32_t c0, int32_t c1, int32_t c2,
                                                   int32_t c3) {
  asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global [%0, {%1, %2, %3, %4}];" ::"l"(desc), "r"(c0), "r"(c1),
               "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const void* desc) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(desc) : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const void* desc, uint32_t bar, int32_t c0,
                                            int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(desc), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
// im2col mode over an NHWC tensor map (cuTensorMapEncodeIm2col): a box of
// pixelsPerColumn consecutive output pixels x channelsPerPixel channels,
// starting at bounding-box position (c, w, h, n), each pixel displaced by the
// filter tap (off_w, off_h); out-of-image taps are zero-filled (padding).
__device__ __forceinline__ void tma_load_im2col_4d(uint32_t dst, const void* desc, uint32_t bar, int32_t c,
                                                   int32_t w, int32_t h, int32_t n, uint16_t off_w,
                                                   uint16_t off_h) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], {%7, %8};" ::"r"(dst),
      "l"(desc), "r"(c), "r"(w), "r"(h), "r"(n), "r"(bar), "h"(off_w), "h"(off_h)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const void* desc, uint32_t bar, int32_t c0, int32_t c1,
                                            int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(desc), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_pair(uint32_t dst, const void* desc, uint32_t leader_bar, int32_t c0,
                                                 int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(desc), "r"(c0), "r"(c1), "r"(c2), "r"(leader_bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d_pair(uint32_t dst, const void* desc, uint32_t leader_bar, int32_t c0,
                                                 int32_t c1, int32_t c2, int32_t c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
      "l"(desc), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(leader_bar)
      : "memory");
}
// Pair loads multicast to the same offset of every CTA in `mask`; each
// destination's complete_tx lands on its pair leader's barrier (the leader_bar
// offset, peer bit cleared), as for the unicast pair form.
__device__ __forceinline__ void tma_load_3d_pair_mcast(uint32_t dst, const void* desc, uint32_t leader_bar, int32_t c0,
                                                       int32_t c1, int32_t c2, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
      "l"(desc), "r"(c0), "r"(c1), "r"(c2), "r"(leader_bar), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d_pair_mcast(uint32_t dst, const void* desc, uint32_t leader_bar, int32_t c0,
                                                       int32_t c1, int32_t c2, int32_t c3, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(dst),
      "l"(desc), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(leader_bar), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const void* desc, uint32_t src, int32_t c0, int32_t c1, int32_t c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(desc),
               "r"(src), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
// Element-wise fp32 add of a shared-memory box into global memory (TMA reduce).
__device__ __forceinline__ void tma_reduce_add_2d(const void* desc, uint32_t src, int32_t c0, int32_t c1) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(desc),
               "r"(src), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_store_4d(const void* desc, uint32_t src, int32_t c0, int32_t c1, int32_t c2,
                                             int32_t c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(desc),
               "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const void* desc, uint32_t bar, int32_t c0, int32_t c1,
                                            int32_t c2, int32_t c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
      "l"(desc), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_reduce_add_3d(const void* desc, uint32_t src, int32_t c0, int32_t c1,
                                                  int32_t c2) {
  asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   desc),
               "r"(src), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void st_shared_v2(uint32_t addr, uint32_t a, uint32_t b) {
  asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ float4 ld_shared_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr)
               : "memory");
  return v;
}
__device__ __forceinline__ void bulk_wait_read0_group() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// Same tile lands at the same smem offset of every CTA in `mask`; each
// destination CTA's barrier at offset `bar` receives complete_tx.
__device__ __forceinline__ void tma_load_2d_mcast(uint32_t dst, const void* desc, uint32_t bar,
                                                  int32_t c0, int32_t c1, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(desc), "r"(c0), "r"(c1), "r"(bar), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_mcast(uint32_t dst, const void* desc, uint32_t bar, int32_t c0,
                                                  int32_t c1, int32_t c2, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
      "l"(desc), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "h"(mask)
      : "memory");
}
// DSM push: copy `bytes` from local smem to another CTA's smem; completion is
// signalled on the destination CTA's barrier (both addresses from mapa).
__device__ __forceinline__ void dsm_bulk_push(uint32_t dst_cluster, uint32_t src_local, uint32_t bytes,
                                              uint32_t dst_bar_cluster) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst_cluster),
      "r"(src_local), "r"(bytes), "r"(dst_bar_cluster)
      : "memory");
}
// TMA store (shared -> global); a bulk-group operation.
__device__ __forceinline__ void tma_store_2d(const void* desc, uint32_t src, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(desc),
               "r"(src), "r"(c0), "r"(c1)
               : "memory");
}
// ---- L2 cache policies (createpolicy) and hinted TMA forms ----
// Weights streamed once get evict_first, the C exchange scratch evict_last (it
// must stay on chip until every ring member has read it); 0 = no hint.
enum L2Hint : int { L2_NORMAL = 0, L2_EVICT_FIRST = 1, L2_EVICT_LAST = 2 };
__device__ __forceinline__ uint64_t l2_policy(int hint) {
  uint64_t p;
  if (hint == L2_EVICT_FIRST)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  else if (hint == L2_EVICT_LAST)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_3d_pair_h(uint32_t dst, const void* desc, uint32_t leader_bar, int32_t c0,
                                                   int32_t c1, int32_t c2, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
      "l"(desc), "r"(c0), "r"(c1), "r"(c2), "r"(leader_bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d_pair_h(uint32_t dst, const void* desc, uint32_t leader_bar, int32_t c0,
                                                   int32_t c1, int32_t c2, int32_t c3, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(dst),
      "l"(desc), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(leader_bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_pair_mcast_h(uint32_t dst, const void* desc, uint32_t leader_bar,
                                                         int32_t c0, int32_t c1, int32_t c2, uint16_t mask,
                                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      ".L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6, %7;" ::"r"(dst),
      "l"(desc), "r"(c0), "r"(c1), "r"(c2), "r"(leader_bar), "h"(mask), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d_pair_mcast_h(uint32_t dst, const void* desc, uint32_t leader_bar,
                                                         int32_t c0, int32_t c1, int32_t c2, int32_t c3,
                                                         uint16_t mask, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      ".L2::cache_hint [%0], [%1, {%2, %3, %4, %5}], [%6], %7, %8;" ::"r"(dst),
      "l"(desc), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(leader_bar), "h"(mask), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d_h(const void* desc, uint32_t src, int32_t c0, int32_t c1, uint64_t pol) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;" ::"l"(
                   desc),
               "r"(src), "r"(c0), "r"(c1), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void tma_store_3d_h(const void* desc, uint32_t src, int32_t c0, int32_t c1, int32_t c2,
                                               uint64_t pol) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3, %4}], [%1], %5;" ::"l"(
                   desc),
               "r"(src), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_l2_3d_h(const void* desc, int32_t c0, int32_t c1, int32_t c2,
                                                     uint64_t pol) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.L2::cache_hint [%0, {%1, %2, %3}], %4;" ::"l"(desc),
               "r"(c0), "r"(c1), "r"(c2), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_l2_4d_h(const void* desc, int32_t c0, int32_t c1, int32_t c2,
                                                     int32_t c3, uint64_t pol) {
  asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.L2::cache_hint [%0, {%1, %2, %3, %4}], %5;" ::"l"(desc),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3), "l"(pol)
               : "memory");
}
// Bulk-group completion (TMA stores / bulk_group copies only -- NOT the
// mbarrier-completed shared::cluster copies).
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// ----------------------------------------------------------------------------
// tcgen05: TMEM allocation, MMA, commit, loads
// ----------------------------------------------------------------------------
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem], kind::f16 (bf16 in, fp32 accumulate).
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive (once) on a local barrier when all previously issued MMAs retire.
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 32 lanes x 32 bit, 16 consecutive columns per thread.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15])
      : "r"(taddr));
  tmem_wait_ld();
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// ---- CTA pair (cta_group::2): two SMs of a cluster pair issue one M=256 MMA ----
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc_pair(uint32_t dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem), "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}
// Issued by the leader CTA only: D[tmem of both CTAs] (+)= A[smem of both] * B[smem of both].
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on the barrier at offset `bar` of every CTA in `mask` when the pair's MMAs retire.
__device__ __forceinline__ void umma_commit_pair(uint32_t bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          bar),
      "h"(mask)
      : "memory");
}
// TMA load into this CTA's smem; transaction bytes are signalled on the leader
// CTA's barrier (cluster address from mapa).
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const void* desc, uint32_t leader_bar, int32_t c0,
                                                 int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(desc), "r"(c0), "r"(c1), "r"(leader_bar)
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  tmem_wait_ld();
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 x kN consecutive TMEM columns of this warp's lane quarter into registers (kN x
// 32x32b.x32 loads behind one tcgen05.wait::ld; the registers are threaded through the
// wait, 64 per asm statement, so no consumer is scheduled before it).
template <int kN>
__device__ __forceinline__ void tmem_ld32xn(uint32_t taddr, float (&v)[32 * kN]) {
  uint32_t r[32 * kN];
#pragma unroll
  for (int g = 0; g < kN; ++g)
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[32 * g + 0]), "=r"(r[32 * g + 1]), "=r"(r[32 * g + 2]), "=r"(r[32 * g + 3]), "=r"(r[32 * g + 4]),
          "=r"(r[32 * g + 5]), "=r"(r[32 * g + 6]), "=r"(r[32 * g + 7]), "=r"(r[32 * g + 8]), "=r"(r[32 * g + 9]),
          "=r"(r[32 * g + 10]), "=r"(r[32 * g + 11]), "=r"(r[32 * g + 12]), "=r"(r[32 * g + 13]),
          "=r"(r[32 * g + 14]), "=r"(r[32 * g + 15]), "=r"(r[32 * g + 16]), "=r"(r[32 * g + 17]),
          "=r"(r[32 * g + 18]), "=r"(r[32 * g + 19]), "=r"(r[32 * g + 20]), "=r"(r[32 * g + 21]),
          "=r"(r[32 * g + 22]), "=r"(r[32 * g + 23]), "=r"(r[32 * g + 24]), "=r"(r[32 * g + 25]),
          "=r"(r[32 * g + 26]), "=r"(r[32 * g + 27]), "=r"(r[32 * g + 28]), "=r"(r[32 * g + 29]),
          "=r"(r[32 * g + 30]), "=r"(r[32 * g + 31])
        : "r"(taddr + 32u * g));
#define FF_TIE8(o) "+r"(r[o]), "+r"(r[o + 1]), "+r"(r[o + 2]), "+r"(r[o + 3]), "+r"(r[o + 4]), "+r"(r[o + 5]), \
                   "+r"(r[o + 6]), "+r"(r[o + 7])
#pragma unroll
  for (int g = 0; g < kN; g += 2) {  // (the first wait completes every load; later ones only tie registers)
    if (g + 1 < kN)
      asm volatile("tcgen05.wait::ld.sync.aligned;"
                   : FF_TIE8(32 * g), FF_TIE8(32 * g + 8), FF_TIE8(32 * g + 16), FF_TIE8(32 * g + 24),
                     FF_TIE8(32 * g + 32), FF_TIE8(32 * g + 40), FF_TIE8(32 * g + 48), FF_TIE8(32 * g + 56)::"memory");
    else
      asm volatile("tcgen05.wait::ld.sync.aligned;"
                   : FF_TIE8(32 * g), FF_TIE8(32 * g + 8), FF_TIE8(32 * g + 16), FF_TIE8(32 * g + 24)::"memory");
  }
#undef FF_TIE8
#pragma unroll
  for (int i = 0; i < 32 * kN; ++i) v[i] = __uint_as_float(r[i]);
}

// Two 32-column TMEM loads (e.g. the gate and up accumulators of a SwiGLU
// chunk) behind a single tcgen05.wait::ld; the registers are threaded through
// the wait so no consumer can be scheduled before it.
__device__ __forceinline__ void tmem_ld32x2(uint32_t taddr0, uint32_t taddr1, float (&v)[32], float (&w)[32]) {
  uint32_t r[32], q[32];
#define FF_LD32(dst, addr)                                                                                       \
  asm volatile(                                                                                                  \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "                                                                  \
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"                                                  \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                 \
      : "=r"(dst[0]), "=r"(dst[1]), "=r"(dst[2]), "=r"(dst[3]), "=r"(dst[4]), "=r"(dst[5]), "=r"(dst[6]),        \
        "=r"(dst[7]), "=r"(dst[8]), "=r"(dst[9]), "=r"(dst[10]), "=r"(dst[11]), "=r"(dst[12]), "=r"(dst[13]),    \
        "=r"(dst[14]), "=r"(dst[15]), "=r"(dst[16]), "=r"(dst[17]), "=r"(dst[18]), "=r"(dst[19]), "=r"(dst[20]), \
        "=r"(dst[21]), "=r"(dst[22]), "=r"(dst[23]), "=r"(dst[24]), "=r"(dst[25]), "=r"(dst[26]), "=r"(dst[27]), \
        "=r"(dst[28]), "=r"(dst[29]), "=r"(dst[30]), "=r"(dst[31])                                              \
      : "r"(addr))
  FF_LD32(r, taddr0);
  FF_LD32(q, taddr1);
#undef FF_LD32
#define FF_TIE8(x, o) "+r"(x[o]), "+r"(x[o + 1]), "+r"(x[o + 2]), "+r"(x[o + 3]), "+r"(x[o + 4]), "+r"(x[o + 5]), \
                      "+r"(x[o + 6]), "+r"(x[o + 7])
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : FF_TIE8(r, 0), FF_TIE8(r, 8), FF_TIE8(r, 16), FF_TIE8(r, 24), FF_TIE8(q, 0), FF_TIE8(q, 8),
                 FF_TIE8(q, 16), FF_TIE8(q, 24)::"memory");
#undef FF_TIE8
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    v[i] = __uint_as_float(r[i]);
    w[i] = __uint_as_float(q[i]);
  }
}

// ----------------------------------------------------------------------------
// UMMA descriptors (sm_100 "version 1" shared-memory matrix descriptors)
// ----------------------------------------------------------------------------
// K-major operand, 128B swizzle: rows of 64 bf16 (128 B), 8-row atoms of
// 1024 B stacked along M/N (SBO = 1024).  Used for A and for the intermediate C.
__device__ __forceinline__ uint64_t desc_kmajor_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)(1) << 16;                 // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;         // SBO
  d |= (uint64_t)1 << 46;                   // version = 1 (sm_100)
  d |= (uint64_t)2 << 61;                   // SWIZZLE_128B
  return d;
}
// MN-major operand, 128B swizzle, for row-major [K][N] weights loaded by TMA in
// boxes of 64 (N, contiguous) x kBoxK (K) elements.  Atoms: 8 K-rows x 128 B.
// SBO = stride between 8-row atoms along K (1024 B); LBO = stride between
// 64-column blocks along N (one full TMA box).
__device__ __forceinline__ uint64_t desc_mnmajor_sw128(uint32_t smem_addr, uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// Instruction descriptor: bf16 x bf16 -> fp32, M x N, A/B majorness.
__host__ __device__ constexpr uint32_t idesc_bf16(uint32_t M, uint32_t N, uint32_t a_mn_major,
                                                  uint32_t b_mn_major) {
  return (1u << 4)                 // D format f32
         | (1u << 7)               // A bf16
         | (1u << 10)              // B bf16
         | (a_mn_major << 15) | (b_mn_major << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

// ----------------------------------------------------------------------------
// misc math
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// two fp32 -> one packed pair of the chain's 2-byte storage type
__device__ __forceinline__ uint32_t pack2(bool f16, float lo, float hi) {
  return f16 ? pack_f16x2(lo, hi) : pack_bf16x2(lo, hi);
}
// instruction descriptor of a bf16 MMA switched to fp16 A/B (kind::f16: format 0 = f16, 1 = bf16)
__host__ __device__ constexpr uint32_t idesc_as(uint32_t idesc, bool f16) {
  return f16 ? (idesc & ~((1u << 7) | (1u << 10))) : idesc;
}
// 16-byte store into another CTA's shared memory (address from mapa)
__device__ __forceinline__ void st_cluster_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared::cluster.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
__device__ __forceinline__ void red_add_v4_f32(float* gaddr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(gaddr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t atom_add_relaxed_gpu_u32(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ uint32_t atom_add_acqrel_gpu_u32(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void st_shared_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_shared_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void red_add_release_gpu_u32(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ float4 ld_global_f4(const float* p) {
  float4 v;
  asm volatile("ld.global.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void st_global_v4(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

}  // namespace ff
