/*
 * ff_dsm_bench.h -- DSM bandwidth microbenchmark (calibrates the dsm.bandwidth[n]
 * entries of the B200 device profile; the reference consumes these as
 * profile inputs, hardware.py:150-275, paper Fig. 4 / Fig. 13 method).
 */
#ifndef FF_DSM_BENCH_H
#define FF_DSM_BENCH_H
#ifdef __cplusplus
extern "C" {
#endif

/* Ring push benchmark: `num_clusters` clusters of `cluster` CTAs; every CTA
 * pushes `iters` chunks of `chunk_bytes` to its right neighbour with `depth`
 * transfers in flight.  Writes the elapsed milliseconds. */
int ff_dsm_push_bench(int cluster, int chunk_bytes, int depth, int iters, int num_clusters, float* ms_out);

/* cudaOccupancyMaxActiveClusters for a `cluster`-CTA launch using `smem_bytes`. */
int ff_max_active_clusters(int cluster, int smem_bytes, int* out);

/* TMA streaming benchmark (per-SM operand feed vs box shape): `ctas` CTAs each
 * stream `iters` stages of `stage_bytes` from a bf16 [rows][cols] matrix in 3D
 * boxes {64, box_rows & 0xffff, box_rows >> 16} (2D {64, box_rows} when the high
 * half is 0) with `stages` in flight and `producers` issuing threads. */
int ff_tma_stream_bench(const void* mat, int rows, int cols, int stages, int iters, int box_rows, int ctas,
                        int producers, int stage_bytes, float* ms_out);

/* Same with TMA multicast: clusters of `csize` CTAs; each CTA fetches 1/csize of
 * every {64, box_rows, box_blocks} box and multicasts it to the whole cluster.
 * flags (csize == 1): bit0 plain non-cluster launch, bit1 producer waits with CTA
 * scope, bit2 consumer arrives locally (else acquire/release.cluster forms). */
int ff_tma_mcast_bench(const void* mat, int rows, int cols, int stages, int iters, int box_rows, int box_blocks,
                       int csize, int ctas, int stage_bytes, int flags, float* ms_out);

/* Diagnostics: one 1-thread kernel writing %globaltimer (ns) to *dst on `stream`;
 * brackets a launch on the GPU's own clock (launch latency / drain tail). */
int ff_stamp_globaltimer(void* dst, void* stream);

/* Diagnostics: an empty kernel with a chain kernel's launch shape (`ctas` x 256
 * threads, `smem_bytes` dynamic smem, clusters of `cluster`, optional 512-column
 * TMEM alloc/dealloc); CTA i writes entry/exit %globaltimer to stamps[2i], [2i+1]. */
int ff_launch_probe(void* stamps, int ctas, int smem_bytes, int cluster, int tmem, void* stream);

/* Diagnostics: `ctas` one-warp CTAs spinning on clock64 for `cycles` (keeps the
 * stream busy without touching memory, so a following launch sees a warm L2). */
int ff_spin(long long cycles, int ctas, void* stream);

/* DSM communication primitives (paper SIII-B dsm_comm; csrc/dsm_primitives.cuh) on one
 * fp32 tile of `floats_per_cta` per CTA, `clusters` clusters of `cluster` CTAs, `iters`
 * back-to-back repetitions (ms_out: event time of the launch).  op: 0 reduce-scatter
 * (Add), 1 all-gather, 2 all-exchange (Add), 3 all-exchange (Mul: silu(gate) * up over
 * CTA pairs), 4 one shuffle-ring hop.  in / out: device [cluster*clusters][floats_per_cta]. */
int ff_dsm_primitive_run(int op, int cluster, int floats_per_cta, int clusters, const float* in, float* out,
                         int iters, float* ms_out);

const char* ff_dsm_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
