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

const char* ff_dsm_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
