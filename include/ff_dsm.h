/*
 * ff_dsm.h -- the DSM communication primitives of the fused chain (paper
 * SIII-B dsm_comm; the reference models their bytes in analyzer.py:331-354
 * and executes them as numpy sums in simulator.py:349,364-367,386-402) run on
 * their own, for tests and for calibrating the dsm.bandwidth[n] entries of
 * the B200 device profile (hardware.py:150-275 grammar).
 */
#ifndef FF_DSM_H
#define FF_DSM_H
#ifdef __cplusplus
extern "C" {
#endif

/* DSM primitives (csrc/dsm_primitives.cuh) on one fp32 tile of `floats_per_cta` per
 * CTA, `clusters` clusters of `cluster` CTAs, `iters` back-to-back repetitions
 * (ms_out: event time of the launch).  op: 0 reduce-scatter (Add), 1 all-gather,
 * 2 all-exchange (Add), 3 all-exchange (Mul: silu(gate) * up over CTA pairs),
 * 4 one shuffle-ring hop.  in / out: device [cluster*clusters][floats_per_cta]. */
int ff_dsm_primitive_run(int op, int cluster, int floats_per_cta, int clusters, const float* in, float* out,
                         int iters, float* ms_out);

/* DSM fabric bandwidth: every CTA of all co-resident clusters of `cluster` CTAs moves
 * data to its right neighbour.  mode 0: bulk push (cp.async.bulk shared::cta ->
 * shared::cluster) from `issuers` (1-4) issuing threads, each with `depth` receive slots
 * of `chunk_bytes` (credit-recycled, issuers*depth*chunk bytes in flight); mode 1:
 * ld.shared::cluster.v4 pull by 256 threads; mode 2: st.shared::cluster.v4 remote
 * stores by 256 threads (modes 1/2 move 128 KiB per CTA per iteration).  Writes the
 * number of co-resident clusters and the event time of the launch. */
int ff_dsm_bandwidth(int mode, int cluster, int chunk_bytes, int depth, int issuers, int iters, int* clusters_out,
                     float* ms_out);

const char* ff_dsm_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* FF_DSM_H */
