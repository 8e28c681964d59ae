/*
 * ff_chain.h -- C ABI of the B200-native fused GEMM-chain runtime.
 *
 * This is the drop-in boundary for the execution path of the reference
 * planner `fuseplan` (arXiv 2512.12949 front-end).  The reference executes a
 * fusion plan with a numpy tile replay; these entry points execute the same
 * plan on an sm_100a GPU.  Plain C types only: no torch / no C++ in the
 * signatures.  All pointers are device pointers unless stated otherwise;
 * `stream` is a cudaStream_t (NULL = legacy default stream).
 *
 * Reference interfaces replaced (file:line in /root/reference/pkg/src/fuseplan):
 *   ff_chain_run_plan      <- simulator.execute_plan      (simulator.py:177-424)
 *                             (called by simulator.verify  simulator.py:461-487,
 *                              search refine               search.py:527-536,
 *                              cli simulate                cli.py:232-249)
 *   ff_plan_lower          <- plan.plan_geometry           (plan.py:222-268)
 *                             + structural_violations      (plan.py:271-324)
 *                             (the plan -> launch geometry step)
 *   ff_chain_launch        <- the per-cluster replay loop  (simulator.py:276-409)
 *                             with an explicit physical configuration
 *   ff_chain_workspace_bytes <- fits_execution_budget      (simulator.py:137-140)
 *   status codes            <- errors.py:1-61 (PlanError / CapacityExceeded /
 *                             FusePlanError); never abort the process.
 */
#ifndef FF_CHAIN_H
#define FF_CHAIN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; mapped back to the reference exception classes in Python */
#define FF_OK 0
#define FF_ERR_PLAN 1        /* PlanError: structurally invalid plan / rule violation */
#define FF_ERR_CAPACITY 2    /* CapacityExceeded: does not fit on-chip */
#define FF_ERR_UNSUPPORTED 3 /* valid plan, but no kernel lowering for it */
#define FF_ERR_CUDA 4        /* CUDA runtime / driver failure */
#define FF_ERR_ARG 5         /* bad argument (null pointer, misaligned, ...) */

/* workload.py:26-32 */
#define FF_KIND_STANDARD 0
#define FF_KIND_GATED 1
#define FF_ACT_IDENTITY 0
#define FF_ACT_RELU 1
#define FF_ACT_SILU 2
#define FF_ACT_GELU_TANH 3 /* extension: GPT-2 FFN (not in the reference catalog) */

/* plan.py:27-30 */
#define FF_LOWERING_NA 0
#define FF_LOWERING_SPATIAL_SPLIT 1
#define FF_LOWERING_DOUBLED_K 2

/* storage / MMA input type of a 2-byte chain (fp32 accumulation either way) */
#define FF_DTYPE_BF16 0
#define FF_DTYPE_F16 1

/* ChainGraph (workload.py:75-110): kind, dims (m,n,k,l), activation. */
typedef struct ffChainDesc {
  int32_t kind;
  int32_t activation;
  int64_t m, n, k, l;
  int32_t element_size; /* bytes per stored scalar; only 2 (bf16 / fp16) executes on the GPU */
  int32_t dtype;        /* FF_DTYPE_BF16 (default, 0) or FF_DTYPE_F16: A, B, D, E and the intermediate C */
} ffChainDesc;

/* FusionPlan (plan.py:121-165).  Dimension index order is (m, n, k, l) = DIMS. */
typedef struct ffPlanDesc {
  uint32_t spatial_mask;   /* bit i set <=> DIMS[i] is spatial */
  int32_t temporal[4];     /* temporal order, outermost first, as DIMS indices */
  int32_t n_temporal;
  int64_t block[4];        /* tiles.block */
  int32_t cluster[4];      /* tiles.cluster: cls_m, cls_n, cls_k, cls_l */
  int32_t gated_lowering;  /* FF_LOWERING_* */
} ffPlanDesc;

/* Shuffle transport of the intermediate C between ring members. */
#define FF_XCHG_DSM 0 /* distributed shared memory pushes inside a thread-block cluster */
#define FF_XCHG_L2 1  /* TMA store / TMA load through an L2-resident scratch (cooperative launch) */
#define FF_XCHG_L2_PAIR 2 /* as FF_XCHG_L2, ring members are CTA pairs issuing cta_group::2 M=256 MMAs */
#define FF_XCHG_L2_DSMR 3 /* as FF_XCHG_L2 (1-CTA members), and the n_splits (2..8) N splits of every E tile
                             form one thread-block cluster that sums their fp32 partials by a DSM
                             reduce-scatter (the paper's dsm_comm reduce_scatter); one unit per ring */

/* Physical launch configuration produced by the lowering. */
typedef struct ffKernelConfig {
  int32_t ring;        /* CTAs sharing one C tile (cls_shuffle of the plan) */
  int32_t n_splits;    /* N splits whose E partials are reduced across rings (inter-cluster reduce) */
  int32_t nb;          /* C chunk width per CTA per n-step (columns) */
  int32_t lb;          /* E columns owned by one CTA (TMEM accumulator width) */
  int32_t exchange;    /* FF_XCHG_DSM | FF_XCHG_L2 | FF_XCHG_L2_PAIR | FF_XCHG_L2_DSMR */
  int32_t m_tiles;     /* derived: ceil(m / 128) */
  int32_t l_clusters;  /* derived: l / (ring * lb) */
  int32_t steps;       /* derived: n-steps per split */
  int32_t units;       /* derived: m_tiles * l_clusters * n_splits work units */
  int32_t rings;       /* derived: co-resident rings launched (persistent over units) */
  int32_t grid_ctas;   /* derived: CTAs launched (rings * ring * CTAs per member) */
} ffKernelConfig;

/* Tensors: row-major, the reference layouts (simulator.py:112-123):
 * A[m,k], B[k,n] (standard) or B0[k,n], B1[k,n] (gated), D[n,l], E[m,l]; bf16 or fp16 (ffChainDesc.dtype). */
typedef struct ffTensors {
  const void* a;
  const void* b;  /* B (standard) or B0 (gated) */
  const void* b1; /* B1 (gated), NULL otherwise */
  const void* d;
  void* e;
} ffTensors;

/* Conv chain (ConvChainConfig, workload.py:168-199): conv(k1 x k1, stride 1,
 * same padding) -> activation -> conv(1 x 1).  The reference lowers it to a
 * GEMM chain over an explicit im2col matrix (conv_chain_to_gemm,
 * workload.py:191-199: m = h*w, k = ic*k1^2, n = oc1, l = oc2); here GEMM0
 * reads the NHWC feature map itself through an im2col TMA tensor map
 * (implicit GEMM, no im2col matrix in HBM).  Tensors for ff_conv_chain_launch:
 *   a = X  [batch][h][w][ic]      (NHWC)
 *   b = W1 [k1][k1][ic][oc1]      (= [k1*k1*ic][oc1] row-major, tap-major K)
 *   d = W2 [oc1][oc2]             (1x1 conv)
 *   e = Y  [batch][h][w][oc2]     (NHWC)
 * k1 > 1 needs ic % 64 == 0 and the dsm / l2 exchange (1-CTA kernels). */
typedef struct ffConvDesc {
  int32_t batch, h, w, ic, oc1, oc2, k1, k2;
  int32_t activation; /* FF_ACT_* applied between the convolutions (ReLU in the reference) */
  int32_t dtype;      /* FF_DTYPE_BF16 or FF_DTYPE_F16 */
} ffConvDesc;

/* GEMM-chain view of a conv chain (m = batch*h*w unpadded). */
int ff_conv_chain_desc(const ffConvDesc* conv, ffChainDesc* out);
/* Physical launch configuration for a conv chain under `exchange`. */
int ff_conv_chain_lower(const ffConvDesc* conv, int32_t num_sms, int32_t exchange, ffKernelConfig* out);
size_t ff_conv_chain_workspace_bytes(const ffConvDesc* conv, const ffKernelConfig* cfg);
/* Replaces execute_plan (simulator.py:177) on a conv preset's chain, reading
 * X instead of its im2col matrix.  `cfg` from ff_conv_chain_lower or from
 * ff_plan_lower_ex on ff_conv_chain_desc. */
int ff_conv_chain_launch(const ffConvDesc* conv, const ffKernelConfig* cfg, const ffTensors* t, void* workspace,
                         size_t ws_bytes, void* stream);

/* Lower a reference plan to a physical launch (no GPU work).  The plan's
 * cls_shuffle ring becomes one thread-block cluster exchanging C over DSM. */
int ff_plan_lower(const ffChainDesc* chain, const ffPlanDesc* plan, int32_t num_sms, ffKernelConfig* out);

/* Same, with an explicit shuffle transport (FF_XCHG_DSM | FF_XCHG_L2). */
int ff_plan_lower_ex(const ffChainDesc* chain, const ffPlanDesc* plan, int32_t num_sms, int32_t exchange,
                     ffKernelConfig* out);

/* Choose the physical launch for a chain without a reference plan (L2 transport). */
int ff_auto_config(const ffChainDesc* chain, int32_t num_sms, ffKernelConfig* out);

/* Same, with an explicit shuffle transport. */
int ff_auto_config_ex(const ffChainDesc* chain, int32_t num_sms, int32_t exchange, ffKernelConfig* out);

/* Workspace (device bytes) the launch needs.  The workspace must be zero-filled
 * once when first allocated; it never needs clearing again (the L2 transport's
 * ready flags are epoch-stamped; split-N counters and the fp32 E region are
 * re-zeroed by the last contributor of each tile).  Launches that may run
 * concurrently (different streams) need separate workspaces. */
size_t ff_chain_workspace_bytes(const ffChainDesc* chain, const ffKernelConfig* cfg);

/* Execute the fused chain with an explicit physical configuration.
 * Stream-ordered, no host synchronisation, no allocation. */
int ff_chain_launch(const ffChainDesc* chain, const ffKernelConfig* cfg, const ffTensors* t, void* workspace,
                    size_t workspace_bytes, void* stream);

/* Lower + launch in one call: the drop-in for simulator.execute_plan.  The plan
 * is lowered under the first transport that executes it (CTA pairs, then the
 * 1-CTA L2 and DSM kernels); ff_plan_workspace_bytes sizes its workspace
 * (0 when the plan has no lowering: ff_chain_run_plan then reports why). */
size_t ff_plan_workspace_bytes(const ffChainDesc* chain, const ffPlanDesc* plan);
int ff_chain_run_plan(const ffChainDesc* chain, const ffPlanDesc* plan, const ffTensors* t, void* workspace,
                      size_t workspace_bytes, void* stream);

/* Debug variant of ff_chain_launch that also writes the bf16 intermediate C[m,n]. */
int ff_chain_launch_debug(const ffChainDesc* chain, const ffKernelConfig* cfg, const ffTensors* t,
                          void* workspace, size_t workspace_bytes, void* c_out, void* stream);

/* Validate an explicit launch (ring, n_splits, nb, lb, exchange) for `chain` and fill its derived
 * fields (m_tiles, l_clusters, steps, units, rings, grid_ctas) as ff_chain_launch will; no GPU work. */
int ff_config_finish(const ffChainDesc* chain, int32_t num_sms, ffKernelConfig* cfg);

/* *out = 1 when a launch of `cfg` (derived fields recomputed for `chain`, as ff_chain_launch does)
 * writes a bit-identical E on every run with the same inputs: no N splits, the DSM reduce-scatter
 * of the splits (FF_XCHG_L2_DSMR), or the CTA-pair kernel's exchange-region finish (one unit per
 * ring); *out = 0 when the N-split partials meet through TMA reduce-adds, whose order follows the
 * CTAs' timing (results agree to fp32 rounding, not bitwise).  Host logic only (no GPU work);
 * describes the planned ring count, i.e. a device where it is co-resident.  Deterministic-mode
 * selection: paper_2512_12949_b200.runtime.lower(..., deterministic=True). */
int ff_config_deterministic(const ffChainDesc* chain, const ffKernelConfig* cfg, int32_t num_sms, int32_t* out);

/* Number of CUDA kernels one ff_chain_launch issues (for launch accounting). */
int ff_chain_kernel_count(const ffChainDesc* chain, const ffKernelConfig* cfg);

/* Diagnostics: device buffer of unsigned long long[grid_ctas][32] that receives
 * per-CTA wait-cycle counters (slots 0-15) and globaltimer stamps (16-31) on
 * every launch (NULL disables; default). */
void ff_set_profile_buffer(void* dev_ptr);

/* Kernel-variant selection (process-wide; default 0 = the tuned kernels), for
 * A/B measurements and the tests that pin every variant against the oracle. */
#define FF_VARIANT_NO_KROT 0x1u          /* common GEMM0 k order in every ring member */
#define FF_VARIANT_NO_QUAD 0x2u          /* plain CTA pairs, no weight-multicast quads */
#define FF_VARIANT_FORCE_QUAD 0x4u       /* quads whenever they can launch */
#define FF_VARIANT_FINISH_REGIONS 0x8u   /* 1-CTA kernels: split-N finish through exchange regions */
#define FF_VARIANT_WEIGHTS_EVICT_FIRST 0x10u /* pair kernel: weight tiles + prefetches with L2 evict_first */
#define FF_VARIANT_SCRATCH_NORMAL 0x20u      /* pair kernel: C exchange scratch with the default L2 priority */
#define FF_VARIANT_WEIGHTS_EVICT_LAST 0x40u  /* pair kernel: weight tiles + prefetches with L2 evict_last */
#define FF_VARIANT_NO_DISCARD 0x80u          /* pair kernel: keep dead exchange scratch in L2 (no discard) */
#define FF_VARIANT_SCRATCH_DISCARD 0x100u    /* pair kernel: also discard the C exchange scratch at exit */
#define FF_VARIANT_NO_SERP 0x200u            /* pair kernel: every unit walks its n-steps in order */
#define FF_VARIANT_E_EVICT_FIRST 0x400u      /* pair kernel: E tile stores with L2 evict_first */
#define FF_VARIANT_NO_TAIL_SPLIT 0x800u      /* pair kernel: keep the last partial wave's units whole */
void ff_set_variant(uint32_t flags);

/* Thread-local message for the last non-OK status. */
const char* ff_last_error(void);

/* Library version string. */
const char* ff_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FF_CHAIN_H */
