// Fused GEMM-chain kernel for sm_100a (FlashFuser dataflow, B200-native).
//
//   standard:  E[m,l] = act(A[m,k] @ B[k,n]) @ D[n,l]
//   gated:     E[m,l] = (silu(A @ B0) * (A @ B1)) @ D
//
// Reference semantics: fuseplan simulator.execute_plan (simulator.py:177-424)
// and the dsm_comm primitives it models (analyzer.py:331-354).
//
// Decomposition.  A "ring" of G CTAs shares the intermediate C of one 128-row
// M tile (cls_shuffle = G):
//   * each CTA owns a kLB-wide column slice of E that it accumulates in TMEM
//     over the whole N range of its split;
//   * N is walked in n-steps of G*kNB columns.  In n-step t ring member p runs
//     GEMM0 for its own kNB-wide chunk of C (TMEM accumulator, double
//     buffered), applies the activation / SwiGLU gate (all_exchange "Mul" of
//     the two branch accumulators) and writes bf16 C to shared memory in the
//     UMMA K-major 128B-swizzled layout -- directly the A operand of GEMM1;
//   * shuffle: every chunk reaches the other G-1 members, which multiply it
//     with the matching D rows into their E slice.  Two transports:
//       kMode 0 (DSM): cp.async.bulk shared::cta -> shared::cluster pushes
//         into 2 receive buffers per CTA, mbarrier complete_tx on landing,
//         counter credits for buffer reuse and landing acks for the source;
//         the ring is one thread-block cluster;
//       kMode 1 (L2): the chunk is TMA-stored to an L2-resident scratch and
//         the members TMA-load it as GEMM1's A operand; a per-chunk epoch
//         flag (st.release / ld.acquire, gpu scope) orders store and loads.
//         Requires a fully co-resident (cooperative) launch.
//     GEMM1 hops of n-step t are interleaved with GEMM0 k-blocks of n-step t+1;
//   * inter-cluster reduce: with S > 1 N splits the E tiles are combined with
//     red.global.add.v4.f32 into an fp32 workspace; the last of the S
//     contributors of a tile casts it to bf16 and re-zeroes it (split_finish;
//     simulator.py:371 "+=" into E); with S == 1 E is stored in bf16;
//   * persistent: each ring processes work units (m tile, l cluster, split)
//     unit = ring_id, ring_id + n_rings, ...; every counter is global across
//     units so the pipelines never drain between units.
//
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer (+TMEM alloc),
// w2 DSM push driver, w3 DSM receive recycler, w4..w7 epilogue.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "ptx.cuh"

namespace ff {

enum Act : int { ACT_IDENTITY = 0, ACT_RELU = 1, ACT_SILU = 2, ACT_GELU_TANH = 3 };
enum Xchg : int { XCHG_DSM = 0, XCHG_L2 = 1 };

struct ChainArgs {
  int M, N, K, L;
  int G;               // ring size
  int S;               // N splits
  int steps;           // n-steps per split
  int split_chunks;    // pair kernel: C chunks (kN0 columns) per N split, ceil(total / n_splits)
  int total_chunks;    // pair kernel: N / kN0 (the last split and its last n-step may be ragged)
  int m_tiles;         // ceil(M / 128)
  int l_clusters;      // L / (G * LB)
  int n_units;         // m_tiles * l_clusters * S
  int n_rings;         // rings launched (persistent)
  int act;
  uint32_t* dev_epoch; // workspace word: epoch of the last completed launch; this launch's flags use +1
  uint32_t* exit_cnt;  // workspace word (zero between launches): CTAs done; the last one advances dev_epoch
  __nv_bfloat16* E;    // output (S == 1)
  float* ws;           // fp32 accumulation workspace (S > 1)
  uint32_t* flags;     // L2 mode: [n_units][steps][G] chunk-ready flags
  float* slab;         // pair kernel: split-N exchange regions [E tile][split][16-B chunk][128 rows]
  uint32_t* tile_cnt;  // split-N arrival counters, one per 128-row E tile (zero between launches)
  __nv_bfloat16* c_debug;  // optional: dump of the bf16 intermediate (tests only)
  int defer;           // pair kernel: hops of step T that run after GEMM0(T+1) (< G)
  int defer_last;      // pair kernel: run the ring's last GEMM0 before all hops of the previous step
  int krot;            // pair kernel: rotate each member's GEMM0 k order by its ring position
  int prefetch;        // pair kernel: L2 prefetch distance for weight tiles (k-blocks / hops), 0 = off
  int finish_tma;      // pair kernel: split finish by bulk copies (one unit per ring, 128/S % 8 == 0)
  int c_slots;         // pair kernel: C exchange slots per ring member (scratch reused every c_slots n-steps)
  int wpolicy;         // pair kernel: L2 hint (L2Hint) for weight tiles and their L2 prefetches
  int cpolicy;         // pair kernel: L2 hint for the C exchange scratch (stores and loads)
  int epolicy;         // pair kernel: L2 hint for the E tile stores (E is never re-read by the kernel)
  int split_cl;        // L2 kernels: the S N splits of an E tile are one thread-block cluster and combine
                       // their fp32 partials by a DSM reduce-scatter (FF_XCHG_L2_DSMR)
  int tail_S;          // pair kernel: > 1 splits the last partial wave's units in N into tail_S units each
  int n_full;          // pair kernel, tail_S > 1: units before the tail units (a whole number of waves)
  int serp;            // pair kernel: a ring's odd units run their n-steps in reverse order, so the
                       // weights the previous unit read last (still in L2) are read first
  int discard;         // pair kernel: drop dead scratch from L2 without a DRAM write-back once its last
                       // reader is done: bit 0 the split-N exchange regions, bit 1 the C scratch
  __nv_bfloat16* cscratch;  // pair kernel: C exchange scratch base (row-major [regions * 256][kN0])
  // conv chain as implicit GEMM (conv_k1 > 1): A is an NHWC feature map read
  // through an im2col tensor map; GEMM0 k-block kb = (filter tap, 64-channel block)
  int conv_k1;         // filter size of the first convolution (0: plain A[M][K])
  int conv_H, conv_W;  // feature map height / width (M = batch * H * W output pixels)
  int conv_cblk;       // input channels / 64
  // 1x1 conv -> act -> conv2_k x conv2_k conv (conv2_k > 1; ring 1, one n-step):
  // C goes to the L2 scratch (NHWC) and GEMM1 k-block kb2 = (tap, 64-channel
  // block of C) reads an im2col box of it once the halo tiles are published
  int conv2_k;
  int conv2_cblk;      // oc1 / 64
  int f16;             // 2-byte storage is fp16 (else bf16): MMA input format, C / E packing
  unsigned long long* prof;  // optional diagnostics: per CTA [FF_PROF_STRIDE] = 16 wait-cycle counters + 16 globaltimer stamps
};

#define FF_PROF_STRIDE 32
// Stamp timeline slot `i` (16..31) of this CTA with the global nanosecond timer.
// Profile row of this CTA (the pair kernel redefines it to its virtual CTA index).
#define FF_PROF_ROW blockIdx.x
#define FF_STAMP(i)                                                        \
  do {                                                                     \
    if (args.prof) args.prof[(FF_PROF_ROW) * FF_PROF_STRIDE + (i)] = globaltimer_ns(); \
  } while (0)
// Accumulate the cycles spent in `stmt` into `acc` when profiling is on.
#define FF_TIMED(acc, stmt)                                           \
  do {                                                                \
    const unsigned long long _t0 = args.prof ? clock64() : 0ull;      \
    stmt;                                                             \
    if (args.prof) acc += clock64() - _t0;                            \
  } while (0)

// Activations on the MUFU tanh unit (tanh.approx.f32, rel. err ~2^-11, far
// below the bf16 rounding of C that follows): silu(x) = x*sigmoid(x) with
// sigmoid(x) = (1 + tanh(x/2)) / 2, gelu_tanh per its definition.  No IEEE
// division (whose FCHK slow path serialised the C drain, profiles/r01).
__device__ __forceinline__ float silu_fast(float x) {
  const float h = 0.5f * x;
  return fmaf(h, tanh_approx(h), h);
}
__device__ __forceinline__ float apply_act(int act, float x) {
  switch (act) {
    case ACT_RELU:
      return fmaxf(x, 0.0f);
    case ACT_SILU:
      return silu_fast(x);
    case ACT_GELU_TANH: {
      const float k0 = 0.7978845608028654f, k1 = 0.044715f;
      const float u = k0 * fmaf(k1 * x, x * x, x);
      const float h = 0.5f * x;
      return fmaf(h, tanh_approx(u), h);
    }
    default:
      return x;
  }
}

// Activation over a register fragment, the switch hoisted out of the loop.
template <int N>
__device__ __forceinline__ void apply_act_frag(int act, float (&v)[N]) {
  if (act == ACT_RELU) {
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = fmaxf(v[i], 0.0f);
  } else if (act == ACT_SILU) {
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = silu_fast(v[i]);
  } else if (act == ACT_GELU_TANH) {
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = apply_act(ACT_GELU_TANH, v[i]);
  }
}

// Launch epoch, kept on the device so that a launch captured in a CUDA graph
// gets a fresh epoch on every replay (a host-side epoch would be frozen into the
// graph and make the previous replay's ready flags look current).  Thread 0 of
// every CTA reads the previous launch's epoch before the setup barrier; after
// it, one idle thread counts the CTA in, and the last CTA to be counted (every
// CTA has read by then) publishes this launch's epoch -- off the critical path.
// Stream order keeps launches disjoint.
// Flags are waited on for equality with the epoch (each flag slot is written
// once per launch), so a slot last written any number of launches ago never
// reads as current; 0 is skipped because it is the zero-filled initial state.
__device__ __forceinline__ uint32_t epoch_begin(const ChainArgs& args) {
  const uint32_t e = ld_relaxed_gpu_u32(args.dev_epoch) + 1u;
  return e != 0u ? e : 1u;
}
__device__ __forceinline__ void epoch_publish(const ChainArgs& args, uint32_t epoch) {
  if (atom_add_acqrel_gpu_u32(args.exit_cnt, 1u) == gridDim.x * gridDim.y * gridDim.z - 1u) {
    *reinterpret_cast<volatile uint32_t*>(args.dev_epoch) = epoch;
    *reinterpret_cast<volatile uint32_t*>(args.exit_cnt) = 0u;
  }
}

// Split-N finish (the reference's inter_cluster_reduce "+=", simulator.py:
// 380-404, plus the final cast): called by the 128 epilogue threads of a CTA
// after its fp32 partial of E tile rows [row0, row0+128) x cols [col0, col0+kCols)
// has been issued into the workspace (TMA reduce-add by `issuer`, or red.add by
// every thread).  Each contributor bumps the tile's arrival counter.
//   shared == false: the S-th (last) arrival reads the finished sum, writes bf16
//     E and re-zeroes the tile and the counter.
//   shared == true (every contributor is in its ring's final unit, so spinning
//     cannot block another unit): each contributor waits for all S arrivals and
//     finishes the row slice [ticket*128/S, (ticket+1)*128/S); the last to
//     finish resets the counter.
// Either way the workspace is zero again when the kernel exits (no memset or
// cast kernel around the launch).  `row` = this thread's index 0..127.
template <int kCols>
__device__ __forceinline__ void split_finish(const ChainArgs& args, uint32_t* counter, uint32_t bcast, bool issuer,
                                             bool tma_reduce, int row0, int row, int col0, uint32_t bar_id,
                                             bool shared) {
  const uint32_t S = (uint32_t)args.S;
  if (!tma_reduce) __threadfence();  // this thread's red.add ops before the arrival
  named_bar_sync(bar_id, 128);
  if (issuer) {
    if (tma_reduce) bulk_wait0();   // reductions performed, not just read from smem
    fence_proxy_async_global();
    __threadfence();
    if (args.prof) args.prof[blockIdx.x * FF_PROF_STRIDE + 25] = globaltimer_ns();
    const uint32_t ticket = atom_add_acqrel_gpu_u32(counter, 1);
    if (shared) {
      uint32_t polls = 0;
      while (ld_acquire_gpu_u32(counter) < S)
        if (++polls == FF_WATCHDOG_POLLS) FF_WD_EXPIRED(ld_acquire_gpu_u32(counter));
    }
    st_shared_u32(bcast, ticket);
  }
  named_bar_sync(bar_id, 128);
  const uint32_t ticket = ld_shared_u32(bcast);
  if (!shared && ticket != S - 1) return;
  fence_proxy_async_global();
  const int r_lo = shared ? (int)(ticket * 128 / S) : 0;
  const int r_hi = shared ? (int)((ticket + 1) * 128 / S) : 128;
  // coalesced pass over rows [r_lo, r_hi) of the row-major [128][kCols] tile:
  // a warp covers 512 contiguous bytes of one row per access.
  constexpr int kV = kCols / 4;  // float4 per tile row
  const int n4 = (r_hi - r_lo) * kV;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
  for (int j0 = 0; j0 < n4; j0 += 128 * 16) {
    float4 f[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int idx = j0 + row + 128 * j;
      const int r = row0 + r_lo + idx / kV;
      f[j] = (idx < n4 && r < args.M) ? ld_global_f4(args.ws + (size_t)r * args.L + col0 + 4 * (idx % kV)) : z;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int idx = j0 + row + 128 * j;
      const int r = row0 + r_lo + idx / kV;
      if (idx < n4 && r < args.M) {
        const size_t off = (size_t)r * args.L + col0 + 4 * (idx % kV);
        *reinterpret_cast<uint2*>(args.E + off) = make_uint2(pack2(args.f16, f[j].x, f[j].y), pack2(args.f16, f[j].z, f[j].w));
        *reinterpret_cast<float4*>(args.ws + off) = z;
      }
    }
  }
  if (issuer) {
    if (!shared)
      *reinterpret_cast<volatile uint32_t*>(counter) = 0u;
    else if (atom_add_acqrel_gpu_u32(counter, 1) == 2 * S - 1)
      *reinterpret_cast<volatile uint32_t*>(counter) = 0u;  // every contributor is past its wait
  }
}

template <bool kGated, int kNB, int kLB, int kStages, int kMode>
struct ChainCfg {
  static constexpr int BM = 128;
  static constexpr int BK = 64;
  static constexpr int kCW = kNB;                      // columns of C in one chunk
  static constexpr int kAcc = kGated ? 2 * kNB : kNB;  // TMEM columns per C accumulator buffer
  static constexpr int kA_BYTES = BM * BK * 2;         // 16 KB (A tile, or a C tile in L2 mode)
  static constexpr int kB_BYTES = (kGated ? 2 : 1) * BK * kNB * 2;
  static constexpr int kD_BYTES = BK * kLB * 2;
  static constexpr int kG0_BYTES = kA_BYTES + kB_BYTES;
  static constexpr int kG1_BYTES = (kMode == XCHG_L2 ? kA_BYTES : 0) + kD_BYTES;
  static constexpr int kG1_DOFF = (kMode == XCHG_L2 ? kA_BYTES : 0);  // D offset inside a stage
  static constexpr int kSTAGE = kG0_BYTES > kG1_BYTES ? kG0_BYTES : kG1_BYTES;
  static constexpr int kCHUNK_BYTES = BM * kCW * 2;
  static constexpr int kRECV = (kMode == XCHG_DSM) ? 2 : 0;
  static constexpr int kOFF_OWN = kStages * kSTAGE;
  static constexpr int kOFF_RECV = kOFF_OWN + kCHUNK_BYTES;
  static constexpr int kOFF_BAR = kOFF_RECV + kRECV * kCHUNK_BYTES;
  static constexpr int kNUM_BARS = 2 * kStages + 13 + 9;  // 13 named barriers + 16 u32 counters
  static constexpr int kSMEM = kOFF_BAR + kNUM_BARS * 8 + 16 + 1024;  // +1024 alignment slack
  static constexpr int kTMEM_E = 2 * kAcc;
  static constexpr int kTMEM_COLS = 512;
  static_assert(2 * kAcc + kLB <= 512, "TMEM budget");
  static_assert(kCW % 64 == 0 && kLB % 64 == 0 && kLB <= 256, "tile shape");
  static_assert(kSTAGE % 1024 == 0 && kCHUNK_BYTES % 1024 == 0, "1024B alignment for SW128");
};

template <bool kGated, int kNB, int kLB, int kStages, int kMode>
__global__ void __launch_bounds__(256, 1)
    ff_chain_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB0,
                    const __grid_constant__ CUtensorMap tmB1, const __grid_constant__ CUtensorMap tmD,
                    const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmCs,
                    const __grid_constant__ CUtensorMap tmE, const __grid_constant__ CUtensorMap tmW,
                    const __grid_constant__ CUtensorMap tmSlab, const __grid_constant__ CUtensorMap tmEr,
                    const ChainArgs args) {
  using C = ChainCfg<kGated, kNB, kLB, kStages, kMode>;
  constexpr bool kDSM = (kMode == XCHG_DSM);
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_base = smem_u32(smem_raw);
  const uint32_t base = (raw_base + 1023u) & ~1023u;
  uint8_t* const smem_gen = smem_raw + (base - raw_base);

  // the previous launch's epoch, loaded first so its latency hides behind the setup
  const uint32_t epoch0 = threadIdx.x == 0 ? epoch_begin(args) : 0u;
  if (threadIdx.x == 0) FF_STAMP(16);
  const int warp = threadIdx.x / 32;
  const int G = args.G;
  // split clusters (FF_XCHG_L2_DSMR): CTA x = ((tile * G) + p) * S + split, cluster rank = split;
  // ring = tile + split * (m_tiles * l_clusters), so unit_of(0) of rank s is split s of the tile
  const int Sc = args.split_cl ? args.S : 1;
  const uint32_t p = kDSM ? cluster_rank() : (uint32_t)((blockIdx.x / Sc) % G);  // ring position
  const int ring = args.split_cl ? (int)(blockIdx.x / (Sc * G)) + (int)(blockIdx.x % Sc) * args.m_tiles * args.l_clusters
                                 : (int)(blockIdx.x / G);
  const int kblocks = args.K / C::BK;
  // GEMM0 k order rotated by ring position (members of a ring and the rings of
  // an m tile would otherwise request the same A box at the same moment)
  const int krot = args.krot ? ((int)p * kblocks / G) : 0;
  const int steps = args.steps;
  // units processed by this ring; the flat list of (unit, n-step) is the "global step" T
  const int my_units = ring < args.n_units ? (args.n_units - ring + args.n_rings - 1) / args.n_rings : 0;
  const int total_steps = my_units * steps;

  struct Unit {
    int m0, l0, n0, id;
  };
  auto unit_of = [&](int i) {  // i-th unit of this ring
    const int u = ring + i * args.n_rings;
    const int mt = u % args.m_tiles;
    const int rest = u / args.m_tiles;
    const int lc = rest % args.l_clusters;
    const int split = rest / args.l_clusters;
    return Unit{mt * C::BM, (lc * G + (int)p) * kLB, split * steps * G * kNB, u};
  };

  // barriers
  const uint32_t bar0 = base + C::kOFF_BAR;
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (kStages + s); };
  const uint32_t bx = bar0 + 8u * (2 * kStages);
  const uint32_t c_full[2] = {bx + 0, bx + 8};
  const uint32_t c_empty[2] = {bx + 16, bx + 24};
  const uint32_t own_full = bx + 32, own_free = bx + 40;
  const uint32_t recv_full[2] = {bx + 48, bx + 56};
  const uint32_t recv_used[2] = {bx + 64, bx + 72};
  const uint32_t e_full = bx + 80, e_empty = bx + 88, e_load = bx + 96;
  auto counter = [&](int h) { return bx + 104 + 4u * h; };  // 16 u32 counters
  const uint32_t ack_count = counter(0);                    // DSM: landed-chunk acks
  const uint32_t tmem_slot = bar0 + 8u * C::kNUM_BARS;
  const uint32_t own_slot = base + C::kOFF_OWN;
  const uint32_t recv_slot[2] = {base + C::kOFF_RECV, base + C::kOFF_RECV + C::kCHUNK_BYTES};

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(c_full[b], 1);
      mbar_init(c_empty[b], 128);
      mbar_init(recv_full[b], 1);
      mbar_init(recv_used[b], 1);
    }
    for (int h = 0; h < 16; ++h) *reinterpret_cast<volatile uint32_t*>(smem_gen + (counter(h) - base)) = 0u;
    mbar_init(own_full, 128);
    // own slot reusable after: MMA hop 0 commit + (DSM: all pushes acked | L2: TMA store done)
    mbar_init(own_free, (G == 1 && args.conv2_k <= 1) ? 1 : 2);
    mbar_init(e_full, 1);
    mbar_init(e_empty, 128);
    mbar_init(e_load, 1);
    fence_mbar_init();
    if (kDSM)
      for (int b = 0; b < 2; ++b) mbar_expect_tx(recv_full[b], C::kCHUNK_BYTES);
  }
  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB0);
    if (kGated) tma_prefetch_desc(&tmB1);
    tma_prefetch_desc(&tmD);
    if (!kDSM && (G > 1 || args.conv2_k > 1)) {
      tma_prefetch_desc(&tmC);
      tma_prefetch_desc(&tmCs);
    }
  }
  if (warp == 1) tmem_alloc<C::kTMEM_COLS>(tmem_slot);
  __shared__ uint32_t s_epoch;
  if (threadIdx.x == 0) s_epoch = epoch0;
  tc_fence_before();
  if (kDSM)
    cluster_sync();  // peers push into our buffers only after our barriers exist
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t*>(smem_gen + (tmem_slot - base));
  const uint32_t epoch = s_epoch;
  if (threadIdx.x == 96) epoch_publish(args, epoch);  // warp 3 lane 0: DSM recycler / idle
  if (threadIdx.x == 0) FF_STAMP(17);

  // slot h of global step T holds GEMM0 k-blocks [h*KB/G, (h+1)*KB/G) of step T+1
  // GEMM0 slice [h * kblocks / G, (h + 1) * kblocks / G) of hop h, walked incrementally (no
  // division per hop: the producer's and the MMA thread's issue latency is the pipeline's)
  struct Slices {
    int lo, hi, rem, q, r, G;
    __device__ void start() { lo = 0, hi = q, rem = r; if (rem >= G) rem -= G, ++hi; }
    __device__ void step() { lo = hi, hi += q, rem += r; if (rem >= G) rem -= G, ++hi; }
  };
  const Slices sl0{0, 0, 0, kblocks / G, kblocks % G, G};
  auto flag_addr = [&](const Unit& u, int t, int origin) {
    return args.flags + ((size_t)u.id * steps + t) * G + origin;
  };

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (elect_one()) {
      unsigned long long w_empty = 0, w_flag = 0;
      const unsigned long long t_start = clock64();
      int stage = 0, phase = 0;
      auto next = [&]() {
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      };
      auto load_gemm0 = [&](int T, int kb0, int kb1) {
        const Unit u = unit_of(T / steps);
        const int n0 = u.n0 + ((T % steps) * G + (int)p) * kNB;
        for (int kbl = kb0; kbl < kb1; ++kbl) {
          // staggered k order across ring members (no runtime division on the per-stage path)
          const int kb = kbl + krot < kblocks ? kbl + krot : kbl + krot - kblocks;
          FF_TIMED(w_empty, mbar_wait(empty_bar(stage), phase ^ 1));
          const uint32_t sb = base + stage * C::kSTAGE;
          mbar_expect_tx(full_bar(stage), C::kG0_BYTES);
          if (args.conv_k1 > 1) {
            // implicit GEMM: 128 output pixels x 64 channels of filter tap (r, s)
            const int cb = kb % args.conv_cblk, tap = kb / args.conv_cblk;
            const int pad = args.conv_k1 / 2, hw = args.conv_H * args.conv_W;
            const int img = u.m0 / hw, rem = u.m0 % hw;
            tma_load_im2col_4d(sb, &tmA, full_bar(stage), cb * 64, rem % args.conv_W - pad, rem / args.conv_W - pad,
                               img, (uint16_t)(tap % args.conv_k1), (uint16_t)(tap / args.conv_k1));
          } else {
            tma_load_2d(sb, &tmA, full_bar(stage), kb * C::BK, u.m0);
          }
          if (kGated) {
            tma_load_2d(sb + C::kA_BYTES, &tmB0, full_bar(stage), n0, kb * C::BK);
            tma_load_2d(sb + C::kA_BYTES + C::BK * kNB * 2, &tmB1, full_bar(stage), n0, kb * C::BK);
          } else {
            // one 3D box: kNB/64 MN-major [64 k x 64 n] tiles 8 KB apart (TMA is per-instruction bound)
            tma_load_3d(sb + C::kA_BYTES, &tmB0, full_bar(stage), 0, kb * C::BK, n0 / 64);
          }
          next();
        }
      };
      auto load_hop = [&](int T, int h) {
        const Unit u = unit_of(T / steps);
        const int t = T % steps;
        if (args.conv2_k > 1) {
          // wait for every 128-pixel tile the k2 x k2 window of this tile reaches
          const int pad = args.conv2_k / 2, W = args.conv_W;
          const int lo = max(0, u.m0 - pad * W - pad), hi = min(args.M - 1, u.m0 + C::BM - 1 + pad * W + pad);
          for (int tile = lo / C::BM; tile <= hi / C::BM; ++tile) {
            const uint32_t* f = args.flags + tile;  // unit id == m tile (ring 1, one step, one l cluster)
            uint32_t polls = 0;
            FF_TIMED(w_flag, while (ld_acquire_gpu_u32(f) != epoch) {
              if (++polls == FF_WATCHDOG_POLLS) FF_WD_EXPIRED(((unsigned long long)ld_acquire_gpu_u32(f) << 32) | epoch);
            });
          }
          fence_proxy_async_global();
          FF_STAMP(27);  // every halo tile's C published
          const int hw = args.conv_H * W, img = u.m0 / hw, rem = u.m0 % hw;
          const int nk = args.conv2_k * args.conv2_k * args.conv2_cblk;
          for (int kb2 = 0; kb2 < nk; ++kb2) {
            const int tap = kb2 / args.conv2_cblk, cb = kb2 % args.conv2_cblk;
            FF_TIMED(w_empty, mbar_wait(empty_bar(stage), phase ^ 1));
            const uint32_t sb = base + stage * C::kSTAGE;
            mbar_expect_tx(full_bar(stage), C::kG1_BYTES);
            tma_load_im2col_4d(sb, &tmC, full_bar(stage), cb * 64, rem % W - pad, rem / W - pad, img,
                               (uint16_t)(tap % args.conv2_k), (uint16_t)(tap / args.conv2_k));
            tma_load_3d(sb + C::kG1_DOFF, &tmD, full_bar(stage), 0, kb2 * C::BK, u.l0 / 64);
            next();
          }
          return;
        }
        const int origin = (int)p >= h ? (int)p - h : (int)p - h + G;
        const int nrow0 = u.n0 + (t * G + origin) * kNB;
        const bool remote_c = !kDSM && h > 0;
        if (remote_c) {
          // wait until ring member `origin` published chunk (unit, t)
          const uint32_t* f = flag_addr(u, t, origin);
          uint32_t polls = 0;
          FF_TIMED(w_flag, while (ld_acquire_gpu_u32(f) != epoch) {
            if (++polls == FF_WATCHDOG_POLLS) FF_WD_EXPIRED(((unsigned long long)ld_acquire_gpu_u32(f) << 32) | epoch);
          });
          fence_proxy_async_global();
        }
        for (int kb2 = 0; kb2 < C::kCW / C::BK; ++kb2) {
          FF_TIMED(w_empty, mbar_wait(empty_bar(stage), phase ^ 1));
          const uint32_t sb = base + stage * C::kSTAGE;
          mbar_expect_tx(full_bar(stage), remote_c ? C::kG1_BYTES : C::kD_BYTES);
          if (remote_c) tma_load_2d(sb, &tmC, full_bar(stage), nrow0 + kb2 * C::BK, u.m0);
          tma_load_3d(sb + C::kG1_DOFF, &tmD, full_bar(stage), 0, nrow0 + kb2 * C::BK, u.l0 / 64);
          next();
        }
      };
      if (total_steps > 0) load_gemm0(0, 0, kblocks);
      for (int T = 0; T < total_steps; ++T) {
        Slices sl = sl0;
        sl.start();
        for (int h = 0; h < G; ++h, sl.step()) {
          if (T + 1 < total_steps) load_gemm0(T + 1, sl.lo, sl.hi);
          load_hop(T, h);
        }
      }
      if (args.prof) {
        unsigned long long* pr = args.prof + blockIdx.x * FF_PROF_STRIDE;
        pr[0] = clock64() - t_start;
        pr[1] = w_empty;
        pr[2] = w_flag;
      }
    }
    // The other 31 lanes wait here, not in a spin loop of their own: two divergent spin-wait
    // paths in one warp can starve the role lane (found on hardware in the pair kernel).
    __syncwarp();
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (elect_one()) {
      unsigned long long w_full0 = 0, w_full1 = 0, w_cempty = 0, w_own = 0, w_eempty = 0;
      const unsigned long long t_start = clock64();
      int stage = 0, phase = 0;
      auto next = [&]() {
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      };
      const uint32_t idesc0 = idesc_as(idesc_bf16(128, kNB, 0, 1), args.f16);
      const uint32_t idesc1 = idesc_as(idesc_bf16(128, kLB, 0, 1), args.f16);
      auto gemm0 = [&](int T, int kb0, int kb1) {
        const int cb = T & 1;
        if (kb0 == 0) {
          FF_TIMED(w_cempty, mbar_wait(c_empty[cb], ((T >> 1) & 1) ^ 1));
          tc_fence_after();
        }
        const uint32_t tacc = tmem_base + cb * C::kAcc;
        for (int kb = kb0; kb < kb1; ++kb) {
          FF_TIMED(w_full0, mbar_wait(full_bar(stage), phase));
          tc_fence_after();
          const uint32_t sb = base + stage * C::kSTAGE;
#pragma unroll
          for (int kk = 0; kk < C::BK / 16; ++kk) {
            const uint64_t ad = desc_kmajor_sw128(sb + kk * 32);
            const uint32_t acc = (kb | kk) ? 1u : 0u;
            if (kGated) {
              const uint64_t b0 = desc_mnmajor_sw128(sb + C::kA_BYTES + kk * 2048, 8192);
              const uint64_t b1 = desc_mnmajor_sw128(sb + C::kA_BYTES + C::BK * kNB * 2 + kk * 2048, 8192);
              umma_bf16(tacc, ad, b0, idesc0, acc);
              umma_bf16(tacc + kNB, ad, b1, idesc0, acc);
            } else {
              const uint64_t bd = desc_mnmajor_sw128(sb + C::kA_BYTES + kk * 2048, 8192);
              umma_bf16(tacc, ad, bd, idesc0, acc);
            }
          }
          umma_commit(empty_bar(stage));
          next();
        }
        if (kb1 == kblocks) umma_commit(c_full[cb]);
      };
      int ri = 0;
      bool e_started = false;
      auto hop = [&](int T, int t, int h) {
        if (t == 0 && h == 0) {
          // new unit: the epilogue must have drained the previous unit's E tile
          const int ui = T / steps;
          if (ui > 0) {
            FF_TIMED(w_eempty, mbar_wait(e_empty, (ui - 1) & 1));
            tc_fence_after();
          }
          e_started = false;
        }
        uint32_t slot = 0;
        int b = 0;
        if (h == 0) {
          FF_TIMED(w_own, mbar_wait(own_full, T & 1));
          slot = own_slot;
        } else if (kDSM) {
          b = ri & 1;
          mbar_wait_cluster(recv_full[b], (ri >> 1) & 1);
          slot = recv_slot[b];
        }
        tc_fence_after();
        const bool from_stage = (!kDSM && h > 0) || args.conv2_k > 1;
        const int nk = args.conv2_k > 1 ? args.conv2_k * args.conv2_k * args.conv2_cblk : C::kCW / C::BK;
        for (int kb2 = 0; kb2 < nk; ++kb2) {
          FF_TIMED(w_full1, mbar_wait(full_bar(stage), phase));
          tc_fence_after();
          const uint32_t sb = base + stage * C::kSTAGE;
          const uint32_t ab = from_stage ? sb : slot + kb2 * (C::BM * C::BK * 2);
#pragma unroll
          for (int kk = 0; kk < C::BK / 16; ++kk) {
            const uint64_t ad = desc_kmajor_sw128(ab + kk * 32);
            const uint64_t bd = desc_mnmajor_sw128(sb + C::kG1_DOFF + kk * 2048, 8192);
            umma_bf16(tmem_base + C::kTMEM_E, ad, bd, idesc1, e_started ? 1u : 0u);
            e_started = true;
          }
          umma_commit(empty_bar(stage));
          next();
        }
        if (h == 0) {
          umma_commit(own_free);
        } else if (kDSM) {
          umma_commit(recv_used[b]);
          ++ri;
        }
        if (t == steps - 1 && h == G - 1) umma_commit(e_full);
      };
      if (total_steps > 0) gemm0(0, 0, kblocks);
      for (int T = 0; T < total_steps; ++T) {
        const int t = T % steps;  // once per step
        Slices sl = sl0;
        sl.start();
        for (int h = 0; h < G; ++h, sl.step()) {
          if (T + 1 < total_steps) gemm0(T + 1, sl.lo, sl.hi);
          hop(T, t, h);
        }
      }
      if (args.prof) {
        unsigned long long* pr = args.prof + blockIdx.x * FF_PROF_STRIDE;
        pr[3] = clock64() - t_start;
        pr[4] = w_full0;
        pr[5] = w_full1;
        pr[6] = w_cempty;
        pr[7] = w_own;
        pr[8] = w_eempty;
      }
    }
    __syncwarp();  // see warp 0
  } else if (warp == 2) {
    // ===== DSM shuffle, send side: direct pushes of the own chunk (kMode 0) =====
    // At hop h ring member q consumes the chunk of origin (q-h) mod G, so
    // origin p pushes to (p+h) mod G in hop order.  Receiver q's global receive
    // index R = T*(G-1) + h-1 selects buffer R & 1; reusing a buffer needs a
    // credit (remote increment of counter h) sent once q consumed receive R-2.
    if (kDSM && G > 1 && elect_one()) {
      for (int T = 0; T < total_steps; ++T) {
        mbar_wait(own_full, T & 1);
        for (int h = 1; h < G; ++h) {
          const uint32_t dest = p + h < (uint32_t)G ? p + h : p + h - G;
          const int R = T * (G - 1) + h - 1;
          if (R >= 2) {
            const int first = (3 - h) <= 0 ? 0 : (3 - h + G - 2) / (G - 1);
            credit_wait(counter(h), (uint32_t)(T - first + 1));
          }
          const int b = R & 1;
          dsm_bulk_push(mapa(recv_slot[b], dest), own_slot, C::kCHUNK_BYTES, mapa(recv_full[b], dest));
        }
        // a shared::cta -> shared::cluster bulk copy completes only through the
        // destination's mbarrier, so the own slot is free once all receivers acked.
        credit_wait(ack_count, (uint32_t)((T + 1) * (G - 1)));
        mbar_arrive(own_free);
      }
    }
    __syncwarp();  // see warp 0
  } else if (warp == 3) {
    // ===== DSM shuffle, receive side: ack landing, recycle, credit (kMode 0) =====
    if (kDSM && G > 1 && elect_one()) {
      const int total = total_steps * (G - 1);
      // h = R % (G-1) + 1 and hn = (R+2) % (G-1) + 1 walked incrementally (no division per receive)
      int h = 1, hn = 2 % (G - 1) + 1;
      for (int R = 0; R < total; ++R) {
        const int b = R & 1;
        const uint32_t ph = (R >> 1) & 1;
        mbar_wait_cluster(recv_full[b], ph);
        credit_add_remote(mapa(ack_count, (int)p >= h ? p - h : p + G - h));
        mbar_wait(recv_used[b], ph);
        if (R + 2 < total) {
          mbar_expect_tx(recv_full[b], C::kCHUNK_BYTES);
          credit_add_remote(mapa(counter(hn), (int)p >= hn ? p - hn : p + G - hn));
        }
        h = h == G - 1 ? 1 : h + 1;
        hn = hn == G - 1 ? 1 : hn + 1;
      }
    }
    __syncwarp();  // see warp 0
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    const int q = warp & 3;  // TMEM lane quadrant
    const int row = q * 32 + (int)lane_id();
    const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16);
    unsigned long long w_cfull = 0, w_ofree = 0, t_e = 0;
    const unsigned long long t_start = clock64();
    for (int T = 0; T < total_steps; ++T) {
      const Unit u = unit_of(T / steps);
      const int t = T % steps;
      const int cb = T & 1;
      FF_TIMED(w_cfull, mbar_wait(c_full[cb], (T >> 1) & 1));
      if (warp == 4 && lane_id() == 0 && T == 0) FF_STAMP(18);  // C chunk 0 accumulated
      tc_fence_after();
      FF_TIMED(w_ofree, mbar_wait(own_free, (T & 1) ^ 1));
      const uint32_t tacc = lane_base + cb * C::kAcc;
#pragma unroll 1
      for (int c0 = 0; c0 < C::kCW; c0 += 16) {
        float v[16];
        tmem_ld16(tacc + c0, v);
        if (kGated) {
          float w[16];
          tmem_ld16(tacc + kNB + c0, w);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = silu_fast(v[i]) * w[i];
        } else {
          apply_act_frag(args.act, v);
        }
        uint32_t pk[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) pk[i] = pack2(args.f16, v[2 * i], v[2 * i + 1]);
        const int sub = c0 / 64;
        const int ch = (c0 % 64) / 8;  // 16-byte chunk inside the 128-byte row
        const uint32_t rowb = own_slot + sub * (C::BM * C::BK * 2) + row * 128;
        st_shared_v4(rowb + ((ch ^ (row & 7)) << 4), pk[0], pk[1], pk[2], pk[3]);
        st_shared_v4(rowb + (((ch + 1) ^ (row & 7)) << 4), pk[4], pk[5], pk[6], pk[7]);
        if (args.c_debug != nullptr && u.m0 + row < args.M) {
          const int ncol = u.n0 + (t * G + (int)p) * kNB + c0;
          uint4* dst = reinterpret_cast<uint4*>(args.c_debug + (size_t)(u.m0 + row) * args.N + ncol);
          dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        }
      }
      if (warp == 4 && lane_id() == 0 && T == 0) FF_STAMP(19);  // C chunk 0 drained to shared memory
      tc_fence_before();
      mbar_arrive(c_empty[cb]);
      fence_proxy_async_smem();
      mbar_arrive(own_full);
      if (!kDSM && (G > 1 || args.conv2_k > 1)) {
        // publish the chunk through L2: TMA store, then release the ready flag
        named_bar_sync(1, 128);
        if (warp == 4 && lane_id() == 0) {
          const int ncol = u.n0 + (t * G + (int)p) * kNB;
#pragma unroll
          for (int sub = 0; sub < C::kCW / 64; ++sub)
            tma_store_2d(&tmCs, own_slot + sub * (C::BM * C::BK * 2), ncol + 64 * sub, u.m0);
          bulk_commit();
          bulk_wait0();
          fence_proxy_async_global();
          st_release_gpu_u32(flag_addr(u, t, (int)p), epoch);
          if (T == 0) FF_STAMP(20);  // C chunk 0 stored to L2 and its flag released
          mbar_arrive(own_free);
        }
        __syncwarp();  // lanes 1-31 must not spin on the next barrier while the issuer publishes
      }
      if (t == steps - 1) {
        // E tile of this unit: TMEM -> registers -> global
        const unsigned long long t_e0 = args.prof ? clock64() : 0ull;
        mbar_wait(e_full, (T / steps) & 1);
        if (warp == 4 && lane_id() == 0) FF_STAMP(30);  // E accumulated (last hop)
        tc_fence_after();
        // E tile through the own slot (free once hop 0, the pushes / the C store are done)
        // in SW128 16 KB tiles, leaving by bulk tensor ops: bf16 TMA stores (S == 1) or
        // fp32 TMA reduce-adds into the split-N workspace (per-thread rows would be 32
        // scattered lines per warp access; measured ~16 GB/s per SM with red.global.add)
        const bool f32 = args.S > 1;
        const int cpt = f32 ? 32 : 64;  // columns per 16 KB tile
        // the ring's final unit stages the whole tile at once in the drained pipeline
        // stages (no load follows); earlier units use the own slot in rounds, once it
        // is free (hop 0 read it, pushes acked / C store done)
        const bool final_unit = (T / steps) == my_units - 1;
        const bool issuer = (warp == 4 && lane_id() == 0);
        if (args.split_cl) continue;  // one unit per ring: the DSM reduce-scatter below (all warps)
        if (final_unit && args.finish_tma) {
          // Split-N reduce-scatter through exchange regions (as the pair kernel's tail):
          // row slice j (R = 128/S rows) of the E tile belongs to split j; rows of other
          // slices go from TMEM registers straight to this split's region as coalesced
          // 512-byte warp stores ([16-byte chunk][128 rows]), own rows to shared memory;
          // after the (tile, split) flags the partners' rows arrive by TMA (128-byte inner
          // boxes), the S partials are summed in split order (deterministic) and one TMA
          // store writes the rows.  No atomics: measured 12.6 MB of TMA reduce-adds for
          // GPT-2s took ~4.5 us of L2 reduction throughput.
          const int S = args.S, R = C::BM / S;
          const int sp = u.id / (args.m_tiles * args.l_clusters);  // this unit's split
          const int tile = (u.m0 / C::BM) * (args.L / kLB) + u.l0 / kLB;
          constexpr int kChunks = kLB / 4;
          const int slice = row / R;
          float* const dst = args.slab + ((size_t)tile * S + sp) * (kChunks * 128 * 4) + row * 4;
          const uint32_t own_row = base + sp * (R * kChunks * 16) + (row - sp * R) * 16;
          auto put16 = [&](int c0, const float* v) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int ch = c0 / 4 + j;
              if (slice != sp)
                st_global_v4(dst + (size_t)ch * 512, __float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]),
                             __float_as_uint(v[4 * j + 2]), __float_as_uint(v[4 * j + 3]));
              else
                st_shared_v4(own_row + ch * (R * 16), __float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]),
                             __float_as_uint(v[4 * j + 2]), __float_as_uint(v[4 * j + 3]));
            }
          };
#pragma unroll 1
          for (int c0 = 0; c0 < kLB;) {
            if (kLB - c0 >= 64) {
              float v[32], w[32];
              tmem_ld32x2(lane_base + C::kTMEM_E + c0, lane_base + C::kTMEM_E + c0 + 32, v, w);
              put16(c0, v);
              put16(c0 + 16, v + 16);
              put16(c0 + 32, w);
              put16(c0 + 48, w + 16);
              c0 += 64;
            } else {
              float v[16];
              tmem_ld16(lane_base + C::kTMEM_E + c0, v);
              put16(c0, v);
              c0 += 16;
            }
          }
          tc_fence_before();
          mbar_arrive(e_empty);
          named_bar_sync(1, 128);  // all region stores issued before the issuer's release (cumulative)
          if (issuer) FF_STAMP(24);
          uint32_t* const flags = args.flags + (1u << 17) + tile * 16;
          if (issuer) {
            st_release_gpu_u32(flags + sp, epoch);
            uint32_t polls = 0;
            for (int j = 0; j < S; ++j) {
              if (j == sp) continue;
              while (ld_relaxed_gpu_u32(flags + j) != epoch)
                if (++polls == FF_WATCHDOG_POLLS) FF_WD_EXPIRED(((unsigned long long)ld_relaxed_gpu_u32(flags + j) << 32) | epoch);
            }
            fence_acq_rel_gpu();
            fence_proxy_async_global();
            if (args.prof) args.prof[blockIdx.x * FF_PROF_STRIDE + 25] = globaltimer_ns();
            mbar_expect_tx(e_load, (uint32_t)((S - 1) * R * kChunks * 16));
            for (int j = 0; j < S; ++j)
              if (j != sp)
                tma_load_3d(base + j * (R * kChunks * 16), &tmSlab, e_load, 0, sp * R / 8, (tile * S + j) * kChunks);
          }
          __syncwarp();  // the issuer's lanes wait for it here, not spinning on own_free / e_load
          mbar_wait(own_free, T & 1);  // the own slot stages the bf16 rows (DSM pushes read it until acked)
          mbar_wait(e_load, 0);
          // sum in split order, cast, stage [kLB/64][R][128 B] SW128 for one TMA store
          const uint8_t* const src = smem_gen;
          const uint32_t ebuf = own_slot;
          const int n_items = R * kChunks;
#pragma unroll 1
          for (int it0 = row; it0 < n_items; it0 += 512) {
            float4 acc[4];
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
              acc[q4] = it0 + 128 * q4 < n_items ? *reinterpret_cast<const float4*>(src + (it0 + 128 * q4) * 16)
                                                 : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
            for (int j = 1; j < S; ++j) {
#pragma unroll
              for (int q4 = 0; q4 < 4; ++q4) {
                if (it0 + 128 * q4 >= n_items) continue;
                const float4 f = *reinterpret_cast<const float4*>(src + j * (R * kChunks * 16) + (it0 + 128 * q4) * 16);
                acc[q4].x += f.x;
                acc[q4].y += f.y;
                acc[q4].z += f.z;
                acc[q4].w += f.w;
              }
            }
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              const int it = it0 + 128 * q4;
              if (it >= n_items) continue;
              const int c = it / R, rr = it % R;
              const int ch = (c % 16) / 2;
              *reinterpret_cast<uint2*>(smem_gen + (ebuf - base) + (c / 16) * (R * 128) + rr * 128 +
                                        ((ch ^ (rr & 7)) << 4) + (c & 1) * 8) =
                  make_uint2(pack2(args.f16, acc[q4].x, acc[q4].y), pack2(args.f16, acc[q4].z, acc[q4].w));
            }
          }
          fence_proxy_async_smem();
          named_bar_sync(1, 128);
          if (issuer) {
            tma_store_3d(&tmEr, ebuf, 0, u.m0 + sp * R, u.l0 / 64);
            bulk_commit();
            FF_STAMP(26);
          }
          if (args.prof) t_e += clock64() - t_e0;
          continue;
        }
        if (!final_unit) mbar_wait(own_free, T & 1);
        const uint32_t stg = final_unit ? base : own_slot;
        const int tpr = final_unit ? (C::kOFF_OWN / 16384) : (C::kCHUNK_BYTES / 16384);  // tiles per round
#pragma unroll 1
        for (int g0 = 0; g0 < kLB; g0 += cpt * tpr) {
          const int g1 = min(kLB, g0 + cpt * tpr);
          // 16 columns of this thread's row into the SW128 staging tile
          auto stage16 = [&](int c0, const float* v) {
            const uint32_t rowb = stg + ((c0 - g0) / cpt) * 16384 + row * 128;
            if (f32) {
              const int j0 = (c0 % 32) / 4;
#pragma unroll
              for (int j = 0; j < 4; ++j)
                st_shared_v4(rowb + (((j0 + j) ^ (row & 7)) << 4), __float_as_uint(v[4 * j]),
                             __float_as_uint(v[4 * j + 1]), __float_as_uint(v[4 * j + 2]),
                             __float_as_uint(v[4 * j + 3]));
            } else {
              uint32_t pk[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) pk[i] = pack2(args.f16, v[2 * i], v[2 * i + 1]);
              const int j0 = (c0 % 64) / 8;
              st_shared_v4(rowb + ((j0 ^ (row & 7)) << 4), pk[0], pk[1], pk[2], pk[3]);
              st_shared_v4(rowb + (((j0 + 1) ^ (row & 7)) << 4), pk[4], pk[5], pk[6], pk[7]);
            }
          };
#pragma unroll 1
          for (int c0 = g0; c0 < g1; c0 += 16) {
            float v[16];
            tmem_ld16(lane_base + C::kTMEM_E + c0, v);
            stage16(c0, v);
          }
          fence_proxy_async_smem();
          named_bar_sync(1, 128);
          if (issuer) {
            for (int c = g0; c < g1; c += cpt) {
              const uint32_t tile = stg + ((c - g0) / cpt) * 16384;
              if (f32)
                tma_reduce_add_2d(&tmW, tile, u.l0 + c, u.m0);
              else
                tma_store_2d(&tmE, tile, u.l0 + c, u.m0);
            }
            bulk_commit();
            bulk_wait_read0_group();
          }
          named_bar_sync(1, 128);
        }
        tc_fence_before();
        mbar_arrive(e_empty);
        if (warp == 4 && lane_id() == 0) FF_STAMP(24);  // E staged and its bulk ops issued
        if (args.S > 1)
          split_finish<kLB>(args, args.tile_cnt + (u.m0 / C::BM) * (args.L / kLB) + u.l0 / kLB, tmem_slot + 8,
                            issuer, true, u.m0, row, u.l0, 1, args.n_units <= args.n_rings);
        if (warp == 4 && lane_id() == 0) FF_STAMP(26);  // split-N finish done
        if (args.prof) t_e += clock64() - t_e0;
      }
    }
    if (warp == 4 && lane_id() == 0) bulk_wait0();  // E stores / reduce-adds performed before exit
    if (args.prof && warp == 4 && lane_id() == 0) {
      unsigned long long* pr = args.prof + blockIdx.x * FF_PROF_STRIDE;
      pr[9] = clock64() - t_start;
      pr[10] = w_cfull;
      pr[11] = w_ofree;
      pr[14] = t_e;
    }
  }

  if (!kDSM && args.split_cl && total_steps > 0) {
    // ============ split-N DSM reduce-scatter (all 8 warps, FF_XCHG_L2_DSMR) ============
    // The paper's dsm_comm reduce_scatter (analyzer.py:348, simulator.py:363-367) on the
    // S fp32 E partials of one tile, one per CTA of the cluster: row slice j (R = 128/S
    // rows) belongs to cluster rank j.  Every thread takes half of one row's columns from
    // TMEM and stores them with st.shared::cluster into the owner's drained pipeline
    // stages, slot [source split][R rows][kLB], 16-byte chunks XOR-swizzled by row (8
    // consecutive rows of a warp hit distinct bank groups).  After a cluster barrier each
    // CTA sums the S partials of its rows in split order (deterministic, bit-reproducible),
    // casts and writes its E rows: no fp32 workspace, no flags, no atomics.
    const int S = args.S, R = C::BM / S;
    const Unit u = unit_of(my_units - 1);
    const int sp = (int)cluster_rank();
    const int wq = warp & 3;
    const int row = wq * 32 + (int)lane_id();
    const uint32_t lane_base = tmem_base + ((uint32_t)(wq * 32) << 16);
    const int c_lo = warp < 4 ? kLB / 2 : 0;
    mbar_wait(e_full, (my_units - 1) & 1);
    __syncwarp();
    tc_fence_after();
    if (threadIdx.x == 128) FF_STAMP(30);
    cluster_sync();  // every CTA's MMAs retired: all stage areas are free to receive
    const uint32_t dst_rank = (uint32_t)(row / R);
    const uint32_t dst_row = base + (uint32_t)((sp * R + row % R) * kLB * 4);
    const uint32_t rdst = dst_rank == (uint32_t)sp ? dst_row : mapa(dst_row, dst_rank);
#pragma unroll 1
    for (int c0 = c_lo; c0 < c_lo + kLB / 2; c0 += 32) {
      float v[32];
      tmem_ld32(lane_base + C::kTMEM_E + c0, v);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t a = rdst + ((((c0 / 4 + j) ^ (row & 7))) << 4);
        if (dst_rank == (uint32_t)sp)
          st_shared_v4(a, __float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]), __float_as_uint(v[4 * j + 2]),
                       __float_as_uint(v[4 * j + 3]));
        else
          st_cluster_v4(a, __float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]), __float_as_uint(v[4 * j + 2]),
                        __float_as_uint(v[4 * j + 3]));
      }
    }
    cluster_sync();  // partials of this CTA's rows have landed (release / acquire at cluster scope)
    if (threadIdx.x == 128) FF_STAMP(24);
    constexpr int kChunks = kLB / 4;  // 16-byte chunks per row
    const int rows_here = min(R, args.M - (u.m0 + sp * R));
#pragma unroll 1
    for (int it = (int)threadIdx.x; it < R * kChunks; it += 256) {
      const int rr = it / kChunks, c = it % kChunks;
      if (rr >= rows_here) break;
      const uint32_t off = (uint32_t)(rr * kLB * 4) + (((c ^ (rr & 7))) << 4);
      float4 a = ld_shared_f4(base + off);
#pragma unroll 1
      for (int j = 1; j < S; ++j) {  // splits in order
        const float4 f = ld_shared_f4(base + (uint32_t)(j * R * kLB * 4) + off);
        a.x += f.x;
        a.y += f.y;
        a.z += f.z;
        a.w += f.w;
      }
      const size_t e_off = (size_t)(u.m0 + sp * R + rr) * args.L + u.l0 + 4 * c;
      *reinterpret_cast<uint2*>(args.E + e_off) = make_uint2(pack2(args.f16, a.x, a.y), pack2(args.f16, a.z, a.w));
    }
    if (threadIdx.x == 128) FF_STAMP(26);
  }
  __syncthreads();
  if (kDSM) cluster_sync();  // no CTA leaves while a peer may still push or credit
  if (threadIdx.x == 0) FF_STAMP(31);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kTMEM_COLS>(tmem_base);
  }
}

}  // namespace ff
