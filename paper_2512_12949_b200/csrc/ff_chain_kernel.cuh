// Fused GEMM-chain kernel for sm_100a (FlashFuser dataflow, B200-native).
//
//   standard:  E[m,l] = act(A[m,k] @ B[k,n]) @ D[n,l]
//   gated:     E[m,l] = (silu(A @ B0) * (A @ B1)) @ D
//
// Reference semantics: fuseplan simulator.execute_plan (simulator.py:177-424)
// and the dsm_comm primitives it models (analyzer.py:331-354).
//
// Decomposition (one cluster = one shuffle ring of G CTAs, cls_shuffle = G):
//   * every CTA owns 128 rows of M (tcgen05 M=128, TMEM lane = row) and a
//     kLB-wide column slice of E that it accumulates in TMEM for the whole
//     N range of its split (the E tile never leaves the SM until the store);
//   * N is walked in "n-steps" of G*kNB columns.  In n-step t, ring member p
//     runs GEMM0 for its own kNB-wide chunk of the intermediate C (TMEM C
//     accumulator, double buffered across n-steps), applies the activation /
//     SwiGLU gate and writes bf16 C into shared memory in the UMMA K-major
//     128B-swizzled layout (so the tile is directly the A operand of GEMM1);
//   * dsm_shuffle: every chunk is pushed over distributed shared memory to
//     the other G-1 ring members (cp.async.bulk shared::cta -> shared::cluster
//     with mbarrier complete_tx, 2 receive buffers, per-hop credit counters).
//     At hop h a CTA multiplies the chunk that originated at ring member
//     (p-h) mod G with the matching D rows into its E tile; the hops of n-step
//     t are interleaved with the GEMM0 k-blocks of n-step t+1;
//   * inter-cluster reduce: when N is split across S clusters the E tiles
//     are combined with red.global.add.v4.f32 into an fp32 workspace, then a
//     finalize kernel casts to bf16 (simulator.py:371 "+=" into E).
//
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer (+TMEM alloc),
// w2 DSM push driver, w3 DSM buffer recycler / credits, w4..w7 epilogue.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "ptx.cuh"

namespace ff {

enum Act : int { ACT_IDENTITY = 0, ACT_RELU = 1, ACT_SILU = 2, ACT_GELU_TANH = 3 };

struct ChainArgs {
  int M, N, K, L;
  int G;               // ring size (CTAs per cluster)
  int S;               // N splits across clusters
  int steps;           // n-steps per split
  int m_tiles;         // ceil(M / 128)
  int l_clusters;      // L / (G * LB)
  int act;
  __nv_bfloat16* E;    // output (used when S == 1)
  float* ws;           // fp32 accumulation workspace (used when S > 1)
  __nv_bfloat16* c_debug;  // optional: dump of the bf16 intermediate (tests only)
  int dbg;                 // debug switches (FF_DEBUG_FLAGS), 0 in production
};

__device__ __forceinline__ float apply_act(int act, float x) {
  switch (act) {
    case ACT_RELU:
      return fmaxf(x, 0.0f);
    case ACT_SILU:
      return x / (1.0f + __expf(-x));
    case ACT_GELU_TANH: {
      const float k0 = 0.7978845608028654f, k1 = 0.044715f;
      float u = k0 * (x + k1 * x * x * x);
      return 0.5f * x * (1.0f + tanhf(u));
    }
    default:
      return x;
  }
}

template <bool kGated, int kNB, int kLB, int kStages>
struct ChainCfg {
  static constexpr int BM = 128;
  static constexpr int BK = 64;
  static constexpr int kCW = kNB;                  // width of one C chunk (columns of C)
  static constexpr int kAcc = kGated ? 2 * kNB : kNB;  // TMEM columns per C accumulator buffer
  static constexpr int kA_BYTES = BM * BK * 2;     // 16 KB
  static constexpr int kB_BYTES = (kGated ? 2 : 1) * BK * kNB * 2;
  static constexpr int kD_BYTES = BK * kLB * 2;
  static constexpr int kG0_BYTES = kA_BYTES + kB_BYTES;
  static constexpr int kSTAGE = kG0_BYTES > kD_BYTES ? kG0_BYTES : kD_BYTES;
  static constexpr int kCHUNK_BYTES = BM * kCW * 2;  // one bf16 C chunk
  static constexpr int kOFF_OWN = kStages * kSTAGE;
  static constexpr int kOFF_RECV = kOFF_OWN + kCHUNK_BYTES;
  static constexpr int kOFF_BAR = kOFF_RECV + 2 * kCHUNK_BYTES;
  static constexpr int kNUM_BARS = 2 * kStages + 13 + 9;  // 13 named barriers + 16 u32 credit counters
  static constexpr int kSMEM = kOFF_BAR + kNUM_BARS * 8 + 16 + 1024;  // +1024 alignment slack
  static constexpr int kTMEM_E = 2 * kAcc;          // E accumulator column offset
  static constexpr int kTMEM_COLS = 512;
  static_assert(2 * kAcc + kLB <= 512, "TMEM budget");
  static_assert(kCW % 64 == 0 && kLB % 64 == 0 && kLB <= 256, "tile shape");
  static_assert(kSTAGE % 1024 == 0 && kCHUNK_BYTES % 1024 == 0, "1024B alignment for SW128");
};

template <bool kGated, int kNB, int kLB, int kStages>
__global__ void __launch_bounds__(256, 1)
    ff_chain_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB0,
                    const __grid_constant__ CUtensorMap tmB1, const __grid_constant__ CUtensorMap tmD,
                    const ChainArgs args) {
  using C = ChainCfg<kGated, kNB, kLB, kStages>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment for the 128B swizzle atoms.
  const uint32_t raw_base = smem_u32(smem_raw);
  const uint32_t base = (raw_base + 1023u) & ~1023u;
  uint8_t* const smem_gen = smem_raw + (base - raw_base);

  const int warp = threadIdx.x / 32;
  const uint32_t p = cluster_rank();  // ring position
  const int G = args.G;

  // cluster -> (m tile, l cluster, n split); m fastest so concurrent clusters share weight tiles in L2
  const int cidx = blockIdx.x / G;
  const int mt = cidx % args.m_tiles;
  const int rest = cidx / args.m_tiles;
  const int lc = rest % args.l_clusters;
  const int split = rest / args.l_clusters;
  const int m0 = mt * C::BM;
  const int l0 = (lc * G + (int)p) * kLB;
  const int n_split0 = split * args.steps * G * kNB;
  const int kblocks = args.K / C::BK;
  const int steps = args.steps;

  // barrier addresses
  const uint32_t bar0 = base + C::kOFF_BAR;
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (kStages + s); };
  const uint32_t bx = bar0 + 8u * (2 * kStages);
  const uint32_t c_full[2] = {bx + 0, bx + 8};
  const uint32_t c_empty[2] = {bx + 16, bx + 24};
  const uint32_t own_full = bx + 32, own_free = bx + 40;
  const uint32_t recv_full[2] = {bx + 48, bx + 56};
  const uint32_t recv_used[2] = {bx + 64, bx + 72};
  const uint32_t e_full = bx + 96;
  auto credit = [&](int h) { return bx + 104 + 4u * h; };  // u32 counters, h = 1..G-1
  const uint32_t ack_count = credit(0);  // landed-chunk acknowledgements from receivers
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
    for (int h = 0; h < 16; ++h) *reinterpret_cast<volatile uint32_t*>(smem_gen + (credit(h) - base)) = 0u;
    mbar_init(own_full, 128);
    mbar_init(own_free, G > 1 ? 2 : 1);
    mbar_init(e_full, 1);
    fence_mbar_init();
    // receive buffers armed for their first use
    for (int b = 0; b < 2; ++b) mbar_expect_tx(recv_full[b], C::kCHUNK_BYTES);
  }
  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB0);
    if (kGated) tma_prefetch_desc(&tmB1);
    tma_prefetch_desc(&tmD);
  }
  if (warp == 1) tmem_alloc<C::kTMEM_COLS>(tmem_slot);
  tc_fence_before();
  // barriers of every CTA must be initialised before any peer pushes into them
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t*>(smem_gen + (tmem_slot - base));

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (elect_one()) {
      int stage = 0, phase = 0;
      auto next = [&]() {
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      };
      // Loads follow the MMA issue order exactly: GEMM0(t+1) k-blocks are
      // interleaved with GEMM1(t) ring hops (slot h = k-blocks [h*KB/G, (h+1)*KB/G)).
      auto load_gemm0 = [&](int t, int kb0, int kb1) {
        const int n0 = n_split0 + (t * G + (int)p) * kNB;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(empty_bar(stage), phase ^ 1);
          const uint32_t sb = base + stage * C::kSTAGE;
          mbar_expect_tx(full_bar(stage), C::kG0_BYTES);
          tma_load_2d(sb, &tmA, full_bar(stage), kb * C::BK, m0);
          if (kGated) {
            tma_load_2d(sb + C::kA_BYTES, &tmB0, full_bar(stage), n0, kb * C::BK);
            tma_load_2d(sb + C::kA_BYTES + C::BK * kNB * 2, &tmB1, full_bar(stage), n0, kb * C::BK);
          } else {
#pragma unroll
            for (int j = 0; j < kNB / 64; ++j)
              tma_load_2d(sb + C::kA_BYTES + j * 8192, &tmB0, full_bar(stage), n0 + 64 * j, kb * C::BK);
          }
          next();
        }
      };
      auto load_hop = [&](int t, int h) {
        const int origin = ((int)p - h + G) % G;
        const int nrow0 = n_split0 + (t * G + origin) * kNB;
        for (int kb2 = 0; kb2 < C::kCW / C::BK; ++kb2) {
          mbar_wait(empty_bar(stage), phase ^ 1);
          const uint32_t sb = base + stage * C::kSTAGE;
          mbar_expect_tx(full_bar(stage), C::kD_BYTES);
#pragma unroll
          for (int j = 0; j < kLB / 64; ++j)
            tma_load_2d(sb + j * 8192, &tmD, full_bar(stage), l0 + 64 * j, nrow0 + kb2 * C::BK);
          next();
        }
      };
      load_gemm0(0, 0, kblocks);
      for (int t = 0; t < steps; ++t) {
        for (int h = 0; h < G; ++h) {
          const int s0 = (args.dbg & 8) ? (h ? kblocks : 0) : h * kblocks / G;
          const int s1 = (args.dbg & 8) ? kblocks : (h + 1) * kblocks / G;
          if (t + 1 < steps) load_gemm0(t + 1, s0, s1);
          load_hop(t, h);
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (elect_one()) {
      int stage = 0, phase = 0;
      auto next = [&]() {
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      };
      constexpr uint32_t idesc0 = idesc_bf16(128, kNB, 0, 1);
      constexpr uint32_t idesc1 = idesc_bf16(128, kLB, 0, 1);
      auto gemm0 = [&](int t, int kb0, int kb1) {
        const int cb = t & 1;
        if (kb0 == 0) {
          mbar_wait(c_empty[cb], ((t >> 1) & 1) ^ 1);
          tc_fence_after();
        }
        const uint32_t tacc = tmem_base + cb * C::kAcc;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(full_bar(stage), phase);
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
      auto hop = [&](int t, int h) {
        uint32_t slot;
        int b = 0;
        if (h == 0) {
          mbar_wait(own_full, t & 1);
          slot = own_slot;
        } else {
          b = ri & 1;
          mbar_wait_cluster(recv_full[b], (ri >> 1) & 1);
          slot = recv_slot[b];
        }
        tc_fence_after();
        for (int kb2 = 0; kb2 < C::kCW / C::BK; ++kb2) {
          mbar_wait(full_bar(stage), phase);
          tc_fence_after();
          const uint32_t sb = base + stage * C::kSTAGE;
          const uint32_t ab = slot + kb2 * (C::BM * C::BK * 2);
#pragma unroll
          for (int kk = 0; kk < C::BK / 16; ++kk) {
            const uint64_t ad = desc_kmajor_sw128(ab + kk * 32);
            const uint64_t bd = desc_mnmajor_sw128(sb + kk * 2048, 8192);
            umma_bf16(tmem_base + C::kTMEM_E, ad, bd, idesc1, e_started ? 1u : 0u);
            e_started = true;
          }
          umma_commit(empty_bar(stage));
          next();
        }
        if (h == 0) {
          umma_commit(own_free);
        } else {
          umma_commit(recv_used[b]);
          ++ri;
        }
      };
      gemm0(0, 0, kblocks);
      for (int t = 0; t < steps; ++t) {
        for (int h = 0; h < G; ++h) {
          const int s0 = (args.dbg & 8) ? (h ? kblocks : 0) : h * kblocks / G;
          const int s1 = (args.dbg & 8) ? kblocks : (h + 1) * kblocks / G;
          if (t + 1 < steps) gemm0(t + 1, s0, s1);
          hop(t, h);
        }
      }
      umma_commit(e_full);
    }
  } else if (warp == 2) {
    // ============ dsm_shuffle, send side: direct pushes of the own chunk ============
    // At hop h ring member q consumes the chunk of origin (q-h) mod G, so origin
    // p pushes its chunk to (p+h) mod G in hop order; no store-and-forward chain.
    // Receiver q's global receive index R = t*(G-1) + h-1 selects buffer R & 1;
    // reusing a buffer needs a credit (remote increment of counter h) sent by
    // the receiver once it consumed receive R-2.
    if (G > 1 && elect_one()) {
      for (int t = 0; t < steps; ++t) {
        mbar_wait(own_full, t & 1);
        for (int h = 1; h < G; ++h) {
          const uint32_t dest = (p + h) % G;
          const int R = t * (G - 1) + h - 1;
          if (R >= 2) {
            // credits on counter h arrive once per step from step `first` on
            const int first = (3 - h) <= 0 ? 0 : (3 - h + G - 2) / (G - 1);
            credit_wait(credit(h), (uint32_t)(t - first + 1));
          }
          if (args.dbg & 2) asm volatile("fence.proxy.async;" ::: "memory");
          const int b = R & 1;
          dsm_bulk_push(mapa(recv_slot[b], dest), own_slot, C::kCHUNK_BYTES, mapa(recv_full[b], dest));
        }
        // A shared::cta -> shared::cluster bulk copy completes only through the
        // destination's mbarrier (it is not a bulk-group op), so the own slot is
        // free once every receiver acknowledged that its copy landed.
        credit_wait(ack_count, (uint32_t)((t + 1) * (G - 1)));
        mbar_arrive(own_free);
      }
    }
  } else if (warp == 3) {
    // ============ dsm_shuffle, receive side: recycle buffers, credit the next writer ============
    if (G > 1 && elect_one()) {
      const int total = steps * (G - 1);
      for (int R = 0; R < total; ++R) {
        const int b = R & 1;
        const uint32_t ph = (R >> 1) & 1;
        // landed: acknowledge to the origin so it may overwrite its own slot
        mbar_wait_cluster(recv_full[b], ph);
        const int h = R % (G - 1) + 1;
        credit_add_remote(mapa(ack_count, (p + G - h) % G));
        // consumed: re-arm the buffer and credit the writer of receive R+2
        mbar_wait(recv_used[b], ph);
        if (R + 2 < total) {
          mbar_expect_tx(recv_full[b], C::kCHUNK_BYTES);
          const int hn = (R + 2) % (G - 1) + 1;
          const uint32_t writer = (p + G - hn) % G;
          credit_add_remote(mapa(credit(hn), writer));
        }
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    const int q = warp & 3;  // TMEM lane quadrant
    const int row = q * 32 + (int)lane_id();
    const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16);
    for (int t = 0; t < steps; ++t) {
      const int cb = t & 1;
      mbar_wait(c_full[cb], (t >> 1) & 1);
      tc_fence_after();
      mbar_wait(own_free, (t & 1) ^ 1);
      if (args.dbg & 4) {
        const long long t0 = clock64();
        while (clock64() - t0 < 40000) {
        }
      }
      const uint32_t tacc = lane_base + cb * C::kAcc;
#pragma unroll 1
      for (int c0 = 0; c0 < C::kCW; c0 += 16) {
        float v[16];
        tmem_ld16(tacc + c0, v);
        if (kGated) {
          float u[16];
          tmem_ld16(tacc + kNB + c0, u);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = (v[i] / (1.0f + __expf(-v[i]))) * u[i];
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = apply_act(args.act, v[i]);
        }
        uint32_t pk[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) pk[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
        const int sub = c0 / 64;
        const int ch = (c0 % 64) / 8;  // 16-byte chunk index inside the 128-byte row
        const uint32_t rowb = own_slot + sub * (C::BM * C::BK * 2) + row * 128;
        st_shared_v4(rowb + (((ch) ^ (row & 7)) << 4), pk[0], pk[1], pk[2], pk[3]);
        st_shared_v4(rowb + (((ch + 1) ^ (row & 7)) << 4), pk[4], pk[5], pk[6], pk[7]);
        if (args.c_debug != nullptr && m0 + row < args.M) {
          const int ncol = n_split0 + (t * G + (int)p) * kNB + c0;
          uint4* dst = reinterpret_cast<uint4*>(args.c_debug + (size_t)(m0 + row) * args.N + ncol);
          dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        }
      }
      tc_fence_before();
      mbar_arrive(c_empty[cb]);
      fence_proxy_async_smem();
      mbar_arrive(own_full);
    }
    // E tile: TMEM -> registers -> global (bf16 store, or fp32 reduce-add across splits)
    mbar_wait(e_full, 0);
    tc_fence_after();
    const int grow = m0 + row;
#pragma unroll 1
    for (int c0 = 0; c0 < kLB; c0 += 16) {
      float v[16];
      tmem_ld16(lane_base + C::kTMEM_E + c0, v);
      if (grow < args.M) {
        if (args.S == 1) {
          uint32_t pk[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) pk[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
          uint4* dst = reinterpret_cast<uint4*>(args.E + (size_t)grow * args.L + l0 + c0);
          dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        } else {
          float* dst = args.ws + (size_t)grow * args.L + l0 + c0;
#pragma unroll
          for (int i = 0; i < 16; i += 4) red_add_v4_f32(dst + i, v[i], v[i + 1], v[i + 2], v[i + 3]);
        }
      }
    }
    tc_fence_before();
  }

  __syncthreads();
  // no CTA may leave while a ring neighbour can still push into it or credit it
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kTMEM_COLS>(tmem_base);
  }
}

// fp32 workspace -> bf16 output (after the inter-cluster reduction)
__global__ void ff_finalize_kernel(const float* __restrict__ ws, __nv_bfloat16* __restrict__ out, size_t n) {
  size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 8;
  const size_t stride = (size_t)gridDim.x * blockDim.x * 8;
  for (; i < n; i += stride) {
    float4 a = *reinterpret_cast<const float4*>(ws + i);
    float4 b = *reinterpret_cast<const float4*>(ws + i + 4);
    uint4 o = make_uint4(pack_bf16x2(a.x, a.y), pack_bf16x2(a.z, a.w), pack_bf16x2(b.x, b.y),
                         pack_bf16x2(b.z, b.w));
    *reinterpret_cast<uint4*>(out + i) = o;
  }
}

}  // namespace ff
