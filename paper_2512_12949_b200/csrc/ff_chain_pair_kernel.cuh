// Fused GEMM-chain kernel, CTA-pair variant (tcgen05 cta_group::2).
//
// Same dataflow as ff_chain_kernel.cuh -- a ring of G members shares the
// intermediate C of an M tile, each member accumulates an E slice in TMEM,
// GEMM1 hops of n-step t are interleaved with GEMM0 k-blocks of n-step t+1,
// and C is exchanged through an L2-resident scratch -- but every ring member
// is a CTA PAIR (a 2-CTA cluster) issuing M=256 MMAs:
//   * CTA q of the pair owns rows [q*128, q*128+128) of the 256-row M tile;
//   * weight operands are split by columns across the pair (CTA q loads half
//     of every B / B0|B1 / D tile), so each weight byte reaches one SM;
//   * the leader (cluster rank 0) issues the MMAs; both producers' TMA loads
//     signal the leader's full barrier; commits multicast to both CTAs.
// TMA shape rule (measured, profiles/r01/tma_stream.log): the TMA unit costs
// ~0.3-0.5 us per instruction regardless of size, so every operand tile is a
// single 32 KB 3D/4D box: k-blocks are 128 deep (stage = 2 x 32 KB), the gated
// branches are fetched by one 4D box from a packed [2][K][N] gate|up weight,
// and the E tile leaves through TMA stores (S == 1) or TMA fp32 reduce-adds
// (S > 1, inter-cluster reduce) staged in shared memory.
// TMEM per CTA: C accumulator (256 columns; gated: two 128-column branch
// accumulators) + E slice (kLB columns).
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer (leader) + TMEM
// alloc, w2/w3 idle, w4..w7 epilogue.
#pragma once
#include "ff_chain_kernel.cuh"

namespace ff {

struct PairMaps {
  CUtensorMap a;    // A [M][K]: 3D {64, M, K/64}, box {64, 128, 2}
  CUtensorMap b;    // std: B [K][N] 3D {64, K, N/64} box {64, 128, 2}; gated packed: [2][K][N] 4D box {64,128,1,2}
  CUtensorMap b1;   // gated, unpacked: B1 (3D, box {64, 128, 1}); b is then B0 with the same box
  CUtensorMap d;    // D [N][L]: 3D {64, N, L/64}, box {64, 128, 2}
  CUtensorMap c;    // C exchange scratch, box {64, 128, 2}: per-(ring, member, slot) regions of 256 rows x kN0
                    // 3D {64, regions*256, kN0/64}; kRagged: the whole intermediate [Mpad][N], 3D {64, Mpad, N/64}
  CUtensorMap e;    // E [M][L] bf16: 2D box {64, 128}
  CUtensorMap w;    // fp32 workspace [M][L]: 2D box {32, 128}
  // single-instruction E tiles for a ring's final unit (stage area as staging):
  CUtensorMap e3;   // E bf16 3D {64, M, L/64}, box {64, 128, kLB/64}
  CUtensorMap w3;   // fp32 workspace 3D {32, M, L/32}, box {32, 128, kLB/32}
  CUtensorMap er;   // E bf16 3D, box {64, 128/S, kLB/64}: one row slice of a tile
  CUtensorMap slab; // split-N exchange regions 3D {32, 16, tiles*S*64} fp32, box {32, 128/S/8, 64} (no swizzle)
};

template <bool kGated, int kLB, int kStages>
struct PairCfg {
  static constexpr int BM = 128;                  // rows per CTA (256 per pair)
  static constexpr int BK = 128;                  // k depth of one stage
  static constexpr int kN0 = kGated ? 128 : 256;  // C columns per pair per n-step
  static constexpr int kCW = kN0;
  static constexpr int kSLOT = 32768;             // one operand tile (A or B / C or D) per stage
  static constexpr int kSTAGE = 2 * kSLOT;
  static constexpr int kCHUNK_BYTES = BM * kCW * 2;  // own C chunk (bf16, K-major SW128 64-col tiles)
  // The own slot (32 KB) stages the drained C chunk for its TMA store (in
  // 128-column rounds) and E tiles.  When the whole chunk fits (gated, 128
  // columns) hop 0 also reads it from there as the MMA A operand; otherwise
  // hop 0 loads the own chunk back from L2 like every other hop, which keeps a
  // third 64 KB pipeline stage for the standard FFN.
  static constexpr int kOWN_BYTES = 32768;
  static constexpr bool kOwnFull = kCHUNK_BYTES <= kOWN_BYTES;
  static constexpr int kOFF_OWN = kStages * kSTAGE;
  static constexpr int kOFF_BAR = kOFF_OWN + kOWN_BYTES;
  static constexpr int kNUM_BARS = 2 * kStages + 8;
  static constexpr int kSMEM = kOFF_BAR + kNUM_BARS * 8 + 16 + 1024;
  static constexpr int kTMEM_E = 256;
  static_assert(256 + kLB <= 512, "TMEM budget");
  static_assert(kLB == 256 || kLB == 128, "E slice: 128 or 256 columns");
};

// kQuad: clusters of 4 = two CTA pairs at the same ring position of two rings
// whose units differ only in the m tile (X = even ring, Y = odd ring).  Their
// weight tiles (B / gate|up for GEMM0, D for the hops) are identical, so each
// is TMA-multicast to both pairs by one of them (alternating per stage): three
// TMA instructions per two stages per CTA instead of four (the TMA unit is
// per-instruction bound: profiles/r01/mcast_relaxed.log).  Stages are freed
// by both leaders' commits (empty-barrier count 2, commit mask 0xF).
#undef FF_PROF_ROW
#define FF_PROF_ROW vcta
// kRagged: N need not fill whole n-steps of every split (see has_chunk); a separate
// instantiation so the common case keeps its exact code.
template <bool kGated, int kLB, int kStages, bool kPackedB, bool kQuad, bool kRagged>
__global__ void __launch_bounds__(256, 1)
    ff_chain_pair_kernel(const __grid_constant__ PairMaps maps, const ChainArgs args) {
  using C = PairCfg<kGated, kLB, kStages>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_base = smem_u32(smem_raw);
  const uint32_t base = (raw_base + 1023u) & ~1023u;
  uint8_t* const smem_gen = smem_raw + (base - raw_base);

  // the previous launch's epoch, loaded first so its latency hides behind the setup
  const uint32_t epoch0 = threadIdx.x == 0 ? epoch_begin(args) : 0u;
  const int warp = threadIdx.x / 32;
  const int G = args.G;                  // ring members (pairs)
  const uint32_t crank = cluster_rank();
  const uint32_t q = crank & 1u;         // half of the pair (0 = leader)
  const uint32_t pq = kQuad ? crank >> 1 : 0u;  // pair within the quad (0 = X, 1 = Y)
  const uint32_t lrank = 2u * pq;        // this pair's leader rank in the cluster
  const bool leader = (q == 0);
  const int vcta = (int)blockIdx.x;
  if (threadIdx.x == 0) FF_STAMP(16);
  const int p = kQuad ? (vcta / 4) % G : (vcta / 2) % G;  // ring position
  const int ring = kQuad ? 2 * ((vcta / 4) / G) + (int)pq : (vcta / 2) / G;
  const uint16_t mcast = (uint16_t)((1u << crank) | (1u << (crank ^ 2u)));  // this CTA and its twin
  const int kblocks = args.K / C::BK;
  // GEMM0 k order rotated by ring position: the 2*G*S CTAs of an m tile would
  // otherwise request the same A box at the same moment (one L2 slice set)
  const int krot = args.krot ? (p * kblocks / G) : 0;
  const int steps = args.steps;
  const int my_units = ring < args.n_units ? (args.n_units - ring + args.n_rings - 1) / args.n_rings : 0;
  // Tail split (multi-unit launches, S == 1, one l cluster): the units of the last, partial wave
  // would leave rings idle, so each is cut in N into tail_S units of steps / tail_S n-steps
  // (units n_full.. in that order, at most one per ring, always the ring's last) that combine
  // through the split-N reduce-scatter.  A ring's global step T then maps to (unit, step)
  // with a shorter last unit.
  const bool has_tail = args.tail_S > 1 && my_units > 0 && ring + (my_units - 1) * args.n_rings >= args.n_full;
  const int steps_t = args.tail_S > 1 ? steps / args.tail_S : steps;
  const int full_steps = (my_units - (has_tail ? 1 : 0)) * steps;
  const int total_steps = full_steps + (has_tail ? steps_t : 0);
  auto ui_of = [&](int T) { return T < full_steps ? T / steps : my_units - 1; };
  auto t_of = [&](int T) { return T < full_steps ? T % steps : T - full_steps; };
  auto steps_of = [&](int ui) { return (has_tail && ui == my_units - 1) ? steps_t : steps; };

  struct Unit {
    int m0, l0, n0, id, split;
  };
  auto unit_of = [&](int i) {
    const int u = ring + i * args.n_rings;
    if (args.tail_S > 1 && u >= args.n_full) {  // tail unit: split (u - n_full) % tail_S of m tile n_full + ..
      const int j = u - args.n_full;
      return Unit{(args.n_full + j / args.tail_S) * 2 * C::BM, p * kLB, (j % args.tail_S) * steps_t * G * C::kN0, u,
                  j % args.tail_S};
    }
    const int mt = u % args.m_tiles;
    const int rest = u / args.m_tiles;
    const int lc = rest % args.l_clusters;
    const int split = rest / args.l_clusters;
    return Unit{mt * 2 * C::BM, (lc * G + p) * kLB, split * (kRagged ? args.split_chunks : steps * G) * C::kN0, u,
                split};
  };
  // ragged n-steps: split s owns chunks [s * split_chunks, min(N / kN0, (s + 1) * split_chunks)),
  // chunk t * G + origin of a split is GEMM0'd by member `origin` in n-step t.  A member
  // without a chunk keeps every barrier handshake (empty GEMM0 commits, drain-less
  // arrivals) and skips the work.  T is the member's global step index.
  // physical n-step (column position) of global step T: a ring's odd units walk their
  // n-steps backwards (serpentine), so the first weights they read are the ones the
  // previous unit read last.  Flags, scratch slots and the schedule keep the logical step.
  auto nstep = [&](int T) {
    const int t = t_of(T), ui = ui_of(T);
    return (!kRagged && args.serp && (ui & 1)) ? steps_of(ui) - 1 - t : t;
  };
  auto has_chunk = [&](int T, int origin) {
    if (!kRagged) return true;
    const int split = unit_of(ui_of(T)).split;
    const int lim = min(args.split_chunks, args.total_chunks - split * args.split_chunks);
    return t_of(T) * G + origin < lim;
  };

  const uint32_t bar0 = base + C::kOFF_BAR;
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (kStages + s); };
  const uint32_t bx = bar0 + 8u * (2 * kStages);
  const uint32_t c_full = bx, c_empty = bx + 8, own_full = bx + 16, own_free = bx + 24;
  const uint32_t e_full = bx + 32, e_empty = bx + 40, e_load = bx + 48;
  const uint32_t c_full1 = bx + 56;  // C(1) in E's columns (swap_e below): its own barrier, since
                                     // c_full could complete twice before the epilogue looks
  const uint32_t tmem_slot = bar0 + 8u * C::kNUM_BARS;
  const uint32_t own_slot = base + C::kOFF_OWN;
  const uint16_t kPairMask = (uint16_t)(0x3u << lrank);
  const uint16_t kStageMask = kQuad ? (uint16_t)0xF : kPairMask;  // stage consumers: both leaders

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full_bar(s), 1);  // the leader's arrive.expect_tx covers both CTAs' bytes
      mbar_init(empty_bar(s), kQuad ? 2 : 1);
    }
    mbar_init(c_full, 1);
    mbar_init(c_empty, 256);  // both CTAs' epilogues arrive on the leader's barrier
    mbar_init(own_full, 256);
    // own slot free again after: the C store read it (+ the MMA's hop 0 when it is the A operand)
    mbar_init(own_free, (C::kOwnFull && G > 1) ? 2 : 1);
    mbar_init(e_full, 1);
    mbar_init(e_empty, 256);
    mbar_init(e_load, 1);
    mbar_init(c_full1, 1);
    fence_mbar_init();
  }
  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&maps.a);
    tma_prefetch_desc(&maps.b);
    if (kGated && !kPackedB) tma_prefetch_desc(&maps.b1);
    tma_prefetch_desc(&maps.d);
    if (G > 1 || !C::kOwnFull) tma_prefetch_desc(&maps.c);
  }
  if (warp == 1) tmem_alloc_pair<512>(tmem_slot);
  __shared__ uint32_t s_epoch;
  if (threadIdx.x == 0) s_epoch = epoch0;
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t*>(smem_gen + (tmem_slot - base));
  const uint32_t epoch = s_epoch;
  if (threadIdx.x == 96) epoch_publish(args, epoch);  // warp 3 lane 0 (idle warp)
  if (threadIdx.x == 0) FF_STAMP(17);

  // GEMM0 of step T+1 is spread over the first G - defer hops of step T; the
  // last `defer` hops run after it, while the epilogue drains C(T+1), so the
  // tensor core does not idle through the drain.  The host sets defer = G-1
  // (one slice: GEMM0(T+1) before every hop of step T); the ring's last GEMM0
  // always runs that way (defer_last): nothing follows it, so all hops are
  // needed to cover its drain, publish and the ring members' skew.
  auto g0_slices = [&](int Tn) { return (Tn == total_steps - 1 && args.defer_last) ? 1 : G - args.defer; };
  auto slot_lo = [&](int Tn, int h) {
    const int g0s = g0_slices(Tn);
    return h < g0s ? h * kblocks / g0s : kblocks;
  };
  // One unit of two n-steps (the M=512 chains): GEMM0(1) runs before any hop of
  // step 0, while the E accumulator is still unused, so it accumulates in E's TMEM
  // columns instead of waiting for the epilogue to drain C(0); E then lives in the
  // drained C columns.  Removes the C-drain bubble from the tensor pipe.
  const bool swap_e = args.defer_last && total_steps == 2 && steps == 2;
  const uint32_t e_col = swap_e ? 0u : (uint32_t)C::kTMEM_E;
  auto c_col = [&](int T) { return (swap_e && T == 1) ? (uint32_t)C::kTMEM_E : 0u; };
  auto flag_addr = [&](const Unit& u, int t, int origin, int half) {
    return args.flags + (((size_t)u.id * steps + t) * G + origin) * 2 + half;
  };
  // C exchange scratch.  Chunk (global step T, origin) of this ring lives in region
  // (ring, origin, T % c_slots); this CTA's half holds rows q*128.. of it.  A slot is
  // rewritten c_slots steps later, once every member has read it: a member that has
  // published its chunk of step T' has finished reading the chunks of step T'-2 (its
  // GEMM0(T') MMAs, committed before the flag, were issued after its hops of T'-2, and
  // tcgen05 MMAs complete in order), so before writing step T the origin waits for
  // every member's flag of step T - c_slots + 2 (c_slots == 3; fewer slots only when a
  // ring has no more steps than slots).  Ragged launches address the whole intermediate.
  auto c_row = [&](const Unit& u, int T, int origin) {
    if (kRagged) return u.m0 + (int)q * C::BM;
    return ((ring * G + origin) * args.c_slots + T % args.c_slots) * (2 * C::BM) + (int)q * C::BM;
  };
  auto c_blk = [&](const Unit& u, int t, int origin) {  // first 64-column block of the chunk
    return kRagged ? (u.n0 + (t * G + origin) * C::kN0) / 64 : 0;
  };
  const uint32_t L_c_empty = mapa(c_empty, lrank), L_own_full = mapa(own_full, lrank),
                 L_e_empty = mapa(e_empty, lrank);
  // Split-N reduce-scatter tail (one unit per ring, S > 1): all eight warps
  // drain the ring's last E partial after the role loops (see below).
  const bool scatter_all = (args.S > 1 && args.finish_tma && total_steps > 0) || has_tail;
  // C scratch discard at exit (one set of regions per ring, addressed per member and slot)
  const bool discard_c = (args.discard & 2) && !kRagged && (G > 1 || !C::kOwnFull) && my_units > 0;
  auto done_flag = [&](int member) { return args.flags + (3u << 16) + ring * G + member; };
  // A tile: two K-major [128 x 64] SW128 tiles; B tile: MN-major [128 k x 64] tiles 16 KB apart
  auto a_desc = [](uint32_t slot, int kk) { return desc_kmajor_sw128(slot + (kk >> 2) * 16384 + (kk & 3) * 32); };
  auto b_desc = [](uint32_t slot, int kk) { return desc_mnmajor_sw128(slot + kk * 2048, 16384); };
  constexpr int kChunks = kLB / 4;  // 16-byte column chunks per E row

#ifndef FF_PRODUCER_SPLIT  // 1: two producer threads (warp 0: A / C + barrier arming + flags; warp 2: weights)
#define FF_PRODUCER_SPLIT 1
#endif
  // TMA producer body.  role 0 issues the A / C boxes, arms the full barriers and polls the
  // ready flags; role 1 issues the weight boxes (B / gate|up, D) and their L2 prefetches;
  // role 2 does both.  Both threads of a split walk the same stage sequence.
  auto producer = [&](const int role) {
    const bool do_ac = role != 1, do_w = role != 0;
    {
      unsigned long long w_empty = 0, w_flag = 0;
      const unsigned long long t_start = clock64();
      int stage = 0, phase = 0;
      uint32_t seq = 0;
      const uint64_t pol_w = l2_policy(args.wpolicy);  // weight tiles (B / gate|up, D)
      const uint64_t pol_c = l2_policy(args.cpolicy);  // C exchange scratch  // stage-load sequence number (identical in both pairs of a quad)
      auto next = [&]() {
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      };
      // Only the leader arms the (leader-owned) full barrier, for the bytes of
      // both CTAs; the peer's loads just complete_tx on it.  A per-stage
      // remote arrive (release.cluster) from the peer halved the TMA feed
      // (profiles/r01/tma_variants.log: cluster-scope barrier ops 57-68 GB/s
      // per SM vs 130 GB/s with CTA-scope ones).
      auto arm = [&]() {
        if (leader) mbar_expect_tx(full_bar(stage), 2 * C::kSTAGE);
      };
      // (unit, step, physical n-step) of a global step, computed once per step: the per-hop
      // integer divisions of the mapping sat on the producer's critical path (+10 us, A/B)
      struct StepAt {
        Unit u;
        int t, ns;
      };
      auto step_at = [&](int T) { return StepAt{unit_of(ui_of(T)), t_of(T), nstep(T)}; };
      auto load_gemm0 = [&](int T, const StepAt& st, int kb0, int kb1) {
        if (kb0 >= kb1 || !has_chunk(T, p)) return;
        const Unit& u = st.u;
        // first 64-column block of this CTA's half of the chunk (gated: of each branch)
        const int nblk = (u.n0 + (st.ns * G + p) * C::kN0) / 64 + (int)q * (C::kN0 / 128);
        for (int kbl = kb0; kbl < kb1; ++kbl) {
          // physical k-block (members start at staggered k); no runtime division on the producer's
          // per-stage path (its issue latency is the pipeline's, see StepAt)
          const int kb = kbl + krot < kblocks ? kbl + krot : kbl + krot - kblocks;
          FF_TIMED(w_empty, mbar_wait(empty_bar(stage), phase ^ 1));
          const uint32_t sb = base + stage * C::kSTAGE;
          const uint32_t lb = mapa(full_bar(stage), lrank);
          if (do_ac) {
            arm();
            tma_load_3d_pair(sb, &maps.a, lb, 0, u.m0 + (int)q * C::BM, kb * (C::BK / 64));
          }
          if (!do_w) {
            next();
            continue;
          }
          const bool mine = !kQuad || ((seq++ & 1u) == pq);  // this pair issues the shared weight tile
          // L2 prefetch of the B tile `prefetch` k-blocks ahead: the weights
          // stream from HBM; the extra lead hides its latency behind 3 stages
#ifdef FF_AB_NO_PREFETCH  // A/B builds only: without the L2 prefetches of weight tiles
          const int pf = 0;
#else
          const int pf = args.prefetch;
#endif
          if (pf && kbl + pf < kblocks && (!kQuad || pq == 0)) {
            const int kbp = kbl + pf + krot < kblocks ? kbl + pf + krot : kbl + pf + krot - kblocks;
            if (!kGated || !kPackedB)
              tma_prefetch_l2_3d_h(&maps.b, 0, kbp * C::BK, nblk, pol_w);
            else
              tma_prefetch_l2_4d_h(&maps.b, 0, kbp * C::BK, nblk, 0, pol_w);
          }
          if (!mine) {
          } else if (kQuad) {
            if (!kGated) {
              tma_load_3d_pair_mcast_h(sb + C::kSLOT, &maps.b, lb, 0, kb * C::BK, nblk, mcast, pol_w);
            } else if (kPackedB) {
              tma_load_4d_pair_mcast_h(sb + C::kSLOT, &maps.b, lb, 0, kb * C::BK, nblk, 0, mcast, pol_w);
            } else {
              tma_load_3d_pair_mcast_h(sb + C::kSLOT, &maps.b, lb, 0, kb * C::BK, nblk, mcast, pol_w);
              tma_load_3d_pair_mcast_h(sb + C::kSLOT + C::kSLOT / 2, &maps.b1, lb, 0, kb * C::BK, nblk, mcast, pol_w);
            }
          } else if (!kGated) {
            tma_load_3d_pair_h(sb + C::kSLOT, &maps.b, lb, 0, kb * C::BK, nblk, pol_w);
          } else if (kPackedB) {
            tma_load_4d_pair_h(sb + C::kSLOT, &maps.b, lb, 0, kb * C::BK, nblk, 0, pol_w);
          } else {
            tma_load_3d_pair_h(sb + C::kSLOT, &maps.b, lb, 0, kb * C::BK, nblk, pol_w);
            tma_load_3d_pair_h(sb + C::kSLOT + C::kSLOT / 2, &maps.b1, lb, 0, kb * C::BK, nblk, pol_w);
          }
          next();
        }
      };
      unsigned long long ready = 0;  // ring members whose C chunk of the current step is published
      auto load_hop = [&](int T, const StepAt& st, int h) {
        const Unit& u = st.u;
        const int t = st.t;
        const int origin = p >= h ? p - h : p - h + G;
        const int ncol0 = u.n0 + (st.ns * G + origin) * C::kN0;
        const int dblk = u.l0 / 64 + (int)q * (kLB / 128);
        const bool from_l2 = h > 0 || !C::kOwnFull;  // C operand of this hop comes from the L2 scratch
        if (h == 0) ready = C::kOwnFull ? 1ull << p : 0ull;
        if (!has_chunk(T, origin)) return;  // ragged n-step: no chunk from this origin
#ifdef FF_AB_NO_FLAG_WAIT  // A/B builds only: cost of the ready-flag polls (results are not valid)
        if (false) {
#else
        if (do_ac && from_l2 && !((ready >> origin) & 1ull)) {
#endif
          // one round trip polls every member whose chunk is still missing
          uint32_t polls = 0;
          FF_TIMED(w_flag, do {
            for (int o0 = 0; o0 < G; o0 += 8) {
              uint32_t v[8];
#pragma unroll
              for (int j = 0; j < 8; ++j)  // independent loads: in flight together
                v[j] = (o0 + j < G && !((ready >> (o0 + j)) & 1ull))
                           ? ld_relaxed_gpu_u32(flag_addr(u, t, o0 + j, (int)q))
                           : epoch - 1u;
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (v[j] == epoch) ready |= 1ull << (o0 + j);
            }
            if (++polls == FF_WATCHDOG_POLLS) FF_WD_EXPIRED(((unsigned long long)origin << 32) | epoch);
          } while (!((ready >> origin) & 1ull)));
          fence_acq_rel_gpu();
          fence_proxy_async_global();
        }
#ifdef FF_AB_NO_DPREFETCH  // A/B builds only: without the L2 prefetches of hop weight tiles
        if (false) {
#else
        if (do_w && args.prefetch && h + args.prefetch < G && (!kQuad || pq == 0)) {  // D rows of a later hop
#endif
          const int o_pf = p - h - args.prefetch + (p - h - args.prefetch < -G ? 2 * G : p - h - args.prefetch < 0 ? G : 0);
          const int ncol_pf = u.n0 + (st.ns * G + o_pf) * C::kN0;
          for (int kb2 = 0; kb2 < C::kCW / C::BK; ++kb2)
            tma_prefetch_l2_3d_h(&maps.d, 0, ncol_pf + kb2 * C::BK, dblk, pol_w);
        }
        const int crow = c_row(u, T, origin), cblk = c_blk(u, t, origin);  // once per hop
        for (int kb2 = 0; kb2 < C::kCW / C::BK; ++kb2) {
          FF_TIMED(w_empty, mbar_wait(empty_bar(stage), phase ^ 1));
          const uint32_t sb = base + stage * C::kSTAGE;
          const uint32_t lb = mapa(full_bar(stage), lrank);
          if (do_ac) {
            if (leader) mbar_expect_tx(full_bar(stage), 2 * (from_l2 ? C::kSTAGE : C::kSLOT));
            if (from_l2) tma_load_3d_pair_h(sb, &maps.c, lb, 0, crow, cblk + kb2 * (C::BK / 64), pol_c);
          }
          if (do_w) {
            if (!kQuad)
              tma_load_3d_pair_h(sb + C::kSLOT, &maps.d, lb, 0, ncol0 + kb2 * C::BK, dblk, pol_w);
            else if ((seq++ & 1u) == pq)
              tma_load_3d_pair_mcast_h(sb + C::kSLOT, &maps.d, lb, 0, ncol0 + kb2 * C::BK, dblk, mcast, pol_w);
          }
          next();
        }
      };
      StepAt cur = step_at(0);
      if (total_steps > 0) load_gemm0(0, cur, 0, kblocks);
      for (int T = 0; T < total_steps; ++T) {
        const StepAt nxt = T + 1 < total_steps ? step_at(T + 1) : cur;
        const int g0s = g0_slices(T + 1);
        for (int h = 0; h < G; ++h) {
          // (the slice bounds only for the hops that carry GEMM0(T+1) k-blocks: slot_lo divides)
          if (T + 1 < total_steps && h < g0s) load_gemm0(T + 1, nxt, slot_lo(T + 1, h), slot_lo(T + 1, h + 1));
          load_hop(T, cur, h);
        }
        cur = nxt;
      }
      if (args.prof && do_ac) {
        unsigned long long* pr = args.prof + vcta * FF_PROF_STRIDE;
        pr[0] = clock64() - t_start;
        pr[1] = w_empty;
        pr[2] = w_flag;
      }
    }
  };
  // Split only rings of several units (measured, interleaved timelines: OPT M=32768 -3.5 %,
  // M=4096 -1 %; one-unit rings: GPT-6.7B +0.6 %, LLaMA-1B +3-6 %)
  const bool split_producer = FF_PRODUCER_SPLIT && my_units > 1;
  if (warp == 0) {
    // ===================== TMA producer (both CTAs) =====================
    if (elect_one()) producer(split_producer ? 0 : 2);
    // The other 31 lanes wait here (not in a spin loop of their own) until the producer lane
    // is done: two divergent spin-wait paths in one warp can starve the role lane (found on
    // hardware with the diagnostic watchdog: the tail issuer's flag polls never ran while its
    // 31 lanes spun on e_load).
    __syncwarp();
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA only) =====================
    if (leader && elect_one()) {
      unsigned long long w_full0 = 0, w_full1 = 0, w_cempty = 0, w_own = 0, w_eempty = 0;
      const unsigned long long t_start = clock64();
      int stage = 0, phase = 0;
      auto next = [&]() {
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      };
      const uint32_t idesc0 = idesc_as(idesc_bf16(256, C::kN0, 0, 1), args.f16);
      const uint32_t idesc1 = idesc_as(idesc_bf16(256, kLB, 0, 1), args.f16);
      auto gemm0 = [&](int T, int kb0, int kb1) {
        if (kb0 >= kb1) return;
        if (kb0 == 0 && !(swap_e && T == 1)) {
          FF_TIMED(w_cempty, mbar_wait_cluster(c_empty, (T & 1) ^ 1));
          tc_fence_after();
        }
        const uint32_t cacc = tmem_base + c_col(T);
        const bool has = has_chunk(T, p);
        for (int kb = kb0; kb < (has ? kb1 : kb0); ++kb) {
          FF_TIMED(w_full0, mbar_wait(full_bar(stage), phase));
          tc_fence_after();
          const uint32_t sb = base + stage * C::kSTAGE;
#pragma unroll
          for (int kk = 0; kk < C::BK / 16; ++kk) {
            const uint64_t ad = a_desc(sb, kk);
            const uint32_t acc = (kb | kk) ? 1u : 0u;
            if (kGated) {
              umma_bf16_pair(cacc, ad, b_desc(sb + C::kSLOT, kk), idesc0, acc);
              umma_bf16_pair(cacc + C::kN0, ad, b_desc(sb + C::kSLOT + C::kSLOT / 2, kk), idesc0, acc);
            } else {
              umma_bf16_pair(cacc, ad, b_desc(sb + C::kSLOT, kk), idesc0, acc);
            }
          }
          umma_commit_pair(empty_bar(stage), kStageMask);
          next();
        }
        if (kb1 == kblocks) umma_commit_pair((swap_e && T == 1) ? c_full1 : c_full, kPairMask);
      };
      bool e_started = false;
      auto hop = [&](int T, int t, int ui, int h) {
        if (t == 0 && h == 0) {
          if (ui > 0) {
            FF_TIMED(w_eempty, mbar_wait_cluster(e_empty, (ui - 1) & 1));
            tc_fence_after();
          }
          e_started = false;
        }
        if (swap_e && T == 0 && h == 0) {  // E goes to C(0)'s columns: drained?
          FF_TIMED(w_cempty, mbar_wait_cluster(c_empty, 0));
        }
        if (C::kOwnFull && h == 0) FF_TIMED(w_own, mbar_wait_cluster(own_full, T & 1));
        tc_fence_after();
        const bool has = has_chunk(T, (p - h + G) % G);
        for (int kb2 = 0; kb2 < (has ? C::kCW / C::BK : 0); ++kb2) {
          FF_TIMED(w_full1, mbar_wait(full_bar(stage), phase));
          tc_fence_after();
          const uint32_t sb = base + stage * C::kSTAGE;
          const uint32_t aslot = (C::kOwnFull && h == 0) ? own_slot + kb2 * 2 * 16384 : sb;
#pragma unroll
          for (int kk = 0; kk < C::BK / 16; ++kk) {
            umma_bf16_pair(tmem_base + e_col, a_desc(aslot, kk), b_desc(sb + C::kSLOT, kk), idesc1,
                             e_started ? 1u : 0u);
            e_started = true;
          }
          umma_commit_pair(empty_bar(stage), kStageMask);
          next();
        }
        if (C::kOwnFull && h == 0) umma_commit_pair(own_free, kPairMask);
        if (t == steps_of(ui) - 1 && h == G - 1) umma_commit_pair(e_full, kPairMask);
      };
      if (total_steps > 0) gemm0(0, 0, kblocks);
      for (int T = 0; T < total_steps; ++T) {
        const int t = t_of(T), ui = ui_of(T);  // once per step (see the producer)
        const int g0s = g0_slices(T + 1);
        for (int h = 0; h < G; ++h) {
          if (T + 1 < total_steps && h < g0s) gemm0(T + 1, slot_lo(T + 1, h), slot_lo(T + 1, h + 1));
          hop(T, t, ui, h);
        }
      }
      // every C load of this pair has landed (its full barriers completed): the ring's
      // scratch is no longer read by this member
      if (discard_c) st_release_gpu_u32(done_flag(p), epoch);
      if (args.prof) {
        unsigned long long* pr = args.prof + vcta * FF_PROF_STRIDE;
        pr[3] = clock64() - t_start;
        pr[4] = w_full0;
        pr[5] = w_full1;
        pr[6] = w_cempty;
        pr[7] = w_own;
        pr[8] = w_eempty;
      }
    }
    __syncwarp();  // see warp 0
  } else if (warp == 2 && split_producer) {
    // ===================== TMA producer, weight boxes (both CTAs) =====================
    if (elect_one()) producer(1);
    __syncwarp();  // see warp 0
  } else if (warp >= 4) {
    // ===================== epilogue (both CTAs) =====================
    const int wq = warp & 3;
    const int row = wq * 32 + (int)lane_id();
    const uint32_t lane_base = tmem_base + ((uint32_t)(wq * 32) << 16);
    const bool issuer = (warp == 4 && lane_id() == 0);
    unsigned long long w_cfull = 0, w_ofree = 0, t_drain = 0, t_store = 0, t_e = 0;
    const unsigned long long t_start = clock64();
    // row r of a 128-byte-row SW128 tile: 16-byte chunk c lives at chunk c ^ (r & 7)
    auto swz = [&](uint32_t tile, int ch) { return tile + row * 128 + ((ch ^ (row & 7)) << 4); };
    const uint64_t pol_c = l2_policy(args.cpolicy);  // C exchange scratch
    const uint64_t pol_e = l2_policy(args.epolicy);  // E tiles
    // before chunk T overwrites slot T % c_slots: every ring member's flag of step
    // T - c_slots + 2, i.e. all of them have read step T - c_slots (see c_row)
    auto wait_slot_free = [&](int T) {
      if (kRagged || T < args.c_slots) return;
      const int Tp = T - args.c_slots + 2;
      const Unit up = unit_of(ui_of(Tp));
      const int tp = t_of(Tp);
      uint32_t polls = 0;
      unsigned long long seen = 0ull;
      const unsigned long long all = G >= 64 ? ~0ull : (1ull << G) - 1ull;
      while (seen != all) {
        for (int o0 = 0; o0 < G; o0 += 8) {
          uint32_t v[8];
#pragma unroll
          for (int j = 0; j < 8; ++j)  // independent loads: in flight together
            v[j] = (o0 + j < G && !((seen >> (o0 + j)) & 1ull)) ? ld_relaxed_gpu_u32(flag_addr(up, tp, o0 + j, (int)q))
                                                                 : epoch;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (o0 + j < G && v[j] == epoch) seen |= 1ull << (o0 + j);
        }
        if (++polls == FF_WATCHDOG_POLLS) FF_WD_EXPIRED((seen << 32) | epoch);
      }
      fence_acq_rel_gpu();
      fence_proxy_async_global();
    };
    // C chunk of global step T: TMEM -> activation / gate -> bf16 SW128 own slot -> L2 scratch + flag
    auto drain_c = [&](int T) {
      const Unit u = unit_of(ui_of(T));
      const int t = t_of(T);
      FF_TIMED(w_cfull, (swap_e && T == 1) ? mbar_wait_cluster(c_full1, 0) : mbar_wait_cluster(c_full, T & 1));
      tc_fence_after();
      if (issuer && T < 2) FF_STAMP(18 + 3 * T);
      FF_TIMED(w_ofree, mbar_wait_cluster(own_free, (T & 1) ^ 1));
      const unsigned long long t_d0 = args.prof ? clock64() : 0ull;
      const bool publish = G > 1 || !C::kOwnFull;  // the chunk goes to the L2 scratch
      constexpr int kRoundCols = C::kOWN_BYTES / (C::BM * 2);  // 128 columns per own-slot round
      const bool has = has_chunk(T, p);
      // With the E/C column swap nothing waits for C(1)'s drain (no GEMM0(2); E already lives in
      // C(0)'s columns), and arriving would let c_empty complete twice before the MMA thread's
      // wait for C(0)'s drain looks -- a parity alias that hung a ragged member without chunks,
      // whose two drains are both immediate (found on hardware by the diagnostic watchdog)
      const bool release_c = !(swap_e && T == 1);
      if (!has) {  // ragged last n-step without a chunk here: the handshakes only
        tc_fence_before();
        if (release_c) mbar_arrive_remote(L_c_empty);
        if (C::kOwnFull) mbar_arrive_remote(L_own_full);
      }
#pragma unroll 1
      for (int r0 = 0; r0 < (has ? C::kCW : 0); r0 += kRoundCols) {
        if (r0 > 0) {  // the previous round's TMA store must have read the own slot
          if (issuer) bulk_wait_read0();
          named_bar_sync(1, 128);
        }
#pragma unroll 1
        for (int c0 = r0; c0 < r0 + kRoundCols; c0 += 32) {
          float v[32];
          if (kGated) {
            float w[32];
            tmem_ld32x2(lane_base + c_col(T) + c0, lane_base + c_col(T) + C::kN0 + c0, v, w);
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = silu_fast(v[i]) * w[i];
          } else {
            tmem_ld32(lane_base + c_col(T) + c0, v);
            apply_act_frag(args.act, v);
          }
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) pk[i] = pack2(args.f16, v[2 * i], v[2 * i + 1]);
          const uint32_t tile = own_slot + ((c0 - r0) / 64) * 16384;
          const int ch = (c0 % 64) / 8;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            st_shared_v4(swz(tile, ch + j), pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
          const int grow = u.m0 + (int)q * C::BM + row;
          if (args.c_debug != nullptr && grow < args.M) {
            const int ncol = u.n0 + (nstep(T) * G + p) * C::kN0 + c0;
            uint4* dst = reinterpret_cast<uint4*>(args.c_debug + (size_t)grow * args.N + ncol);
#pragma unroll
            for (int j = 0; j < 4; ++j) dst[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
          }
        }
        if (r0 + kRoundCols >= C::kCW && release_c) {  // C accumulator fully read: GEMM0 of the next step may start
          tc_fence_before();
          mbar_arrive_remote(L_c_empty);
        }
        fence_proxy_async_smem();
        if (C::kOwnFull) mbar_arrive_remote(L_own_full);
        if (publish) {
          named_bar_sync(1, 128);
          if (issuer) {
            if (r0 == 0) wait_slot_free(T);
            tma_store_3d_h(&maps.c, own_slot, 0, c_row(u, T, p), c_blk(u, t, p) + r0 / 64, pol_c);
            bulk_commit();
          }
        }
      }
      if (args.prof) t_drain += clock64() - t_d0;
      if (issuer && T < 2) FF_STAMP(19 + 3 * T);
      const unsigned long long t_s0 = args.prof ? clock64() : 0ull;
      if (publish && issuer) {
        if (has) {
          bulk_wait0();
          fence_proxy_async_global();
          st_release_gpu_u32(flag_addr(u, t, p, (int)q), epoch);
        }
        mbar_arrive(own_free);
      }
      __syncwarp();  // lanes 1-31 must not spin on the next barrier while the issuer publishes
      if (args.prof) t_store += clock64() - t_s0;
      if (issuer && T < 2) FF_STAMP(20 + 3 * T);
    };
    int next_c = 0;  // first C chunk not yet drained
    for (int T = 0; T < total_steps; ++T) {
      if (next_c <= T) {
        drain_c(T);
        next_c = T + 1;
      }
      const Unit u = unit_of(ui_of(T));
      const int t = t_of(T);
      if (t == steps_of(ui_of(T)) - 1 && !(scatter_all && T == total_steps - 1)) {
        // The next unit's first C chunk is ready mid-way through this unit's last hops:
        // drain and publish it before this unit's E, so the tensor core can start the
        // next GEMM0 while E drains (not with kOwnFull: the own slot then still holds
        // that chunk as hop 0's operand when E needs it for staging).
        if (!C::kOwnFull && T + 1 < total_steps) {
          drain_c(T + 1);
          next_c = T + 2;
        }
        // E slice: TMEM -> registers -> SW128 smem tiles in the own slot -> TMA
        // store (bf16) or TMA reduce-add into the fp32 workspace (N splits).
        const unsigned long long t_e0 = args.prof ? clock64() : 0ull;
        mbar_wait_cluster(e_full, ui_of(T) & 1);
        tc_fence_after();
        if (issuer) FF_STAMP(30);
        mbar_wait_cluster(own_free, (next_c - 1) & 1);  // own slot no longer read by hop 0 / the last C store
        const int erow = u.m0 + (int)q * C::BM;
        // Staging: the own slot (2 x 16 KB tiles), or -- for the ring's final
        // unit, when every pipeline stage has been consumed (e_full) and no
        // further load is coming -- the whole stage area, so the E tile leaves
        // in one round of TMA stores / reduce-adds.
        const bool final_unit = ui_of(T) == my_units - 1;
        const uint32_t stg = final_unit ? base : own_slot;
        const int kTiles = final_unit ? (kStages * C::kSTAGE) / 16384 : C::kOWN_BYTES / 16384;
        const bool bf16_out = (args.S == 1);
        const int cols_per_tile = bf16_out ? 64 : 32;
        uint32_t* const tile_counter = args.tile_cnt + (erow / C::BM) * (args.L / kLB) + u.l0 / kLB;
        if (final_unit) {
          // whole E tile staged at once: [kLB/cols_per_tile][128 rows][128 B] SW128 tiles, one TMA instruction
#pragma unroll 1
          for (int c0 = 0; c0 < kLB; c0 += 32) {
            float v[32];
            tmem_ld32(lane_base + e_col + c0, v);
            const uint32_t tile = base + (c0 / cols_per_tile) * 16384;
            if (bf16_out) {
              uint32_t pk[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) pk[i] = pack2(args.f16, v[2 * i], v[2 * i + 1]);
              const int ch = (c0 % 64) / 8;
#pragma unroll
              for (int j = 0; j < 4; ++j)
                st_shared_v4(swz(tile, ch + j), pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
            } else {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                st_shared_v4(swz(tile, j), __float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]),
                             __float_as_uint(v[4 * j + 2]), __float_as_uint(v[4 * j + 3]));
            }
          }
          tc_fence_before();
          mbar_arrive_remote(L_e_empty);
          fence_proxy_async_smem();
          named_bar_sync(1, 128);
          if (issuer) {
            if (bf16_out)
              tma_store_3d_h(&maps.e3, base, 0, erow, u.l0 / 64, l2_policy(args.epolicy));
            else
              tma_reduce_add_3d(&maps.w3, base, 0, erow, u.l0 / 32);
            bulk_commit();
            FF_STAMP(24);
          }
          if (!bf16_out) {
            split_finish<kLB>(args, tile_counter, tmem_slot + 8, issuer, true, erow, row, u.l0, 1, false);
            if (issuer) FF_STAMP(26);
          }
        } else {
#pragma unroll 1
        for (int g0 = 0; g0 < kLB; g0 += cols_per_tile * kTiles) {
          const int g1 = (g0 + cols_per_tile * kTiles < kLB) ? g0 + cols_per_tile * kTiles : kLB;
#pragma unroll 1
          for (int c0 = g0; c0 < g1; c0 += 32) {
            float v[32];
            tmem_ld32(lane_base + e_col + c0, v);
            const uint32_t tile = stg + ((c0 - g0) / cols_per_tile) * 16384;
            if (bf16_out) {
              uint32_t pk[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) pk[i] = pack2(args.f16, v[2 * i], v[2 * i + 1]);
              const int ch = (c0 % 64) / 8;
#pragma unroll
              for (int j = 0; j < 4; ++j)
                st_shared_v4(swz(tile, ch + j), pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
            } else {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                st_shared_v4(swz(tile, j), __float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]),
                             __float_as_uint(v[4 * j + 2]), __float_as_uint(v[4 * j + 3]));
            }
          }
          if (g1 == kLB) {  // every E column read: the next unit's hops may start (before the last store)
            tc_fence_before();
            mbar_arrive_remote(L_e_empty);
          }
          fence_proxy_async_smem();
          named_bar_sync(1, 128);
          if (issuer) {
            for (int c0 = g0; c0 < g1; c0 += cols_per_tile) {
              const uint32_t tile = stg + ((c0 - g0) / cols_per_tile) * 16384;
              if (bf16_out)
                tma_store_2d_h(&maps.e, tile, u.l0 + c0, erow, pol_e);
              else
                tma_reduce_add_2d(&maps.w, tile, u.l0 + c0, erow);
            }
            bulk_commit();
            bulk_wait_read0_group();
          }
          named_bar_sync(1, 128);
        }
        if (issuer) FF_STAMP(24);
        if (!bf16_out) {
          split_finish<kLB>(args, tile_counter, tmem_slot + 8, issuer, true, erow, row, u.l0, 1, false);
          if (issuer) FF_STAMP(26);
        }
        }
        if (args.prof) t_e += clock64() - t_e0;
      }
    }
    if (issuer) bulk_wait_read0();  // smem sources of the E stores read before exit (writes drain at grid end)
    if (args.prof && issuer) {
      unsigned long long* pr = args.prof + vcta * FF_PROF_STRIDE;
      pr[9] = clock64() - t_start;
      pr[10] = w_cfull;
      pr[11] = w_ofree;
      pr[12] = t_drain;
      pr[13] = t_store;
      pr[14] = t_e;
    }
  }

  if (scatter_all) {
    // ===================== split-N reduce-scatter (all 8 warps) =====================
    // The ring's final E partial (fp32, this CTA's 128 rows x kLB columns) never
    // touches shared memory: row slice j (R = 128/S rows) belongs to split j.
    // Threads holding rows of another split's slice write them straight from
    // TMEM registers into this split's exchange region, laid out
    // [16-byte column chunk][row] so that a warp's 32 rows form one contiguous
    // 512-byte store (and later load); then the CTA flags the region.  Threads
    // holding rows of the own slice wait for the partners' flags, sum the S
    // partials in split order (deterministic, own partial from TMEM), cast to
    // bf16 and stage the rows for one TMA store of E.  Warp w reads TMEM lane
    // quarter w%4; warps 0-3 take the upper half of the columns.
    const Unit u = unit_of(my_units - 1);
    const int S = has_tail ? args.tail_S : args.S, R = C::BM / S, sp = u.split;
    const int erow = u.m0 + (int)q * C::BM;
    const int wq = warp & 3;
    const int row = wq * 32 + (int)lane_id();
    const int tid = (int)threadIdx.x;
    const bool issuer = (tid == 128);
    const uint32_t lane_base = tmem_base + ((uint32_t)(wq * 32) << 16);
    const int c_lo = warp < 4 ? kLB / 2 : 0;
    const int slice = row / R;
    // E tile index of the exchange regions / flags (tail units: counted from the first tail m tile)
    const int tile = ((erow - (has_tail ? args.n_full * 2 * C::BM : 0)) / C::BM) * (args.L / kLB) + u.l0 / kLB;
    // exchange region of (tile, split s): [kChunks][128 rows] x 16 B
    auto region = [&](int s_) { return args.slab + ((size_t)tile * S + s_) * (kChunks * 128 * 4); };
    auto slab_flag = [&](int s_) { return args.flags + (1u << 17) + tile * 16 + s_; };
    // Only the epilogue warps, which observed every earlier completion of e_full in order, wait
    // for the last unit's: a warp that has not would read parity (my_units - 1) & 1 against a
    // barrier still in an earlier phase (with a tail unit, parity 1 before the first completion
    // passes at once -- found on hardware: the tail's upper column halves were read too early).
    if (warp >= 4) mbar_wait_cluster(e_full, (my_units - 1) & 1);
    __syncthreads();
    tc_fence_after();
    if (issuer) FF_STAMP(30);
    // shared memory (drained stages): slot j != sp = [kChunks][R rows][16 B] partner j's
    // partial of this split's rows (TMA), then the bf16 E rows [kLB/64][R][128 B] (SW128)
    // for one TMA store.  The own partial of this split's rows stays in TMEM until the sum.
    const uint32_t slot0 = base;
    const uint32_t ebuf = base + S * R * kChunks * 16;
    // Every thread loads its row's half of the E partial (kLB/2 columns) from TMEM once,
    // with a single wait: rows of another split's slice go straight to this split's
    // exchange region, rows of this split's slice stay in registers for the sum.
    constexpr int kHalf = kLB / 2;
    // S >= 4: 128/S rows leave 2 of 8 warps owning the split's rows, so the sum runs on all 256
    // threads through shared memory (LLaMA-1B, S = 4: tail ~1 us shorter); S = 2 keeps the owners'
    // register sum, which reads half the shared-memory bytes (GPT-6.7B: ~1.5 us shorter than the
    // wide sum; profiles/r02/s6/tail_sum_ab.log)
    const bool wide_sum = S >= 4;
    float ev[kHalf];
    tmem_ld32xn<kHalf / 32>(lane_base + e_col + c_lo, ev);
#ifndef FF_AB_TAIL  // A/B builds only (results invalid): 1 no region stores, 2 + no partner wait/load, 3 no sum
#define FF_AB_TAIL 0
#endif
    if (slice != sp && FF_AB_TAIL != 1 && FF_AB_TAIL != 2) {
      float* const dst = region(sp) + row * 4 + (size_t)(c_lo / 4) * 512;
#pragma unroll
      for (int k = 0; k < kHalf / 4; ++k)
        st_global_v4(dst + (size_t)k * 512, __float_as_uint(ev[4 * k]), __float_as_uint(ev[4 * k + 1]),
                     __float_as_uint(ev[4 * k + 2]), __float_as_uint(ev[4 * k + 3]));
    } else if (slice == sp && wide_sum) {
      // own rows into (otherwise unused) slot sp, laid out like the partners' slots: the sum below
      // then spreads over all 256 threads instead of the 2 * 128/S row owners
      const uint32_t own = slot0 + sp * (R * kChunks * 16) + (row - sp * R) * 16 + (c_lo / 4) * (R * 16);
#pragma unroll
      for (int k = 0; k < kHalf / 4; ++k)
        st_shared_v4(own + k * (R * 16), __float_as_uint(ev[4 * k]), __float_as_uint(ev[4 * k + 1]),
                     __float_as_uint(ev[4 * k + 2]), __float_as_uint(ev[4 * k + 3]));
    }
    // the barrier orders every thread's region stores before the issuer's
    // gpu-scope release (cumulative; the split-K semaphore pattern), no
    // per-thread fence
    __syncthreads();
    if (issuer) {
      FF_STAMP(24);
      st_release_gpu_u32(slab_flag(sp), epoch);
      if (args.prof) args.prof[vcta * FF_PROF_STRIDE + 25] = globaltimer_ns();
      uint32_t polls = 0;
      for (int j = 0; j < S && FF_AB_TAIL != 2; ++j) {
        if (j == sp) continue;
        while (ld_relaxed_gpu_u32(slab_flag(j)) != epoch)
          if (++polls == FF_WATCHDOG_POLLS) FF_WD_EXPIRED(((unsigned long long)ld_relaxed_gpu_u32(slab_flag(j)) << 32) | epoch);
      }
      fence_acq_rel_gpu();
      fence_proxy_async_global();
      if (args.prof) args.prof[vcta * FF_PROF_STRIDE + 27] = globaltimer_ns();
      if (FF_AB_TAIL != 2) {
        mbar_expect_tx(e_load, (uint32_t)((S - 1) * R * kChunks * 16));
        for (int j = 0; j < S; ++j)
          if (j != sp)
            tma_load_3d(slot0 + j * (R * kChunks * 16), &maps.slab, e_load, 0, sp * R / 8, (tile * S + j) * kChunks);
      }
    }
    __syncwarp();  // the issuer's lanes wait for it here, not spinning on e_load (it would starve the polls)
    if (FF_AB_TAIL != 2) mbar_wait(e_load, 0);
    if (issuer && args.prof) args.prof[vcta * FF_PROF_STRIDE + 28] = globaltimer_ns();
    // wide sum: the S slots in split order (deterministic), cast, stage bf16 [kLB/64][R][128 B]
    // (SW128) for one TMA store: 16-byte items (column chunk c, row rr) of the split's R rows, item
    // it = c * R + rr, consecutive threads on consecutive rows (512 contiguous bytes per warp and slot)
    if (wide_sum) {
      const int n_items = R * kChunks;
#pragma unroll 1
      for (int it0 = tid; it0 < n_items; it0 += 4 * 256) {
        float4 acc[4];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) acc[q4] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
        for (int j = 0; j < S && FF_AB_TAIL != 3; ++j) {
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            if (it0 + 256 * q4 >= n_items) continue;
            const float4 f = ld_shared_f4(slot0 + j * (R * kChunks * 16) + (it0 + 256 * q4) * 16);
            acc[q4].x += f.x;
            acc[q4].y += f.y;
            acc[q4].z += f.z;
            acc[q4].w += f.w;
          }
        }
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const int it = it0 + 256 * q4;
          if (it >= n_items) continue;
          const int c = it / R, rr = it - c * R;
          const int ch = (c % 16) / 2;
          st_shared_v2(ebuf + (c / 16) * (R * 128) + rr * 128 + ((ch ^ (rr & 7)) << 4) + (c & 1) * 8,
                       pack2(args.f16, acc[q4].x, acc[q4].y), pack2(args.f16, acc[q4].z, acc[q4].w));
        }
      }
    } else if (slice == sp) {
      // owners' sum (deterministic order: own partial, then the partners in split order), cast,
      // stage bf16.  The own partial is in registers; a warp's 32 rows of one 16-byte column
      // chunk of a partner slot are 512 contiguous bytes, and the bf16 row stores are SW128
      // (8 rows cover all banks).
      const int rr = row - sp * R;
      const uint32_t part = slot0 + rr * 16 + (c_lo / 4) * (R * 16);
#pragma unroll
      for (int k = 0; k < kHalf / 4; k += 8) {  // 32 columns per round
#pragma unroll 1
        for (int j = 0; j < S && FF_AB_TAIL != 3; ++j) {
          if (j == sp) continue;
          float4 f[8];
#pragma unroll
          for (int i = 0; i < 8; ++i)
            f[i] = ld_shared_f4(part + j * (R * kChunks * 16) + (k + i) * (R * 16));
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            ev[4 * (k + i)] += f[i].x;
            ev[4 * (k + i) + 1] += f[i].y;
            ev[4 * (k + i) + 2] += f[i].z;
            ev[4 * (k + i) + 3] += f[i].w;
          }
        }
        const int c0 = c_lo + 4 * k;  // first column of the round
        const int ch = (c0 % 64) / 8;
        const uint32_t dst = ebuf + (c0 / 64) * (R * 128) + rr * 128;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          st_shared_v4(dst + (((ch + i) ^ (rr & 7)) << 4), pack2(args.f16, ev[4 * k + 8 * i], ev[4 * k + 8 * i + 1]),
                       pack2(args.f16, ev[4 * k + 8 * i + 2], ev[4 * k + 8 * i + 3]),
                       pack2(args.f16, ev[4 * k + 8 * i + 4], ev[4 * k + 8 * i + 5]),
                       pack2(args.f16, ev[4 * k + 8 * i + 6], ev[4 * k + 8 * i + 7]));
      }
    }
    if (issuer && args.prof) args.prof[vcta * FF_PROF_STRIDE + 22] = globaltimer_ns();
    fence_proxy_async_smem();
    __syncthreads();
    if (issuer) {
      tma_store_3d_h(&maps.er, ebuf, 0, erow + sp * R, u.l0 / 64, l2_policy(args.epolicy));
      bulk_commit();
      FF_STAMP(26);
      bulk_wait_read0();
    }
    // (off the critical path: after the sum, the discards no longer delay its loads)
    if (args.discard & 1) {  // the partners' rows of this slice are read exactly once: drop them from L2
      const int lines = kChunks * R / 8;  // 128-byte lines of one (region, slice) block
      for (int j = 0; j < S; ++j) {
        if (j == sp) continue;
        const uint8_t* blk = reinterpret_cast<const uint8_t*>(region(j)) + sp * R * 16;
        for (int i = tid; i < lines; i += 256)
          discard_l2_line(blk + (size_t)(i / (R / 8)) * 2048 + (i % (R / 8)) * 128);
      }
    }
  }

  if (discard_c) {
    // once every member of the ring has read its last chunk, drop this CTA's half of its own
    // chunk regions (c_slots x 128 rows x kN0 columns) from L2 instead of writing them back;
    // the done flags were published right after the members' last hops, long before their
    // tails end, so the poll finds them set
    if (warp == 2) {
      uint32_t polls = 0;
      for (int j = (int)lane_id(); j < G; j += 32)
        while (ld_relaxed_gpu_u32(done_flag(j)) != epoch)
          if (++polls == FF_WATCHDOG_POLLS) FF_WD_EXPIRED(((unsigned long long)ld_relaxed_gpu_u32(done_flag(j)) << 32) | epoch);
      fence_acq_rel_gpu();
    }
    __syncthreads();
    constexpr int kRowLines = C::kN0 * 2 / 128;
    const int lines = args.c_slots * C::BM * kRowLines;
    for (int i = (int)threadIdx.x; i < lines; i += 256) {
      const int slot = i / (C::BM * kRowLines), r = (i / kRowLines) % C::BM, c = i % kRowLines;
      const size_t row = (size_t)((ring * G + p) * args.c_slots + slot) * (2 * C::BM) + (int)q * C::BM + r;
      discard_l2_line(reinterpret_cast<const uint8_t*>(args.cscratch) + row * (C::kN0 * 2) + c * 128);
    }
  }
  __syncthreads();
  cluster_sync();
  if (threadIdx.x == 0) FF_STAMP(31);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair<512>(tmem_base);
  }
}

#undef FF_PROF_ROW
#define FF_PROF_ROW blockIdx.x

}  // namespace ff
