// Host side of the fused-chain runtime: plan lowering, TMA descriptors,
// launch, and the C ABI declared in include/ff_chain.h.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <mutex>
#include <string>

#include "../../include/ff_chain.h"
#include "ff_chain_kernel.cuh"
#include "ff_chain_pair_kernel.cuh"

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

// CapacityExceeded (errors.py:32-45): `tensor` does not fit at or above tier `floor`
// by `unplaced` bytes; the Python binding rebuilds the exception from this text.
int fail_capacity(const char* tensor, const char* floor, long long unplaced, const std::string& msg) {
  return fail(FF_ERR_CAPACITY, std::string(tensor) + ":" + floor + ":" + std::to_string(unplaced) + "|" + msg);
}

CUtensorMapDataType elem_type(const ffChainDesc* ch) {
  return ch->dtype == FF_DTYPE_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
}

// ---------------------------------------------------------------------------
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
// ---------------------------------------------------------------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

using EncodeIm2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeIm2colFn encode_im2col_fn() {
  static EncodeIm2colFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeIm2colFn>(p);
  });
  return fn;
}

// NHWC bf16 feature map [n][h][w][c] -> im2col map for a k1 x k1, stride-1,
// same-padding convolution: boxes of 128 output pixels x 64 channels (one
// 128-byte SW128 row per pixel, the K-major UMMA A layout).  Bounding box
// corners -pad / pad-(k1-1) make the traversal enumerate exactly the h x w
// output positions; the tap offsets (s, r) then address the input pixel and
// out-of-image taps read zeros.
bool make_map_im2col(CUtensorMap* map, const void* ptr, int channels, int w, int h, int batch, int k,
                     CUtensorMapDataType dt) {
  EncodeIm2colFn fn = encode_im2col_fn();
  if (!fn) return false;
  const int pad = k / 2;
  cuuint64_t dims[4] = {(cuuint64_t)channels, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)batch};
  cuuint64_t strides[3] = {(cuuint64_t)channels * 2, (cuuint64_t)w * channels * 2,
                           (cuuint64_t)h * w * channels * 2};
  int lower[2] = {-pad, -pad};
  int upper[2] = {pad - (k - 1), pad - (k - 1)};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(map, dt, 4, const_cast<void*>(ptr), dims, strides, lower, upper, 64,
                  128, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  // Same descriptor fix-up as CUTLASS's make_im2col_tma_copy for drivers
  // <= 13.1 on tensors below 128 KB (cute/atom/copy_traits_sm90_im2col.hpp).
  int drv = 0;
  if (cudaDriverGetVersion(&drv) == cudaSuccess && drv <= 13010 &&
      (uint64_t)batch * h * w * channels * 2 < 131072)
    reinterpret_cast<uint64_t*>(map)[1] &= ~(1ull << 21);
  return true;
}

// Row-major bf16 matrix [rows][cols] -> 2-D map with a (box_cols x box_rows) box, 128B swizzle.
bool make_map(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_cols,
              uint32_t box_rows, CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Generic N-D map (dims innermost first; strides in bytes for dims 1..rank-1).
bool make_map_nd(CUtensorMap* map, CUtensorMapDataType dt, int rank, const void* ptr, const uint64_t* dims,
                 const uint64_t* strides, const uint32_t* box,
                 CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = 1;
    if (i + 1 < rank) st[i] = strides[i];
  }
  return fn(map, dt, rank, const_cast<void*>(ptr), d, st, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
            swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

constexpr int kMaxDevices = 64;

int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  return dev;
}

// SM count of the current device (cached per device ordinal).
int num_sms_cached() {
  static std::atomic<int> n[kMaxDevices];
  const int dev = current_device();
  int v = n[dev].load(std::memory_order_relaxed);
  if (v <= 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    n[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

// One-time per-(kernel, device) function attributes: attributes apply to the
// current device only, so a process that launches on several GPUs sets them on
// each.  Returns the first error (sticky per device).
template <typename Fn>
cudaError_t once_per_device(std::once_flag (&flags)[kMaxDevices], cudaError_t (&errs)[kMaxDevices], Fn fn) {
  const int dev = current_device();
  std::call_once(flags[dev], [&] { errs[dev] = fn(); });
  return errs[dev];
}

// Launches that spin on other CTAs' flags need the whole grid co-resident: they
// are cooperative.  A profiler that replays kernels (ncu) cannot replay a
// cooperative cluster launch, so with one attached (CUDA_INJECTION64_PATH, or
// FF_NO_COOPERATIVE=1) the attribute is dropped; the grid is sized to
// co-residency either way and a replaying profiler runs one kernel at a time.
bool profiler_attached() {
  for (const char* v : {"CUDA_INJECTION64_PATH", "NSIGHT_COMPUTE_HOST_PORT", "NV_COMPUTE_PROFILER_PERFWORKS_DIR"})
    if (std::getenv(v) != nullptr) return true;
  const char* pre = std::getenv("LD_PRELOAD");
  return pre != nullptr && (std::strstr(pre, "nsight") || std::strstr(pre, "Injection") || std::strstr(pre, "ncu"));
}
bool cooperative_allowed() {
  static const bool ok = std::getenv("FF_NO_COOPERATIVE") == nullptr && !profiler_attached();
  return ok;
}

// Launch with the cooperative attribute (the last of `attrs`); only a device or
// driver without cooperative support (cudaErrorNotSupported) gets a plain
// launch -- every other refusal, e.g. a grid too large to be co-resident, fails.
template <typename... KArgs, typename... Args>
cudaError_t launch_coop(cudaLaunchConfig_t& lc, void (*kern)(KArgs...), Args&&... args) {
  if (!cooperative_allowed()) lc.numAttrs -= 1;
  cudaError_t e = cudaLaunchKernelEx(&lc, kern, args...);
  if (e == cudaErrorNotSupported && cooperative_allowed()) {
    cudaGetLastError();
    lc.numAttrs -= 1;
    e = cudaLaunchKernelEx(&lc, kern, args...);
  }
  return e;
}

// ---------------------------------------------------------------------------
// kernel table
// ---------------------------------------------------------------------------
template <bool kGated, int kNB, int kLB, int kMode>
struct StagesFor {
  static constexpr int kBudget = 232448;
  using Probe = ff::ChainCfg<kGated, kNB, kLB, 1, kMode>;
  static constexpr int kFixed = Probe::kSMEM - Probe::kSTAGE - 2 * 8;  // everything but the stages
  static constexpr int kMax = (kBudget - kFixed - 64) / (Probe::kSTAGE + 16);
  static constexpr int value = kMax > 6 ? 6 : kMax;
};

// Co-resident clusters of a given size on a 148-SM B200 with ~225 KB smem per
// CTA (cudaOccupancyMaxActiveClusters, profiles/r01/dsm_bandwidth.log): the
// offline estimate used by the lowering (no device needed); launches clamp to
// the occupancy API's answer for the actual kernel and device.
int table_active_clusters(int cluster, int num_sms) {
  int n;
  switch (cluster) {
    case 1: n = 148; break;
    case 2: n = 74; break;
    case 4: n = 33; break;
    case 8: n = 15; break;
    case 16: n = 7; break;
    default: n = (148 / cluster) * 3 / 4; break;
  }
  return num_sms >= 148 ? n : (n * num_sms) / 148 > 0 ? (n * num_sms) / 148 : 1;
}

unsigned long long* g_prof = nullptr;  // diagnostics: per-CTA counters + timeline (ff_set_profile_buffer)
uint32_t g_variant = 0;  // kernel-variant selection for A/B runs and tests (ff_set_variant, FF_VARIANT_*)

struct WsLayout {
  size_t e_off, c_off, f_off, n_off, s_off, total;
  bool e_memset;  // fp32 E larger than the zero zone: clear it before the launch
};
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
// Workspace: [flags: fixed 1 MiB at offset 0][split arrival counters: fixed
// 256 KiB][fp32 E: fixed 32 MiB zone][C scratch].  The flags region only ever
// holds epoch stamps, so a stale stamp is always older than the current
// launch's epoch.  The counters and the fp32 E zone are zero between launches:
// the last contributor of every E tile re-zeroes its tile and counter
// (split_finish), and no config puts C scratch inside them, so a workspace
// zero-filled once stays valid whatever configs share it.  A split chain whose
// fp32 E exceeds the zone spills past it and clears it with a memset first.
// flag region (u32 words): [0, 2^17) ring chunk-ready flags, [2^17, 3*2^16) split-N slab
// flags, [3*2^16, 2^18 - 1) the pair kernel's per-(ring, member) "done reading the C
// scratch" flags; its last word holds the device epoch
constexpr size_t kFlagBytes = 1u << 20;
constexpr size_t kRingFlagBytes = 512u << 10;
constexpr size_t kCntBytes = 256u << 10;
constexpr size_t kEZoneBytes = 32u << 20;
// Pair kernel: N not a whole number of ring steps per split (ragged last n-step).
bool pair_ragged(const ffChainDesc* ch, const ffKernelConfig* c) {
  return ch->n != (int64_t)c->n_splits * c->steps * c->ring * c->nb;
}
// Pair kernel, non-ragged: C exchange slots per ring member.  A ring that runs more
// n-steps than slots reuses them every 3 steps (the kernel's c_row / wait_slot_free);
// one unit per ring keeps one slot per step.
int pair_c_slots(const ffKernelConfig* c) {
  return c->units > c->rings ? 3 : std::min(3, std::max(1, (int)c->steps));
}
// Pair kernel, multi-unit S == 1 launches: the last wave holds rem = units % rings units and
// would leave rings - rem rings idle; each of them is split in N into tail_S units (at most one
// per ring) of steps / tail_S n-steps that combine through the split-N reduce-scatter
// (OPT M=32768: 128 units on 9 rings, rem 2 -> 8 quarter units: 14.25 waves instead of 15).
int pair_tail_splits(const ffChainDesc* ch, const ffKernelConfig* c) {
  if (g_variant & FF_VARIANT_NO_TAIL_SPLIT) return 1;
  if (c->n_splits != 1 || c->l_clusters != 1 || c->units <= c->rings || pair_ragged(ch, c)) return 1;
  const int rem = c->units % c->rings;
  if (rem == 0) return 1;
  for (int st : {8, 4, 2})
    if (rem * st <= c->rings && c->steps % st == 0) return st;
  return 1;
}

WsLayout ws_layout(const ffChainDesc* ch, const ffKernelConfig* c, bool conv2 = false) {
  WsLayout w{};
  const bool pair = c->exchange == FF_XCHG_L2_PAIR;
  const bool dsmr = c->exchange == FF_XCHG_L2_DSMR;  // split partials meet in DSM: no fp32 E, no slab
  const size_t e_bytes = c->n_splits > 1 && !dsmr ? (size_t)ch->m * ch->l * sizeof(float) : 0;
  // C scratch: L2 transport with a ring > 1; the standard-FFN pair kernel also
  // reads its own chunk back from it (hop 0), so it always needs one.
  // (a k2 x k2 second convolution reads the whole intermediate back through im2col boxes)
  const bool c_scratch =
      c->exchange != FF_XCHG_DSM && (c->ring > 1 || conv2 || (pair && ch->kind != FF_KIND_GATED));
  w.f_off = 0;
  w.n_off = kFlagBytes;
  w.e_off = kFlagBytes + kCntBytes;
  w.e_memset = e_bytes > kEZoneBytes;
  // everything after the fp32 E zone starts past its full 32 MiB: regions of one
  // config must never overlap the zero-invariant zone another config relies on
  // (a gated ring-1 split config once put its exchange regions there)
  size_t off = w.e_off + std::max(e_bytes, kEZoneBytes);
  w.c_off = off;
  if (c_scratch) {
    if (pair && !pair_ragged(ch, c))  // per-(ring, member, slot) regions of 256 rows x nb columns
      off = align256(off + (size_t)c->rings * c->ring * pair_c_slots(c) * 256 * c->nb * 2);
    else  // the whole intermediate
      off = align256(off + (size_t)c->m_tiles * (pair ? 256 : 128) * ch->n * 2);
  }
  // pair kernel split-N reduce-scatter: one fp32 [M][L] slab per split (no zero invariant)
  w.s_off = off;
  if (c->n_splits > 1 && !dsmr)  // split-N exchange regions (pair kernel, and the 1-CTA kernels' final units)
    off = align256(off + (size_t)c->n_splits * (size_t)c->m_tiles * (pair ? 256 : 128) * ch->l * sizeof(float));
  else if (pair && pair_tail_splits(ch, c) > 1)  // tail units: regions for the last wave's m tiles only
    off = align256(off + (size_t)pair_tail_splits(ch, c) * (size_t)(c->units % c->rings) * 256 * ch->l * sizeof(float));
  w.total = off;
  return w;
}


// Split-N finish by exchange regions (pair kernel): one unit per ring, S | 128
// with 8-row slices, and the slab flags of every E tile fit their region.
bool pair_finish_regions(const ffChainDesc* ch, const ffKernelConfig* c, int rings) {
  return c->n_splits > 1 && c->n_splits <= 8 && c->units <= rings && 128 % c->n_splits == 0 &&
         (128 / c->n_splits) % 8 == 0 && (size_t)((ch->m + 255) / 256) * 2 * (ch->l / 256) * 16 < (1u << 16);
}

template <bool kGated, int kNB, int kLB, int kMode>
int launch_impl(const ffChainDesc* ch, const ffKernelConfig* cfg, const ffTensors* t, void* ws,
                void* c_debug, cudaStream_t stream, const ffConvDesc* conv) {
  constexpr int kStages = StagesFor<kGated, kNB, kLB, kMode>::value;
  static_assert(kStages >= 2, "not enough shared memory for a pipeline");
  using C = ff::ChainCfg<kGated, kNB, kLB, kStages, kMode>;
  auto kern = ff::ff_chain_kernel<kGated, kNB, kLB, kStages, kMode>;

  static std::once_flag once[kMaxDevices];
  static cudaError_t errs[kMaxDevices];
  const cudaError_t attr_err = once_per_device(once, errs, [&] {
    cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSMEM);
    if (r == cudaSuccess && kMode == ff::XCHG_DSM)
      r = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return r;
  });
  if (attr_err != cudaSuccess)
    return fail(FF_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(attr_err));

  const uint64_t M = ch->m, N = ch->n, K = ch->k, L = ch->l;
  const bool implicit = conv != nullptr && conv->k1 > 1;
  const bool conv2 = conv != nullptr && conv->k2 > 1;  // k2 x k2 second conv: GEMM1 over im2col(C)
  const WsLayout wl = ws_layout(ch, cfg, conv2);
  uint8_t* wsb = reinterpret_cast<uint8_t*>(ws);
  CUtensorMap mA, mB0, mB1, mD, mC, mCs;
  const CUtensorMapDataType dt = elem_type(ch);
  bool ok = implicit ? make_map_im2col(&mA, t->a, conv->ic, conv->w, conv->h, conv->batch, conv->k1, dt)
                     : make_map(&mA, t->a, M, K, 64, 128, dt);
  // B (standard chains) and D as 3D views {64 columns, rows, column blocks}: one TMA box fetches
  // every 64-column block of a stage (kNB/64 or kLB/64 tiles of [64 rows][64 cols], 8 KB apart)
  if (kGated) {
    ok = ok && make_map(&mB0, t->b, K, N, 64, 64, dt);
  } else {
    const uint64_t db[3] = {64, K, N / 64}, sb[2] = {N * 2, 128};
    const uint32_t bb[3] = {64, 64, kNB / 64};
    ok = ok && make_map_nd(&mB0, dt, 3, t->b, db, sb, bb);
  }
  ok = ok && make_map(&mB1, kGated ? t->b1 : t->b, K, N, 64, 64, dt);
  {
    const uint64_t drows = conv2 ? (uint64_t)conv->k2 * conv->k2 * N : N;
    const uint64_t dd[3] = {64, drows, L / 64}, sd[2] = {L * 2, 128};
    const uint32_t bd[3] = {64, 64, kLB / 64};
    ok = ok && make_map_nd(&mD, dt, 3, t->d, dd, sd, bd);
  }
  const bool l2x = (kMode == ff::XCHG_L2 && cfg->ring > 1);
  const bool cs = l2x || conv2;  // C scratch in use: [m_tiles*128][N] 2D view (publish stores, ring hops)
  ok = ok && make_map(&mCs, cs ? (const void*)(wsb + wl.c_off) : t->a, cs ? (uint64_t)cfg->m_tiles * 128 : M,
                      cs ? N : K, 64, 128, dt);
  if (conv2)  // GEMM1 operand: the scratch as an NHWC map [batch][h][w][oc1], im2col boxes of the k2 x k2 window
    ok = ok && make_map_im2col(&mC, wsb + wl.c_off, (int)N, conv->w, conv->h, conv->batch, conv->k2, dt);
  else
    mC = mCs;
  CUtensorMap mE, mW;  // E tile outputs: bf16 E [M][L] box {64, 128}; fp32 split-N workspace [M][L] box {32, 128}
  CUtensorMap mSlab, mEr;  // split-N exchange regions / E row slices (final-unit reduce-scatter)
  const int S = std::max(1, cfg->n_splits), R = 128 / S;
  {
    const uint64_t de[2] = {L, M}, se[1] = {L * 2};
    const uint32_t be[2] = {64, 128};
    ok = ok && make_map_nd(&mE, dt, 2, t->e, de, se, be);
    const uint64_t sw[1] = {L * 4};
    const uint32_t bw[2] = {32, 128};
    ok = ok && make_map_nd(&mW, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, wsb + wl.e_off, de, sw, bw);
    const uint64_t tiles = (uint64_t)cfg->m_tiles * (L / kLB);
    const uint64_t ds[3] = {32, 16, tiles * S * (kLB / 4)}, ss[2] = {128, 2048};
    const uint32_t bs[3] = {32, (uint32_t)std::max(1, R / 8), kLB / 4};
    ok = ok && make_map_nd(&mSlab, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, cfg->n_splits > 1 ? (const void*)(wsb + wl.s_off)
                                                                                        : t->e,
                           ds, ss, bs, CU_TENSOR_MAP_SWIZZLE_NONE);
    const uint64_t dr[3] = {64, M, L / 64}, sr[2] = {L * 2, 128};
    const uint32_t br[3] = {64, (uint32_t)std::min(128, R), kLB / 64};
    ok = ok && make_map_nd(&mEr, dt, 3, t->e, dr, sr, br);
  }
  if (!ok) return fail(FF_ERR_CUDA, "cuTensorMapEncodeTiled failed (alignment or driver entry point)");

  cudaLaunchConfig_t lc = {};
  lc.blockDim = dim3(256, 1, 1);
  lc.dynamicSmemBytes = C::kSMEM;
  lc.stream = stream;
  // Every launch is cooperative: ring members spin on each other's flags (L2
  // transport), split contributors on each other's arrivals (shared finish, exchange
  // regions), so the whole grid must be co-resident.  DSM rings are clusters.
  cudaLaunchAttribute attr[2];
  int nattr = 0;
  int rings;
  const bool split_cl = cfg->exchange == FF_XCHG_L2_DSMR;
  if (split_cl) {
    // the S N splits of an E tile form one cluster (their fp32 partials meet in DSM): every
    // (tile, member) cluster must be co-resident, one unit per ring
    const int S = cfg->n_splits;
    attr[nattr].id = cudaLaunchAttributeClusterDimension;
    attr[nattr].val.clusterDim.x = S;
    attr[nattr].val.clusterDim.y = 1;
    attr[nattr].val.clusterDim.z = 1;
    ++nattr;
    lc.gridDim = dim3(S, 1, 1);
    lc.attrs = attr;
    lc.numAttrs = nattr;
    int active = 0;
    if (cudaOccupancyMaxActiveClusters(&active, kern, &lc) != cudaSuccess || active <= 0) {
      cudaGetLastError();
      active = table_active_clusters(S, num_sms_cached());
    }
    if ((int64_t)cfg->units * cfg->ring > (int64_t)active * S)
      return fail(FF_ERR_UNSUPPORTED, "DSM reduce-scatter: (tile, member) clusters exceed co-residency");
    if ((size_t)128 * kLB * 4 > (size_t)C::kOFF_OWN)
      return fail(FF_ERR_UNSUPPORTED, "DSM reduce-scatter: E tile larger than the pipeline stages");
    rings = cfg->units;
  } else if (kMode == ff::XCHG_DSM) {
    attr[nattr].id = cudaLaunchAttributeClusterDimension;
    attr[nattr].val.clusterDim.x = cfg->ring;
    attr[nattr].val.clusterDim.y = 1;
    attr[nattr].val.clusterDim.z = 1;
    ++nattr;
    lc.gridDim = dim3(cfg->ring, 1, 1);
    lc.attrs = attr;
    lc.numAttrs = nattr;
    int active = 0;
    if (cudaOccupancyMaxActiveClusters(&active, kern, &lc) != cudaSuccess || active <= 0) {
      cudaGetLastError();
      active = table_active_clusters(cfg->ring, num_sms_cached());
    }
    rings = std::min(cfg->units, active);
  } else {
    rings = std::min(cfg->units, num_sms_cached() / cfg->ring);
    if (rings < 1) return fail(FF_ERR_UNSUPPORTED, "ring larger than the number of SMs");
  }
  attr[nattr].id = cudaLaunchAttributeCooperative;
  attr[nattr].val.cooperative = 1;
  ++nattr;
  lc.attrs = attr;
  lc.numAttrs = nattr;
  lc.gridDim = dim3(rings * cfg->ring, 1, 1);

  ff::ChainArgs a{};
  a.M = (int)M;
  a.N = (int)N;
  a.K = (int)K;
  a.L = (int)L;
  a.G = cfg->ring;
  a.S = cfg->n_splits;
  a.steps = cfg->steps;
  a.m_tiles = cfg->m_tiles;
  a.l_clusters = cfg->l_clusters;
  a.n_units = cfg->units;
  a.n_rings = rings;
  a.act = ch->activation;
  a.dev_epoch = reinterpret_cast<uint32_t*>(wsb + wl.f_off) + (kFlagBytes / 4 - 1);  // last flag-region word
  a.exit_cnt = reinterpret_cast<uint32_t*>(wsb + wl.n_off) + (kCntBytes / 4 - 1);    // last counter word
  a.E = reinterpret_cast<__nv_bfloat16*>(t->e);
  a.ws = reinterpret_cast<float*>(wsb + wl.e_off);
  a.flags = reinterpret_cast<uint32_t*>(wsb + wl.f_off);
  a.tile_cnt = reinterpret_cast<uint32_t*>(wsb + wl.n_off);
  a.c_debug = reinterpret_cast<__nv_bfloat16*>(c_debug);
  a.prof = g_prof;
  a.f16 = ch->dtype == FF_DTYPE_F16 ? 1 : 0;
  a.krot = (g_variant & FF_VARIANT_NO_KROT) ? 0 : 1;
  a.slab = reinterpret_cast<float*>(wsb + wl.s_off);
  a.split_cl = split_cl ? 1 : 0;
  // final-unit split-N reduce-scatter through exchange regions (FF_VARIANT_FINISH_REGIONS, opt-in): one
  // unit per ring, 8-row slices, the S slots (the whole fp32 tile) in the drained stages
  // and the bf16 row slice in the own slot.  Measured slower than the TMA reduce-add +
  // last-arriver finish for GPT-2s (29.7 vs 26.6 us, profiles/r01/timeline_gpt2s_regions.log):
  // with S = 8 both move ~11-13 MB of fp32 partials into a dirty L2 at once, and the
  // region path adds the partner loads
  a.finish_tma = !split_cl && S > 1 && S <= 8 && 128 % S == 0 && R % 8 == 0 && cfg->units <= rings && !conv2 &&
                 (size_t)128 * kLB * 4 <= (size_t)C::kOFF_OWN && (size_t)R * kLB * 2 <= (size_t)C::kCHUNK_BYTES &&
                 (size_t)cfg->m_tiles * (L / kLB) * 16 < (1u << 17) && (g_variant & FF_VARIANT_FINISH_REGIONS);
  if (implicit || conv2) {
    a.conv_k1 = implicit ? conv->k1 : 0;
    a.conv_H = conv->h;
    a.conv_W = conv->w;
    a.conv_cblk = conv->ic / 64;
    a.conv2_k = conv2 ? conv->k2 : 0;
    a.conv2_cblk = (int)(N / 64);
  }

  if (wl.e_memset) {
    cudaError_t e0 = cudaMemsetAsync(wsb + wl.e_off, 0, (size_t)M * L * sizeof(float), stream);
    if (e0 != cudaSuccess) return fail(FF_ERR_CUDA, std::string("memset: ") + cudaGetErrorString(e0));
  }
  cudaError_t e = launch_coop(lc, kern, mA, mB0, mB1, mD, mC, mCs, mE, mW, mSlab, mEr, a);
  if (e != cudaSuccess) return fail(FF_ERR_CUDA, std::string("cudaLaunchKernelEx: ") + cudaGetErrorString(e));

  return FF_OK;
}

template <bool kGated>
struct PairStages {
  using Probe = ff::PairCfg<kGated, 256, 1>;
  static constexpr int kFixed = Probe::kSMEM - Probe::kSTAGE - 2 * 8;
  static constexpr int kMax = (232448 - kFixed - 64) / (Probe::kSTAGE + 16);
  static constexpr int value = kMax > 4 ? 4 : kMax;
};

template <bool kGated, bool kPacked, bool kQuad, bool kRagged>
int launch_pair_impl(const ffChainDesc* ch, const ffKernelConfig* cfg, const ffTensors* t, void* ws, void* c_debug,
                     cudaStream_t stream, const ffConvDesc*) {
  constexpr int kStages = PairStages<kGated>::value;
  static_assert(kStages >= 2, "not enough shared memory for a pipeline");
  using C = ff::PairCfg<kGated, 256, kStages>;
  auto kern = ff::ff_chain_pair_kernel<kGated, 256, kStages, kPacked, kQuad, kRagged>;
  static std::once_flag once[kMaxDevices];
  static cudaError_t errs[kMaxDevices];
  static int max_clusters[kMaxDevices];  // co-resident clusters of this kernel (occupancy API), per device
  const cudaError_t attr_err = once_per_device(once, errs, [&] {
    cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSMEM);
    if (r != cudaSuccess) return r;
    cudaLaunchConfig_t probe = {};
    cudaLaunchAttribute cl[1];
    cl[0].id = cudaLaunchAttributeClusterDimension;
    cl[0].val.clusterDim.x = kQuad ? 4 : 2;
    cl[0].val.clusterDim.y = 1;
    cl[0].val.clusterDim.z = 1;
    probe.gridDim = dim3(kQuad ? 4 : 2, 1, 1);
    probe.blockDim = dim3(256, 1, 1);
    probe.dynamicSmemBytes = C::kSMEM;
    probe.attrs = cl;
    probe.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &probe) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = kQuad ? table_active_clusters(4, num_sms_cached()) : num_sms_cached() / 2;
    }
    max_clusters[current_device()] = n;
    return cudaSuccess;
  });
  if (attr_err != cudaSuccess)
    return fail(FF_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(attr_err));

  const uint64_t M = ch->m, N = ch->n, K = ch->k, L = ch->l;
  const WsLayout wl = ws_layout(ch, cfg);
  uint8_t* wsb = reinterpret_cast<uint8_t*>(ws);
  const uint64_t mpad = (uint64_t)cfg->m_tiles * 256;
  // Tensor maps are pure functions of (chain, config, pointers): encoding the
  // eleven of them costs several microseconds of host time per launch, so the
  // last few sets are kept per thread and reused when a caller launches again
  // on the same buffers (serving loops, benchmarks, graph capture).
  // tail split of the last partial wave: planned on cfg->rings (the workspace layout's
  // basis); used only when that many rings are co-resident
  const int tail_S = pair_tail_splits(ch, cfg);
  struct Key {
    ffChainDesc ch;
    int32_t ring, n_splits, nb, lb, m_tiles, units, rings, steps, tail;
    const void *a, *b, *b1, *d;
    void *e, *ws;
  };
  Key key;
  std::memset(&key, 0, sizeof(key));
  key.ch = *ch;
  key.units = cfg->units;
  key.rings = cfg->rings;
  key.steps = cfg->steps;
  key.tail = tail_S;
  key.ring = cfg->ring;
  key.n_splits = cfg->n_splits;
  key.nb = cfg->nb;
  key.lb = cfg->lb;
  key.m_tiles = cfg->m_tiles;
  key.a = t->a;
  key.b = t->b;
  key.b1 = t->b1;
  key.d = t->d;
  key.e = t->e;
  key.ws = ws;
  struct Entry {
    Key key;
    ff::PairMaps maps;
    bool valid;
  };
  thread_local Entry cache[16] = {};  // serving loops rotate buffers
  thread_local int cache_next = 0;
  ff::PairMaps maps;
  bool hit = false;
  for (auto& en : cache)
    if (en.valid && std::memcmp(&en.key, &key, sizeof(key)) == 0) {
      maps = en.maps;
      hit = true;
      break;
    }
  const auto BF = elem_type(ch);  // bf16 or fp16 storage
  bool ok = true;
  if (!hit) {
  {  // A [M][K] as {64, M, K/64}
    const uint64_t d[3] = {64, M, K / 64}, st[2] = {K * 2, 128};
    const uint32_t b[3] = {64, 128, 2};
    ok = ok && make_map_nd(&maps.a, BF, 3, t->a, d, st, b);
  }
  if (kGated && kPacked) {  // packed [2][K][N] as {64, K, N/64, 2}
    const uint64_t d[4] = {64, K, N / 64, 2}, st[3] = {N * 2, 128, K * N * 2};
    const uint32_t b[4] = {64, 128, 1, 2};
    ok = ok && make_map_nd(&maps.b, BF, 4, t->b, d, st, b);
    maps.b1 = maps.b;
  } else {
    const uint64_t d[3] = {64, K, N / 64}, st[2] = {N * 2, 128};
    const uint32_t b[3] = {64, 128, kGated ? 1u : 2u};
    ok = ok && make_map_nd(&maps.b, BF, 3, t->b, d, st, b);
    ok = ok && make_map_nd(&maps.b1, BF, 3, kGated ? t->b1 : t->b, d, st, b);
  }
  {  // D [N][L] as {64, N, L/64}
    const uint64_t d[3] = {64, N, L / 64}, st[2] = {L * 2, 128};
    const uint32_t b[3] = {64, 128, 2};
    ok = ok && make_map_nd(&maps.d, BF, 3, t->d, d, st, b);
  }
  {  // C exchange scratch: regions [rings*G*slots][256 rows][nb] as {64, regions*256, nb/64}
     // (ragged: the whole intermediate [mpad][N] as {64, mpad, N/64})
    const bool l2x = cfg->ring > 1 || !kGated;
    const uint64_t rows = kRagged ? mpad : (uint64_t)cfg->rings * cfg->ring * pair_c_slots(cfg) * 256;
    const uint64_t cols = kRagged ? N : (uint64_t)C::kN0;
    const uint64_t d[3] = {64, l2x ? rows : M, l2x ? cols / 64 : K / 64}, st[2] = {(l2x ? cols : K) * 2, 128};
    const uint32_t b[3] = {64, 128, 2};
    ok = ok && make_map_nd(&maps.c, BF, 3, l2x ? (const void*)(wsb + wl.c_off) : t->a, d, st, b);
  }
  {  // E [M][L] bf16, box {64, 128}
    const uint64_t d[2] = {L, M}, st[1] = {L * 2};
    const uint32_t b[2] = {64, 128};
    ok = ok && make_map_nd(&maps.e, BF, 2, t->e, d, st, b);
  }
  {  // fp32 workspace [M][L], box {32, 128}
    const uint64_t d[2] = {L, M}, st[1] = {L * 4};
    const uint32_t b[2] = {32, 128};
    ok = ok && make_map_nd(&maps.w, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, cfg->n_splits > 1 ? (const void*)(wsb + wl.e_off) : t->e,
                           d, st, b);
  }
  {  // whole-tile / row-slice 3D views of E and the fp32 workspace (final-unit epilogue)
    // split row slice (the reduce-scatter tail needs S <= 8, pair_finish_regions; the maps
    // are encoded for every launch, so keep their boxes legal for any S)
    const int s_eff = tail_S > 1 ? tail_S : std::max(1, cfg->n_splits);  // splits meeting in the tail
    const uint32_t rs = std::max(1u, 128u / (uint32_t)s_eff);
    const uint64_t de[3] = {64, M, L / 64}, se[2] = {L * 2, 128};
    const uint32_t be[3] = {64, 128, 256 / 64}, ber[3] = {64, rs, 256 / 64};
    ok = ok && make_map_nd(&maps.e3, BF, 3, t->e, de, se, be);
    ok = ok && make_map_nd(&maps.er, BF, 3, t->e, de, se, ber);
    const void* wp = cfg->n_splits > 1 ? (const void*)(wsb + wl.e_off) : t->e;
    const uint64_t dw[3] = {32, M, L / 32}, sw[2] = {L * 4, 128};
    const uint32_t bw[3] = {32, 128, 256 / 32};
    ok = ok && make_map_nd(&maps.w3, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, wp, dw, sw, bw);
    // split-N exchange regions [E tile][split][16-byte chunk][128 rows] x 16 B as a 3D
    // {8 rows x 4 floats, 16 row groups, chunk}: box {32, 128/S/8, 64} = one split's
    // rows of a slice, 128-byte inner rows (lands as [chunk][row][16 B] in smem)
    const uint64_t S = (uint64_t)s_eff;
    const void* sp = s_eff > 1 ? (const void*)(wsb + wl.s_off) : t->e;
    // tail units: regions for the last wave's m tiles only (ws_layout)
    const uint64_t tiles = (uint64_t)(tail_S > 1 ? cfg->units % cfg->rings : cfg->m_tiles) * 2 * (L / 256);
    const uint64_t ds[3] = {32, 16, tiles * S * 64}, ss[2] = {128, 2048};
    const uint32_t bs[3] = {32, std::max(1u, rs / 8), 64};
    ok = ok && make_map_nd(&maps.slab, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, sp, ds, ss, bs, CU_TENSOR_MAP_SWIZZLE_NONE);
  }
    if (ok) {
      cache[cache_next].key = key;
      cache[cache_next].maps = maps;
      cache[cache_next].valid = true;
      cache_next = (cache_next + 1) % 16;
    }
  }
  if (!ok) return fail(FF_ERR_CUDA, "cuTensorMapEncodeTiled failed (alignment or driver entry point)");

  if (cfg->ring > 64) return fail(FF_ERR_UNSUPPORTED, "ring of more than 64 pairs");
  // co-resident rings: pairs the occupancy API guarantees for this kernel on this device
  const int pairs = max_clusters[current_device()] * (kQuad ? 2 : 1);
  int rings = std::min(cfg->units, pairs / cfg->ring);
  if (kQuad) rings &= ~1;  // rings in X/Y couples
  // the C scratch is laid out for cfg->rings rings; fewer co-resident rings than
  // planned (another tenant's occupancy) may need slot reuse the layout lacks
  if (!kRagged && rings < cfg->units && pair_c_slots(cfg) < 3)
    return fail(FF_ERR_UNSUPPORTED, "fewer co-resident CTA pairs than the launch was planned for");
  if (rings < 1) return fail(FF_ERR_UNSUPPORTED, "ring of pairs larger than the GPU");
  ff::ChainArgs a{};
  a.M = (int)M;
  a.N = (int)N;
  a.K = (int)K;
  a.L = (int)L;
  a.G = cfg->ring;
  a.S = cfg->n_splits;
  a.steps = cfg->steps;
  a.total_chunks = (int)(N / C::kN0);
  a.split_chunks = (a.total_chunks + cfg->n_splits - 1) / cfg->n_splits;
  a.m_tiles = cfg->m_tiles;
  a.l_clusters = cfg->l_clusters;
  a.n_units = cfg->units;
  a.n_rings = rings;
  // tail split (pair_tail_splits): plain pairs only (quad twins must share weights), and only
  // on the planned ring count the workspace was laid out for
  if (!kQuad && tail_S > 1 && rings == cfg->rings) {
    a.tail_S = tail_S;
    a.n_full = cfg->units - cfg->units % rings;
    a.n_units = a.n_full + (cfg->units % rings) * tail_S;
  } else {
    a.tail_S = 1;
    a.n_full = cfg->units;
  }
  a.act = ch->activation;
  a.dev_epoch = reinterpret_cast<uint32_t*>(wsb + wl.f_off) + (kFlagBytes / 4 - 1);  // last flag-region word
  a.exit_cnt = reinterpret_cast<uint32_t*>(wsb + wl.n_off) + (kCntBytes / 4 - 1);    // last counter word
  a.E = reinterpret_cast<__nv_bfloat16*>(t->e);
  a.ws = reinterpret_cast<float*>(wsb + wl.e_off);
  a.flags = reinterpret_cast<uint32_t*>(wsb + wl.f_off);
  a.tile_cnt = reinterpret_cast<uint32_t*>(wsb + wl.n_off);
  a.slab = reinterpret_cast<float*>(wsb + wl.s_off);
  a.c_debug = reinterpret_cast<__nv_bfloat16*>(c_debug);
  a.prof = g_prof;
  a.f16 = ch->dtype == FF_DTYPE_F16 ? 1 : 0;
  // hops deferred past GEMM0(T+1): about one C drain (+ its store for the
  // standard FFN, whose hop 0 reads the own chunk back from L2) worth of MMA
  // GEMM0 of step t+1 entirely before the remote hops of step t (defer = G-1): since the epilogue
  // drains C ahead of E at unit boundaries this beats spreading it over the first G/4 hops
  // (OPT M=4096 -1.5 %, A/B; profiles/r01/cfgs_defer.log had 3/4 before that change)
  a.defer = cfg->ring - 1;
  // split-N reduce-scatter through per-split slabs (else: atomic reduce-add + last-arriver finish)
  a.finish_tma = pair_finish_regions(ch, cfg, rings);
  // L2 prefetch of weight tiles 2 k-blocks / hops ahead (profiles/r01/cold_prefetch.log): launches of one or two
  // waves read the weights from HBM and gain (GPT-6.7B -6 us, LLaMA-1B -2 us, OPT M=4096 -1 %); rings of many
  // units find them in L2, where the prefetch instructions only occupy the TMA unit (OPT M=32768: -2 % without;
  // r02 s6f / s6g A/Bs)
#ifndef FF_AB_PREFETCH_DIST  // A/B builds only: another prefetch distance
#define FF_AB_PREFETCH_DIST 2
#endif
  a.prefetch = cfg->units > 2 * rings ? 0 : FF_AB_PREFETCH_DIST;
  // staggered GEMM0 k order (measured: GPT-6.7B 118.8 -> 114.7 us, profiles/r01/krot.log);
  // FF_VARIANT_NO_KROT restores the common order
  a.krot = (g_variant & FF_VARIANT_NO_KROT) ? 0 : 1;
  a.defer_last = 1;
  a.c_slots = kRagged ? 0 : pair_c_slots(cfg);
  // L2 policies (A/B timelines in profiles/r02/l2_policy_ab.log): the C exchange scratch
  // is evict_last (GPT-6.7B -1.1 us, LLaMA-1B -1.3 us); weights keep the default
  // priority (evict_first made GPT-6.7B 6 % slower: the prefetched lines were evicted
  // before their TMA loads) unless a variant asks otherwise
  a.wpolicy = (g_variant & FF_VARIANT_WEIGHTS_EVICT_FIRST) ? ff::L2_EVICT_FIRST
              : (g_variant & FF_VARIANT_WEIGHTS_EVICT_LAST) ? ff::L2_EVICT_LAST
                                                            : ff::L2_NORMAL;
  a.cpolicy = (g_variant & FF_VARIANT_SCRATCH_NORMAL) ? ff::L2_NORMAL : ff::L2_EVICT_LAST;
  a.epolicy = (g_variant & FF_VARIANT_E_EVICT_FIRST) ? ff::L2_EVICT_FIRST : ff::L2_NORMAL;
  // dead split-N exchange regions leave L2 without a DRAM write-back (FF_VARIANT_NO_DISCARD: keep
  // them).  Measured (profiles/r02/discard_ab.md): GPT-6.7B DRAM 286.0 -> 277.8 MB (1.004x the
  // algorithmic bytes), LLaMA-1B 118.2 -> 105.9 MB, no time cost; also discarding the C scratch
  // at exit (FF_VARIANT_SCRATCH_DISCARD) moves no further bytes and costs 1-2 us
  a.discard = (g_variant & FF_VARIANT_NO_DISCARD) ? 0 : (g_variant & FF_VARIANT_SCRATCH_DISCARD) ? 3 : 1;
  a.cscratch = reinterpret_cast<__nv_bfloat16*>(wsb + wl.c_off);
  // rings that run several units: odd units walk their n-steps backwards so they start on
  // the weights the previous unit read last (OPT M=4096: second wave of units re-read the
  // weights from DRAM; FF_VARIANT_NO_SERP restores the common order)
  a.serp = (!kRagged && rings < cfg->units && !(g_variant & FF_VARIANT_NO_SERP)) ? 1 : 0;
  if (wl.e_memset) {
    cudaError_t e0 = cudaMemsetAsync(wsb + wl.e_off, 0, (size_t)M * L * sizeof(float), stream);
    if (e0 != cudaSuccess) return fail(FF_ERR_CUDA, std::string("memset: ") + cudaGetErrorString(e0));
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(rings * cfg->ring * 2, 1, 1);
  lc.blockDim = dim3(256, 1, 1);
  lc.dynamicSmemBytes = C::kSMEM;
  lc.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kQuad ? 4 : 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = 1;
  lc.attrs = attr;
  lc.numAttrs = 2;  // cooperative + cluster: the rings spin on each other's flags (launch_coop)
  cudaError_t e = launch_coop(lc, kern, maps, a);
  if (e != cudaSuccess) return fail(FF_ERR_CUDA, std::string("cudaLaunchKernelEx(pair): ") + cudaGetErrorString(e));
  return FF_OK;
}

// Quad (weight-multicast) variant when the units come in m-tile couples that
// share their weights: an even number of m tiles, an even number of rings of
// at most one unit each... any even ring count works (units 2j / 2j+1 pair up).
bool quad_ok(const ffKernelConfig* cfg, bool gated) {
  if (g_variant & FF_VARIANT_NO_QUAD) return false;  // A/B and tests: force the plain pair kernel
  if (cfg->m_tiles % 2 || cfg->units % 2) return false;
  const int pair_rings = std::min(cfg->units, num_sms_cached() / (2 * cfg->ring));
  int rings = std::min(pair_rings, 4 * table_active_clusters(4, num_sms_cached()) / (2 * cfg->ring)) & ~1;
  if (rings < 2) return false;
  if (g_variant & FF_VARIANT_FORCE_QUAD) return true;  // A/B and tests: quad whenever it can launch
  // Quads wherever they launch.  The chip runs these chains at its board power cap, so the
  // quad's halved L2 reads of the weights show up as energy per chain and clock, not as feed:
  // GPT-6.7B sustained (profiles/r02/s6/quad_energy.log) 122.0-123.0 vs 124.1-126.0 us per step at
  // 3-4 % less energy, bench.py headline 1186 vs 1174 TF/s (bench_ab_quad.log), although an interleaved
  // A/B -- both variants sharing one power state -- had plain pairs 1 % ahead (s5/ab_quad_long.log).
  // LLaMA-1B: +2.6 % on plain pairs; OPT M=4096 is 0.8 % faster on 9 plain rings but moves 171.6
  // instead of 161.7 MB of DRAM (9 rings of C scratch, a 9 + 7 second wave; r02s5v vs r02s5o)
  // quads need an even ring count: when that costs a wave of units (OPT M=32768: 128 units
  // on 8 quad rings = 16 waves vs 9 pair rings = 15), plain pairs win (-2.4 %, A/B)
  const int waves_quad = (cfg->units + rings - 1) / rings, waves_pair = (cfg->units + pair_rings - 1) / pair_rings;
  return waves_quad <= waves_pair;
}

template <bool kGated, bool kPacked>
int launch_pair_q(const ffChainDesc* ch, const ffKernelConfig* cfg, const ffTensors* t, void* ws, void* c_debug,
                  cudaStream_t stream, const ffConvDesc* conv) {
  // ragged n-steps (N not a whole number of ring steps per split): plain pairs only
  if (ch->n != (int64_t)cfg->n_splits * cfg->steps * cfg->ring * cfg->nb)
    return launch_pair_impl<kGated, kPacked, false, true>(ch, cfg, t, ws, c_debug, stream, conv);
  // (a tail-split launch needs plain pairs: quad twins share weight tiles, tail units do not)
  return quad_ok(cfg, kGated) && pair_tail_splits(ch, cfg) == 1
             ? launch_pair_impl<kGated, kPacked, true, false>(ch, cfg, t, ws, c_debug, stream, conv)
                      : launch_pair_impl<kGated, kPacked, false, false>(ch, cfg, t, ws, c_debug, stream, conv);
}

int launch_pair_dispatch(const ffChainDesc* ch, const ffKernelConfig* cfg, const ffTensors* t, void* ws,
                         void* c_debug, cudaStream_t stream, const ffConvDesc* conv) {
  if (conv != nullptr && conv->k1 > 1) return fail(FF_ERR_UNSUPPORTED, "implicit-GEMM conv needs the 1-CTA kernel");
  if (ch->kind != FF_KIND_GATED) return launch_pair_q<false, false>(ch, cfg, t, ws, c_debug, stream, conv);
  // gate|up packed as one [2][K][N] tensor: one TMA box fetches both branches
  const bool packed = reinterpret_cast<const uint8_t*>(t->b1) ==
                      reinterpret_cast<const uint8_t*>(t->b) + (size_t)ch->k * ch->n * 2;
  return packed ? launch_pair_q<true, true>(ch, cfg, t, ws, c_debug, stream, conv)
                : launch_pair_q<true, false>(ch, cfg, t, ws, c_debug, stream, conv);
}

using LaunchFn = int (*)(const ffChainDesc*, const ffKernelConfig*, const ffTensors*, void*, void*, cudaStream_t,
                         const ffConvDesc*);

// Can N be cut into S splits of this config's chunks?  The 1-CTA kernels need
// whole n-steps in equal splits; the pair kernel takes ceil(chunks / S) chunks
// per split and a ragged last n-step (the last split shorter), as long as
// every split keeps at least one chunk.
bool splits_ok(const ffChainDesc* ch, const ffKernelConfig* c, int64_t S) {
  if (S < 1) return false;
  if (c->exchange != FF_XCHG_L2_PAIR) return ch->n % (S * c->ring * c->nb) == 0;
  if (ch->n % c->nb) return false;
  const int64_t chunks = ch->n / c->nb, per = (chunks + S - 1) / S;
  return chunks - (S - 1) * per >= 1;
}

LaunchFn select_kernel(bool gated, int nb, int lb, int mode) {
  if (mode == FF_XCHG_L2_PAIR) {
    if (nb != (gated ? 128 : 256) || lb != 256) return nullptr;
    return &launch_pair_dispatch;
  }
#define FF_CASE(G, NB, LB)                                                    \
  if (gated == G && nb == NB && lb == LB)                                     \
    return mode == FF_XCHG_DSM ? &launch_impl<G, NB, LB, ff::XCHG_DSM>        \
                               : &launch_impl<G, NB, LB, ff::XCHG_L2>; /* L2 and L2_DSMR */
  FF_CASE(false, 128, 256)
  FF_CASE(false, 128, 128)
  FF_CASE(false, 128, 64)
  FF_CASE(false, 64, 256)
  FF_CASE(false, 64, 128)
  FF_CASE(false, 64, 64)
  FF_CASE(true, 64, 256)
  FF_CASE(true, 64, 128)
  FF_CASE(true, 64, 64)
#undef FF_CASE
  return nullptr;
}

int validate_chain(const ffChainDesc* ch) {
  if (!ch) return fail(FF_ERR_ARG, "null chain descriptor");
  if (ch->kind != FF_KIND_STANDARD && ch->kind != FF_KIND_GATED) return fail(FF_ERR_ARG, "unknown chain kind");
  if (ch->activation < 0 || ch->activation > FF_ACT_GELU_TANH) return fail(FF_ERR_ARG, "unknown activation");
  if (ch->element_size != 2)
    return fail(FF_ERR_UNSUPPORTED, "GPU path executes 2-byte storage (bf16 / fp16, element_size 2) only");
  if (ch->dtype != FF_DTYPE_BF16 && ch->dtype != FF_DTYPE_F16) return fail(FF_ERR_ARG, "unknown dtype");
  if (ch->m < 1 || ch->n < 64 || ch->k < 64 || ch->l < 64)
    return fail(FF_ERR_UNSUPPORTED, "extents below one 64-wide tile");
  if (ch->k % 64 || ch->n % 64 || ch->l % 64)
    return fail(FF_ERR_UNSUPPORTED, "n, k, l must be multiples of 64 for the sm_100a kernel");
  if (ch->m > (1ll << 31) || ch->n > (1ll << 31) || ch->k > (1ll << 31) || ch->l > (1ll << 31))
    return fail(FF_ERR_UNSUPPORTED, "extent too large");
  return FF_OK;
}

// Fill derived fields and check that a physical configuration is executable.
int finish_config(const ffChainDesc* ch, ffKernelConfig* c, int num_sms) {
  const bool gated = ch->kind == FF_KIND_GATED;
  if (c->exchange != FF_XCHG_DSM && c->exchange != FF_XCHG_L2 && c->exchange != FF_XCHG_L2_PAIR &&
      c->exchange != FF_XCHG_L2_DSMR)
    return fail(FF_ERR_ARG, "unknown exchange");
  if (c->exchange == FF_XCHG_L2_DSMR && (c->n_splits < 2 || c->n_splits > 8 || 128 % c->n_splits))
    return fail(FF_ERR_UNSUPPORTED, "DSM reduce-scatter needs 2, 4 or 8 N splits (one cluster per E tile)");
  const int width = c->exchange == FF_XCHG_L2_PAIR ? 2 : 1;  // CTAs per ring member
  if (c->ring < 1 || c->ring > (c->exchange == FF_XCHG_DSM ? 16 : num_sms / width))
    return fail(FF_ERR_UNSUPPORTED, "ring size out of range (DSM rings are clusters of <= 16 CTAs)");
  if (c->n_splits < 1) return fail(FF_ERR_UNSUPPORTED, "n_splits must be >= 1");
  if (!select_kernel(gated, c->nb, c->lb, c->exchange)) return fail(FF_ERR_UNSUPPORTED, "no kernel for (nb, lb)");
  if (c->exchange == FF_XCHG_L2_PAIR && (ch->k % 128 || c->lb != 256))
    return fail(FF_ERR_UNSUPPORTED, "pair kernel needs k % 128 == 0 and 256-column E slices");
  const int64_t lcover = (int64_t)c->ring * c->lb;
  if (ch->l % lcover) return fail(FF_ERR_UNSUPPORTED, "ring * lb must divide l");
  if (!splits_ok(ch, c, c->n_splits))
    return fail(FF_ERR_UNSUPPORTED, c->exchange == FF_XCHG_L2_PAIR
                                        ? "nb must divide n and every N split must keep a chunk"
                                        : "n_splits * ring * nb must divide n");
  c->l_clusters = (int32_t)(ch->l / lcover);
  {  // pair kernel: ceil(chunks / S) chunks per split, the last n-step possibly ragged
    const int64_t per = (ch->n / c->nb + c->n_splits - 1) / c->n_splits;
    c->steps = (int32_t)((per + c->ring - 1) / c->ring);
  }
  const int rows = 128 * width;
  c->m_tiles = (int32_t)((ch->m + rows - 1) / rows);
  const int64_t units = (int64_t)c->m_tiles * c->l_clusters * c->n_splits;
  if (units > (1ll << 30)) return fail(FF_ERR_UNSUPPORTED, "grid too large");
  c->units = (int32_t)units;
  const int64_t max_rings =
      c->exchange == FF_XCHG_DSM ? table_active_clusters(c->ring, num_sms) : num_sms / (c->ring * width);
  c->rings = (int32_t)std::min<int64_t>(units, max_rings);
  if (c->exchange == FF_XCHG_L2_DSMR) {
    // every split cluster co-resident at once (one unit per ring, the tiles' S CTAs meet in DSM)
    if (units * c->ring > (int64_t)table_active_clusters(c->n_splits, num_sms) * c->n_splits)
      return fail(FF_ERR_UNSUPPORTED, "DSM reduce-scatter needs every (tile, member) cluster co-resident");
    c->rings = (int32_t)units;
  }
  c->grid_ctas = c->rings * c->ring * width;
  return FF_OK;
}

int pick_lb(int64_t cover, int max_ring) {
  for (int lb : {256, 128, 64})
    if (cover % lb == 0 && cover / lb <= max_ring) return lb;
  return 0;
}

// Grow the number of N splits while the units do not yet fill the co-resident rings.
void fill_machine(const ffChainDesc* ch, ffKernelConfig* c, int num_sms) {
  const int width = c->exchange == FF_XCHG_L2_PAIR ? 2 : 1;
  const int max_rings =
      c->exchange == FF_XCHG_DSM ? table_active_clusters(c->ring, num_sms) : num_sms / (c->ring * width);
  const bool dsmr = c->exchange == FF_XCHG_L2_DSMR;
  if (dsmr && c->n_splits < 2 && splits_ok(ch, c, 2)) c->n_splits = 2;  // a split cluster needs >= 2 splits
  for (;;) {
    const int64_t per = (int64_t)((ch->m + 128 * width - 1) / (128 * width)) * (ch->l / ((int64_t)c->ring * c->lb));
    const int64_t next = (int64_t)c->n_splits * 2;
    if (dsmr && (next > 8 || per * next * c->ring > (int64_t)table_active_clusters((int)next, num_sms) * next)) break;
    if (per * next > max_rings) break;
    if (!splits_ok(ch, c, next)) break;
    c->n_splits = (int32_t)next;
  }
}

}  // namespace

extern "C" {

const char* ff_last_error(void) { return g_last_error.c_str(); }

// Diagnostics: when non-NULL, kernels write per-CTA wait-cycle counters
// (unsigned long long[grid_ctas][16]) into this device buffer.
void ff_set_profile_buffer(void* dev_ptr) { g_prof = reinterpret_cast<unsigned long long*>(dev_ptr); }
void ff_set_variant(uint32_t flags) { g_variant = flags; }

#ifdef FF_DIAG_WATCHDOG
// Diagnostic builds only: out[0] = waits expired since the last call, out[1 + 2i] = source line << 40 |
// block << 20 | thread and out[2 + 2i] = wait-specific info of the first 512; then cleared.
int ff_diag_read(unsigned long long* out) {
  cudaError_t e = cudaMemcpyFromSymbol(out, ff::ff_diag, sizeof(ff::ff_diag));
  static const unsigned long long z[1 + 2 * 512] = {};
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(ff::ff_diag, z, sizeof(z));
  return e == cudaSuccess ? FF_OK : FF_ERR_CUDA;
}
#endif
const char* ff_version(void) { return "ff_chain 0.1.0 sm_100a"; }

int ff_auto_config_ex(const ffChainDesc* ch, int32_t num_sms, int32_t exchange, ffKernelConfig* out) {
  int rc = validate_chain(ch);
  if (rc) return rc;
  if (!out) return fail(FF_ERR_ARG, "null output");
  if (num_sms <= 0) num_sms = 148;
  ffKernelConfig c = {};
  c.exchange = exchange;
  const bool gated = ch->kind == FF_KIND_GATED;
  const int max_ring = exchange == FF_XCHG_DSM ? 16 : (exchange == FF_XCHG_L2_PAIR ? num_sms / 2 : num_sms);
  // E slice width lb (widest first), then the largest ring of lb slices whose
  // n-step (ring * nb C columns) divides N; l slices the ring does not cover
  // become l clusters (each recomputes GEMM0 for its part of L)
  const bool pair = exchange == FF_XCHG_L2_PAIR;
  const int nb_opts[2] = {pair ? (gated ? 128 : 256) : (gated ? 64 : 128), pair ? 0 : 64};
  c.lb = 0;
  for (int lb : {256, 128, 64}) {
    if (c.lb || ch->l % lb || (pair && lb != 256)) continue;
    const int64_t slices = ch->l / lb;
    for (int64_t ring = std::min<int64_t>(slices, max_ring); ring >= 1 && !c.lb; --ring) {
      if (slices % ring) continue;
      for (int nb : nb_opts)
        if (nb && ch->n % ((pair ? 1 : ring) * nb) == 0) {
          c.lb = lb;
          c.ring = (int32_t)ring;
          c.nb = nb;
          break;
        }
    }
  }
  if (!c.lb) return fail(FF_ERR_UNSUPPORTED, "no ring of E slices whose C chunks tile n");
  c.n_splits = 1;
  fill_machine(ch, &c, num_sms);
  // A chain too small to occupy half the SMs with rings of one CTA (a latency-bound
  // conv tile row): narrower E slices, i.e. more l clusters that each recompute
  // their cheap GEMM0 (conv C5: 25 -> 100 CTAs, 15.3 -> 13.3 us, profiles/r01/conv_sweep.log)
  if (exchange != FF_XCHG_L2_PAIR && c.ring == 1) {
    const int64_t m_tiles = (ch->m + 127) / 128;
    while (c.lb > 64 && m_tiles * (ch->l / c.lb) * c.n_splits < num_sms / 2) c.lb /= 2;
  }
  rc = finish_config(ch, &c, num_sms);
  if (rc) return rc;
  *out = c;
  return FF_OK;
}

int ff_auto_config(const ffChainDesc* ch, int32_t num_sms, ffKernelConfig* out) {
  return ff_auto_config_ex(ch, num_sms, FF_XCHG_L2, out);
}

int ff_plan_lower_ex(const ffChainDesc* ch, const ffPlanDesc* plan, int32_t num_sms, int32_t exchange,
                     ffKernelConfig* out) {
  int rc = validate_chain(ch);
  if (rc) return rc;
  if (!plan || !out) return fail(FF_ERR_ARG, "null plan or output");
  if (num_sms <= 0) num_sms = 148;
  const bool gated = ch->kind == FF_KIND_GATED;
  if (gated && plan->gated_lowering == FF_LOWERING_NA)
    return fail(FF_ERR_PLAN, "gated chain requires a lowering (spatial_split or doubled_k)");
  if (!gated && plan->gated_lowering != FF_LOWERING_NA)
    return fail(FF_ERR_PLAN, "standard chain cannot carry a gated lowering");
  const int32_t cm = plan->cluster[0], cn = plan->cluster[1], ck = plan->cluster[2], cl = plan->cluster[3];
  if (cm < 1 || cn < 1 || ck < 1 || cl < 1) return fail(FF_ERR_PLAN, "cluster dims must be positive");
  if (cl % ck) return fail(FF_ERR_PLAN, "cls_k does not divide cls_l");
  if ((cn * ck) % cl) return fail(FF_ERR_PLAN, "cls_l does not divide cls_n*cls_k");
  if ((plan->spatial_mask >> 3) & 1u) return fail(FF_ERR_PLAN, "output-column dimension is grid-spatial");
  const int64_t ext[4] = {ch->m, ch->n, gated && plan->gated_lowering == FF_LOWERING_DOUBLED_K ? 2 * ch->k : ch->k,
                          ch->l};
  for (int d = 0; d < 4; ++d)
    if (plan->block[d] <= 0 || ext[d] % plan->block[d]) return fail(FF_ERR_PLAN, "block tile does not divide extent");

  // Logical -> physical:
  //  * the plan's l cover of one cluster (cls_l * blk_l) becomes one shuffle
  //    ring of CTAs holding <= 256 TMEM columns of E each;
  //  * cls_reduce sets and grid-spatial N clusters become N splits whose E
  //    partials are reduced across rings (inter-cluster reduce);
  //  * M trips (any blk_m) become independent 128-row work units (M is never
  //    reduced), distributed over co-resident rings;
  //  * the gated branches (spatial_split or doubled_k) execute as two TMEM
  //    accumulators of one CTA, combined by the epilogue (all_exchange Mul).
  ffKernelConfig c = {};
  c.exchange = exchange;
  const int64_t lcover = (int64_t)cl * plan->block[3];
  c.lb = pick_lb(lcover, exchange == FF_XCHG_DSM ? 16 : (exchange == FF_XCHG_L2_PAIR ? num_sms / 2 : num_sms));
  if (!c.lb || (exchange == FF_XCHG_L2_PAIR && c.lb < 128))
    return fail(FF_ERR_UNSUPPORTED, "plan's l cover cannot be split into ring members of <= 256 columns");
  c.ring = (int32_t)(lcover / c.lb);
  const int64_t ncover = (int64_t)cn * plan->block[1];  // cluster n cover (plan.py:236)
  const int64_t grid_n = ((plan->spatial_mask >> 1) & 1u) ? ch->n / ncover : 1;
  const int32_t reduce_sets = (cn * ck) / cl;
  c.n_splits = (int32_t)(grid_n * reduce_sets);
  c.nb = exchange == FF_XCHG_L2_PAIR ? (gated ? 128 : 256) : (gated ? 64 : 128);
  if (exchange == FF_XCHG_L2_DSMR)
    while (c.n_splits > 8) c.n_splits /= 2;  // one portable cluster of split partners
  while (c.n_splits > 1 && !splits_ok(ch, &c, c.n_splits)) c.n_splits /= 2;
  if (!splits_ok(ch, &c, c.n_splits) && exchange != FF_XCHG_L2_PAIR) c.nb = 64;
  if (!splits_ok(ch, &c, c.n_splits)) return fail(FF_ERR_UNSUPPORTED, "n cannot be partitioned into ring chunks");
  fill_machine(ch, &c, num_sms);
  rc = finish_config(ch, &c, num_sms);
  if (rc) return rc;
  *out = c;
  return FF_OK;
}

int ff_plan_lower(const ffChainDesc* ch, const ffPlanDesc* plan, int32_t num_sms, ffKernelConfig* out) {
  return ff_plan_lower_ex(ch, plan, num_sms, FF_XCHG_DSM, out);
}

size_t ff_chain_workspace_bytes(const ffChainDesc* ch, const ffKernelConfig* cfg_in) {
  if (!ch || !cfg_in) return 0;
  ffKernelConfig cfg = *cfg_in;
  if (finish_config(ch, &cfg, 148)) return 0;
  return ws_layout(ch, &cfg).total;
}

int ff_config_finish(const ffChainDesc* ch, int32_t num_sms, ffKernelConfig* cfg) {
  int rc = validate_chain(ch);
  if (rc) return rc;
  if (!cfg) return fail(FF_ERR_ARG, "null config");
  ffKernelConfig c = *cfg;
  rc = finish_config(ch, &c, num_sms > 0 ? num_sms : 148);
  if (rc) return rc;
  *cfg = c;
  return FF_OK;
}

int ff_config_deterministic(const ffChainDesc* ch, const ffKernelConfig* cfg, int32_t num_sms, int32_t* out) {
  int rc = validate_chain(ch);
  if (rc) return rc;
  if (!cfg || !out) return fail(FF_ERR_ARG, "null config or output");
  if (num_sms <= 0) num_sms = 148;
  ffKernelConfig c = *cfg;
  rc = finish_config(ch, &c, num_sms);
  if (rc) return rc;
  // Every E element is summed in a fixed order when nothing is summed across CTAs (one N split:
  // the ring accumulates all of N in one TMEM tile; the pair kernel's tail units meet through the
  // exchange regions, own partial first, then the partners in split order), when the S splits of a
  // tile reduce over DSM in split order (FF_XCHG_L2_DSMR), or when the pair kernel finishes its
  // splits through the exchange regions (one unit per ring, pair_finish_regions).  Otherwise the
  // split partials meet through TMA reduce-adds into the fp32 zone, whose add order follows the
  // CTAs' timing.
  bool det;
  if (c.n_splits == 1 || c.exchange == FF_XCHG_L2_DSMR)
    det = true;
  else if (c.exchange == FF_XCHG_L2_PAIR)
    det = pair_finish_regions(ch, &c, c.rings);
  else
    det = false;  // 1-CTA DSM / L2 rings with N splits (the region finish is an opt-in variant)
  *out = det ? 1 : 0;
  return FF_OK;
}

int ff_chain_kernel_count(const ffChainDesc* ch, const ffKernelConfig* cfg) {
  if (!ch || !cfg) return 0;
  // split-N reduction and the bf16 cast finish inside the chain kernel; only
  // an fp32 E beyond the workspace's zero zone adds a memset
  return ws_layout(ch, cfg).e_memset ? 2 : 1;
}

static int launch_common(const ffChainDesc* ch, const ffKernelConfig* cfg_in, const ffTensors* t, void* ws,
                         size_t ws_bytes, void* c_debug, void* stream, const ffConvDesc* conv = nullptr) {
  int rc = validate_chain(ch);
  if (rc) return rc;
  if (!cfg_in || !t || !t->a || !t->b || !t->d || !t->e) return fail(FF_ERR_ARG, "null tensor pointer");
  const bool gated = ch->kind == FF_KIND_GATED;
  if (gated && !t->b1) return fail(FF_ERR_ARG, "gated chain needs B1");
  for (const void* p : {t->a, t->b, t->d, (const void*)t->e})
    if (reinterpret_cast<uintptr_t>(p) % 16) return fail(FF_ERR_ARG, "tensors must be 16-byte aligned");
  ffKernelConfig cfg = *cfg_in;
  rc = finish_config(ch, &cfg, num_sms_cached());
  if (rc) return rc;
  const size_t need = ws_layout(ch, &cfg, conv != nullptr && conv->k2 > 1).total;
  if (need && (ws == nullptr || ws_bytes < need)) return fail(FF_ERR_ARG, "workspace too small");
  // L2 ready flags live in the lower half of the flag region (the pair
  // kernel's split slab flags use the upper half)
  if (cfg.exchange != FF_XCHG_DSM &&
      (size_t)cfg.units * cfg.steps * cfg.ring * 2 * sizeof(uint32_t) > kRingFlagBytes)
    return fail(FF_ERR_UNSUPPORTED, "too many (unit, step, member) chunks for the flag region");
  if (cfg.n_splits > 1 && (size_t)((ch->m + 255) / 256) * 2 * (ch->l / cfg.lb) * sizeof(uint32_t) >= kCntBytes)
    return fail(FF_ERR_UNSUPPORTED, "too many E tiles for the split arrival counters");
  if (ws && reinterpret_cast<uintptr_t>(ws) % 256) return fail(FF_ERR_ARG, "workspace must be 256-byte aligned");
  LaunchFn fn = select_kernel(gated, cfg.nb, cfg.lb, cfg.exchange);
  return fn(ch, &cfg, t, ws, c_debug, reinterpret_cast<cudaStream_t>(stream), conv);
}

int ff_chain_launch(const ffChainDesc* ch, const ffKernelConfig* cfg, const ffTensors* t, void* ws,
                    size_t ws_bytes, void* stream) {
  return launch_common(ch, cfg, t, ws, ws_bytes, nullptr, stream);
}

int ff_chain_launch_debug(const ffChainDesc* ch, const ffKernelConfig* cfg, const ffTensors* t, void* ws,
                          size_t ws_bytes, void* c_out, void* stream) {
  return launch_common(ch, cfg, t, ws, ws_bytes, c_out, stream);
}

// ---- conv chain (workload.py:168-199) as an implicit GEMM ----
int ff_conv_chain_desc(const ffConvDesc* cv, ffChainDesc* out) {
  if (!cv || !out) return fail(FF_ERR_ARG, "null conv descriptor or output");
  if (cv->batch < 1 || cv->h < 1 || cv->w < 1 || cv->ic < 1 || cv->oc1 < 1 || cv->oc2 < 1 || cv->k1 < 1 || cv->k2 < 1)
    return fail(FF_ERR_ARG, "conv extents must be positive");
  if (cv->k2 != 1 && cv->k1 != 1)
    return fail(FF_ERR_UNSUPPORTED, "one of the two convolutions must be pointwise (1x1)");
  if (cv->k1 % 2 == 0 || cv->k2 % 2 == 0) return fail(FF_ERR_UNSUPPORTED, "same padding needs an odd filter size");
  if (cv->k2 > 1 && cv->oc1 > 128)  // the whole 128-pixel intermediate tile stays in one CTA's TMEM / smem
    return fail_capacity("C", "smem", (long long)(cv->oc1 - 128) * 128 * 2,
                         "k2 x k2 second conv keeps every CTA's whole intermediate tile (oc1 <= 128 channels) on chip");
  if (cv->k2 > 1 && (cv->oc1 % 64 || (cv->oc2 != 64 && cv->oc2 != 128 && cv->oc2 != 256)))
    return fail(FF_ERR_UNSUPPORTED, "k2 x k2 second conv: oc1 in {64, 128}, oc2 in {64, 128, 256}");
  if (cv->k2 > 1 && (cv->k2 / 2 > 127 || cv->h > 65535 || cv->w > 65535))
    return fail(FF_ERR_UNSUPPORTED, "filter / feature map outside the im2col TMA ranges");
  if (cv->k1 > 1 && cv->ic % 64)
    return fail(FF_ERR_UNSUPPORTED, "implicit-GEMM conv needs input channels in multiples of 64");
  if (cv->k1 > 1 && (cv->k1 / 2 > 127 || cv->h > 65535 || cv->w > 65535))
    return fail(FF_ERR_UNSUPPORTED, "filter / feature map outside the im2col TMA ranges");
  ffChainDesc ch = {};
  ch.kind = FF_KIND_STANDARD;
  ch.activation = cv->activation;
  ch.m = (int64_t)cv->batch * cv->h * cv->w;
  ch.n = cv->oc1;
  ch.k = (int64_t)cv->k1 * cv->k1 * cv->ic;
  ch.l = cv->oc2;
  ch.element_size = 2;
  ch.dtype = cv->dtype;
  *out = ch;
  return validate_chain(&ch);
}

int ff_conv_chain_lower(const ffConvDesc* cv, int32_t num_sms, int32_t exchange, ffKernelConfig* out) {
  ffChainDesc ch;
  int rc = ff_conv_chain_desc(cv, &ch);
  if (rc) return rc;
  if (cv->k1 > 1 && exchange == FF_XCHG_L2_PAIR)
    return fail(FF_ERR_UNSUPPORTED, "implicit-GEMM conv runs on the 1-CTA kernels (dsm / l2 exchange)");
  if (cv->k2 > 1) {
    // 1x1 conv -> act -> k2 x k2 conv: every CTA computes the whole intermediate
    // (all oc1 channels) of its 128-pixel tile, publishes it through the L2
    // scratch, and GEMM1 reads im2col boxes of it once its neighbour tiles
    // (the k2 x k2 halo rows) are published too
    if (exchange != FF_XCHG_L2) return fail(FF_ERR_UNSUPPORTED, "k2 x k2 second conv runs on the l2 exchange");
    if (!out) return fail(FF_ERR_ARG, "null output");
    ffKernelConfig c = {};
    c.exchange = FF_XCHG_L2;
    c.ring = 1;
    c.n_splits = 1;
    c.nb = cv->oc1;
    c.lb = cv->oc2;
    rc = finish_config(&ch, &c, num_sms <= 0 ? 148 : num_sms);
    if (rc) return rc;
    if (c.units > c.rings) return fail(FF_ERR_UNSUPPORTED, "feature map needs more 128-pixel tiles than SMs");
    *out = c;
    return FF_OK;
  }
  return ff_auto_config_ex(&ch, num_sms, exchange, out);
}

size_t ff_conv_chain_workspace_bytes(const ffConvDesc* cv, const ffKernelConfig* cfg_in) {
  ffChainDesc ch;
  if (ff_conv_chain_desc(cv, &ch) || !cfg_in) return 0;
  ffKernelConfig cfg = *cfg_in;
  if (finish_config(&ch, &cfg, 148)) return 0;
  return ws_layout(&ch, &cfg, cv->k2 > 1).total;
}

int ff_conv_chain_launch(const ffConvDesc* cv, const ffKernelConfig* cfg, const ffTensors* t, void* ws,
                         size_t ws_bytes, void* stream) {
  ffChainDesc ch;
  int rc = ff_conv_chain_desc(cv, &ch);
  if (rc) return rc;
  if (cfg && cv->k1 > 1 && cfg->exchange == FF_XCHG_L2_PAIR)
    return fail(FF_ERR_UNSUPPORTED, "implicit-GEMM conv runs on the 1-CTA kernels (dsm / l2 exchange)");
  if (cfg && cv->k2 > 1 &&
      (cfg->exchange != FF_XCHG_L2 || cfg->ring != 1 || cfg->n_splits != 1 || cfg->nb != cv->oc1 || cfg->lb != cv->oc2))
    return fail(FF_ERR_UNSUPPORTED, "k2 x k2 second conv needs the configuration of ff_conv_chain_lower");
  if (cfg && cv->k2 > 1) {  // every tile's CTA co-resident: the halo waits must not block an unscheduled tile
    ffKernelConfig c2 = *cfg;
    int rc2 = finish_config(&ch, &c2, num_sms_cached());
    if (rc2) return rc2;
    if (c2.units > c2.rings) return fail(FF_ERR_UNSUPPORTED, "feature map needs more 128-pixel tiles than SMs");
  }
  return launch_common(&ch, cfg, t, ws, ws_bytes, nullptr, stream, cv);
}

// The plan's lowering under the first transport that executes it: CTA pairs
// (cta_group::2, the production kernel), then the 1-CTA L2 and DSM kernels.
static int lower_plan_any(const ffChainDesc* ch, const ffPlanDesc* plan, ffKernelConfig* cfg) {
  int rc = FF_ERR_UNSUPPORTED;
  for (int x : {FF_XCHG_L2_PAIR, FF_XCHG_L2, FF_XCHG_DSM}) {
    rc = ff_plan_lower_ex(ch, plan, num_sms_cached(), x, cfg);
    if (rc != FF_ERR_UNSUPPORTED) return rc;
  }
  return rc;
}

size_t ff_plan_workspace_bytes(const ffChainDesc* ch, const ffPlanDesc* plan) {
  ffKernelConfig cfg;
  if (lower_plan_any(ch, plan, &cfg)) return 0;
  return ws_layout(ch, &cfg).total;
}

int ff_chain_run_plan(const ffChainDesc* ch, const ffPlanDesc* plan, const ffTensors* t, void* ws,
                      size_t ws_bytes, void* stream) {
  ffKernelConfig cfg;
  int rc = lower_plan_any(ch, plan, &cfg);
  if (rc) return rc;
  return launch_common(ch, &cfg, t, ws, ws_bytes, nullptr, stream);
}

}  // extern "C"
