// mp_gather.cu — step a5: gather every window's crop from its full-resolution
// RGB24 frame and bilinearly resample it to its size class's detector-input
// dims (PAPER.md:152 — the detector runs batched "at each of those sizes";
// resampling convention R15/R16 in DESIGN.md §3).  HBM-bound: this kernel
// carries ~99% of the path's bytes.
//
// Launches:
//   memset               per-class window counters
//   gather_prep_kernel   grid-stride over the windows (n_win read on device):
//                        validate, count per class (shared then one global
//                        atomic per CTA), per-class slot -> window index lists,
//                        and the per-class exact integer tap tables (i0,
//                        lambda) for both axes (R15).
//   gather_kernel<fmt>   persistent, warp-specialised, one CTA per SM.
//                        Warp 8 = producer: the next tile's window record and
//                        tap bounds are prefetched while it waits for a free
//                        stage; then the tile's tap slices (two 1-D bulk copies)
//                        and its source box (ONE 3-D TMA tensor copy over the
//                        frame batch on the strided entry point, or one 1-D
//                        bulk copy per source row on the pointer-array entry
//                        point) land in a 2- or 3-stage shared-memory ring completing
//                        on an mbarrier (complete_tx).  Warps 0-7 = consumers:
//                        output columns lane + 32j (packed f32x2 math),
//                        separable lerps reusing staged rows, streaming stores.
#include <cuda.h>
#include <stdio.h>

#include <atomic>
#include <mutex>
#include <stdlib.h>

#include "mp_internal.cuh"

namespace mpk {

constexpr int kProducerWarps = 1;
#ifndef MP_TILE_CHUNK
#define MP_TILE_CHUNK 2
#endif
constexpr int kTileChunk = MP_TILE_CHUNK;   // tiles per dynamic-scheduling ticket
#ifndef MP_KCW
#define MP_KCW 8
#endif
// consumer warps per CTA (each owns a block of TR / cw output rows): cw_of()
#ifndef MP_KCW_U8
#define MP_KCW_U8 12
#endif
// u8 output from RGB24 runs 12 consumer warps (the fixed-tap consumer is
// latency-bound at 8: 128 registers x 416 threads; gather alone c2 0.860 ->
// 0.748 ms, c3 3.62 -> 3.02, c4 2.39 -> 1.92; f32 is faster with 8: c2 1.369
// vs 1.429 ms; 16 warps spill; profiles/ab/r02_consumer_warps_r43.jsonl)
__host__ __device__ constexpr int cw_of(int fmt, int src) {
  return (fmt == MP_OUT_U8_NHWC && src == 0) ? MP_KCW_U8 : MP_KCW;
}
constexpr int kStages = 2;      // default ring depth (A.stages; MP_GATHER_STAGES overrides, <= kMaxStages)
constexpr int kStagesF32 = 3;   // f32 output: 3 x 40 KB (measured c2 1.424 -> 1.389 ms, c3 6.86 -> 6.35, c4 4.22 -> 4.27
                                // against 2 x 44 KB; 2 x 40 KB is slower, 1.53)
constexpr int kMaxStages = 8;
// Shared memory per SM left free by the gather's ring for co-running side
// CTAs: the largest plan / remap-NMS tier CTA is ~53 KB (+1 KB driver reserve).
constexpr size_t kSideReserve = 56 * 1024;
constexpr int kHdrBytes = 64;
constexpr int kMaxTW = 256;
constexpr int kMaxTR = 192;   // Rw <= 8 rows per consumer warp (<= 16 warps); r43 tiles <= 64 row groups
constexpr int kXtapBytes = (kMaxTW + 2) * 8, kYtapBytes = (kMaxTR + 2) * 8;
constexpr int kTapBytes = kXtapBytes + kYtapBytes;
constexpr int kStageDataBudget = 40 * 1024;        // dense classes, RGB f32 output (three stages, kStagesF32)
constexpr int kStageDataBudgetWide = 56 * 1024;    // RGB f32 classes with ow > 512 (full-frame windows)
constexpr int kStageDataBudgetNV12 = 44 * 1024;    // dense classes, NV12 f32 output (two stages: 3 x 40 KB measured
                                                   // 1.311 -> 1.346 ms on c2)
constexpr int kStageDataBudgetU8 = 80 * 1024;      // dense classes, u8 output: the consumer is the bound (4x fewer
                                                   // bytes written), and taller tiles mean fewer horizontal lerps per
                                                   // output row (measured: c2 1.32 -> 1.18 ms, c3 6.08 -> 5.58,
                                                   // c4 3.63 -> 3.27; f32 is slower with larger stages)
constexpr int kSparseStageBudget = 96 * 1024;      // row-sparse classes (measured: 44 KB -> 1.44 ms, 96 KB -> 0.93 ms
                                                   // for the c2 proxy-input downscale; bytes in flight per SM)
constexpr int kDataOff = (kHdrBytes + kTapBytes + 127) / 128 * 128;   // TMA destination: 128-B aligned

struct GatherArgs {
  int k, W, H, pitch, F, fmt, stage_bytes, stages, debug, tensor, src;
  int wait_mode;             // bit 0: producer sleeps on empty slots, bit 1: consumers sleep on full slots
  int rpf;                   // row-sparse: rows per frame in the 2-D row view of the frame batch
  int max_windows;           // capacity of the windows buffer: n_win = min(frame_off[F], max_windows)
  int lam_off;               // MP_LAM_SMEM builds: byte offset of the per-warp lambda-pair scratch
  int r43[kMaxClasses];      // u8 NHWC from RGB24, exact 4:3 downscale on both axes: fixed-tap consumer
  int obuf_off;              // byte offset of the r43 consumer's per-warp output-row buffers (0: none)
  int ncol[kMaxClasses];
  int box_w[kMaxClasses], box_h[kMaxClasses];
  int w[kMaxClasses], h[kMaxClasses], ow[kMaxClasses], oh[kMaxClasses];
  int TW[kMaxClasses], TR[kMaxClasses], nct[kMaxClasses], tpw[kMaxClasses];
  int cap[kMaxClasses], list_off[kMaxClasses], xtab_off[kMaxClasses], ytab_off[kMaxClasses];
  int uv_off[kMaxClasses];   // NV12: byte offset of the staged chroma box (after the luma box)
  int box_huv[kMaxClasses];  // NV12: staged chroma box rows
  int sparse[kMaxClasses];   // row-sparse staging: only each output row's tap rows are staged
  int pair_bytes[kMaxClasses];   // row-sparse: staged bytes per output row (RGB 2 rows, NV12 4 rows)
  float cvt[6];              // NV12 (R23): cy, -cy*yo, crv, cgu, cgv, cbu (fp32 of the fp64 coefficients)
  void* out[kMaxClasses];
};

enum { kSrcRGB24 = 0, kSrcNV12 = 1 };


// One TMA tensor map per size class (box = the class's staged tile footprint);
// NV12 adds one per class for the chroma plane at m[kMaxClasses + q].
struct TmapArray {
  CUtensorMap m[2 * kMaxClasses];
};

struct TileHdr {
  int valid, k, slot, oy0, ox0, rows, cols, stride;
  int x, b0, r_lo, xs, ys;   // window x, staged byte origin, first staged row, tap slice shifts
  int ya;                    // NV12: absolute first staged luma row (its chroma row is ya >> 1)
  int wy;                    // window y
  int pad[1];
};
static_assert(sizeof(TileHdr) <= kHdrBytes, "header");

// R15 exact integer taps: n = (2d+1)*in - out; i0 = floor(n / 2out) (n<0 -> 0),
// lambda = (n mod 2out) / 2out (fp32 of exact integers, one rounding);
// i0 >= in-1 -> (in-1, 0); i1 = min(i0+1, in-1).
__device__ __forceinline__ void tap(int in, int out, int d, int& i0, float& lam) {
  const int n = (2 * d + 1) * in - out;
  int a = 0, rem = 0;
  if (n >= 0) {
    a = n / (2 * out);
    rem = n - a * 2 * out;
  }
  if (a >= in - 1) {
    a = in - 1;
    rem = 0;
  }
  i0 = a;
  lam = __fdiv_rn((float)rem, (float)(2 * out));
}

// Packed f32x2 FMA on 64-bit register pairs (PTX fma.rn.f32x2, sm_100+): an
// operand kept as ONE b64 value stays in an aligned register pair, so the
// per-column weight pairs are not re-packed (2 MOVs) before every FFMA2.
__device__ __forceinline__ unsigned long long pk2(float2 v) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(v.x), "f"(v.y));
  return r;
}
__device__ __forceinline__ float2 upk2(unsigned long long v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ float2 ffma2_w(float2 a, unsigned long long w, float2 c) {   // a * w + c
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk2(a)), "l"(w), "l"(pk2(c)));
  return upk2(r);
}

#ifdef MP_LAM_SMEM
constexpr int kMaxNP = 4;   // column pairs per lane (NCOL <= 8)
__device__ __forceinline__ unsigned long long lds64(unsigned int addr) {
  unsigned long long v;
  asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(addr));
  return v;
}
#endif

__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {   // packed a - b (FADD2 with negated operand)
  return __fadd2_rn(a, make_float2(-b.x, -b.y));
}

// u8 -> (2^23 + u8) as an fp32 bit pattern; subtracting 2^23 afterwards is exact.
__device__ __forceinline__ float u8m(uint32_t b) { return __int_as_float(0x4B000000u + b); }

// (U, V) byte of a 16-bit chroma pair -> (2^23 + byte) as fp32 bits
// (selector 0x7540: byte 0 = U, 0x7541: byte 1 = V).
__device__ __forceinline__ float uvf(uint32_t pair, uint32_t sel) {
  return __int_as_float(__byte_perm(pair, 0x4B000000u, sel));
}

// clamp to [0, 255] in one VIMNMX.RELU: non-negative fp32 bit patterns order
// like int32 and negative ones (incl. -0.0) are negative ints -> +0.0.
__device__ __forceinline__ float clamp255(float v) {
  return __int_as_float(__vimin_s32_relu(__float_as_int(v), 0x437F0000));
}

// R16 for a pair of values already in [0, 255] (RGB lerps are convex
// combinations of bytes; NV12 values are clamped first): floor(v + 0.5) as
// the low byte of the fp32 bits of RD(fp32(v + 0.5) + 2^23) — packed, no
// float->int conversion (v + 0.5 rounded in fp32, as the R16 decision is).
__device__ __forceinline__ float2 u8_round2(float2 v) {
  return __fadd2_rd(__fadd2_rn(v, make_float2(0.5f, 0.5f)), make_float2(8388608.0f, 8388608.0f));
}

// floor(v) of values already offset by +0.5 (see kHalf in consume_tile)
__device__ __forceinline__ float2 u8_floor2(float2 v) {
  return __fadd2_rd(v, make_float2(8388608.0f, 8388608.0f));
}

__device__ __forceinline__ int tiles_total(const GatherArgs& A, const int* cnt) {
  int T = 0;
  for (int q = 0; q < A.k; q++) T += min(cnt[q], A.cap[q]) * A.tpw[q];
  return T;
}

constexpr int kPrepThreads = 256;

__global__ void __launch_bounds__(kPrepThreads) gather_prep_kernel(GatherArgs A, const mp_window* __restrict__ win,
                                                                   const int* __restrict__ frame_off,
                                                                   int* __restrict__ ws_cnt, int* __restrict__ ws_list,
                                                                   int2* __restrict__ ws_tap, int n_taps,
                                                                   int* __restrict__ d_status) {
  __shared__ int cnt[kMaxClasses];
  if (threadIdx.x < kMaxClasses) cnt[threadIdx.x] = 0;
  __syncthreads();
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gstride = gridDim.x * blockDim.x;
  // tap tables: entry e -> (class, axis, d); x taps of class q at xtab_off[q], y taps at ytab_off[q]
  for (int e = gtid; e < n_taps; e += gstride) {
    int q = 0;
    while (q + 1 < A.k && e >= A.xtab_off[q + 1]) q++;
    const bool xaxis = e < A.ytab_off[q];
    const int d = xaxis ? e - A.xtab_off[q] : e - A.ytab_off[q];
    int i0;
    float lam;
    if (xaxis) tap(A.w[q], A.ow[q], d, i0, lam);
    else tap(A.h[q], A.oh[q], d, i0, lam);
    ws_tap[e] = make_int2(i0, __float_as_int(lam));
  }
  // a plan that overflowed its window buffer reports the true total in
  // frame_off[F]; only the max_windows records in the buffer exist
  const int n_all = frame_off[A.F];
  const int n_win = min(n_all, A.max_windows);
  if (gtid == 0 && n_all > A.max_windows) set_status(d_status, MP_ERR_CAPACITY);
  for (int i = gtid; i < n_win; i += gstride) {
    const mp_window w = win[i];
    const int q = w.size_idx;
    if (q < 0 || q >= A.k || w.frame < 0 || w.frame >= A.F || w.w != A.w[q] || w.h != A.h[q] || w.x < 0 ||
        w.y < 0 || w.x + w.w > A.W || w.y + w.h > A.H || w.slot < 0) {
      set_status(d_status, MP_ERR_INVALID);
      continue;
    }
    atomicAdd(&cnt[q], 1);
    if (w.slot >= A.cap[q]) {
      set_status(d_status, MP_ERR_CAPACITY);
      continue;
    }
    ws_list[A.list_off[q] + w.slot] = i;
  }
  __syncthreads();
  if (threadIdx.x < A.k && cnt[threadIdx.x]) atomicAdd(&ws_cnt[threadIdx.x], cnt[threadIdx.x]);
}

// Consumer: warp `wid` owns output rows [wid*R, (wid+1)*R) of the tile
// (R = ceil(rows / kCW)); lane owns output columns lane + 32*j, j < NCOL
// (consecutive lanes = consecutive columns: conflict-free byte loads from the
// staged box, 128-B coalesced stores; pairs of columns share one packed f32x2
// datapath).  Separable evaluation in source-row order: each staged source row
// is lerped horizontally once (ping-pong register sets) and an output row is
// emitted as soon as its lower source row is ready.  The right/bottom taps
// are always +1 pixel / +1 row: where R15 clamps (i0 = in-1) lambda is 0, so
// the extra (finite) staged byte has no effect.
extern __shared__ __align__(128) unsigned char smem[];

// Experiment knobs (MP_GATHER_BUDGET_KB, _TILE, _WAIT, _STAGES, _DEBUG) are
// read from the environment only in builds with -DMP_EXPERIMENT_KNOBS (the
// dev sweeps of scripts/time_gather.py); the production library ignores them.
static std::atomic<int> g_sm_reserve{0};   // mp_gather_set_sm_reserve

extern "C" mp_status mp_gather_set_sm_reserve(int32_t sms) {
  if (sms < 0 || sms > 1024) return MP_ERR_INVALID;
  g_sm_reserve.store(sms, std::memory_order_relaxed);
  return MP_OK;
}

static inline const char* knob(const char* name) {
#ifdef MP_EXPERIMENT_KNOBS
  return getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

template <int FMT, int NCOL, int SRC>
__device__ __forceinline__ void consume_tile(const GatherArgs& A, const TileHdr* hdr, unsigned int soff, int wid,
                                             int lane) {
  constexpr int kCW = cw_of(FMT, SRC);
  constexpr int NP = NCOL / 2;
  const int2* xt = reinterpret_cast<const int2*>(&smem[soff + kHdrBytes]);
  const int2* yt = reinterpret_cast<const int2*>(&smem[soff + kHdrBytes + kXtapBytes]) + hdr->ys;
  const unsigned int doff = soff + kDataOff;
  const int q = hdr->k, rows = hdr->rows, cols = hdr->cols;
  const int x0 = (SRC == kSrcNV12 ? hdr->x : 3 * hdr->x) - hdr->b0, r_lo = hdr->r_lo;
  xt += hdr->xs;
  const unsigned int stride = (unsigned int)hdr->stride;
  const int R = (rows + kCW - 1) / kCW;
  const int rb0 = wid * R, rb1 = min(rows, rb0 + R);
  if (rb0 >= rb1 || lane >= cols) return;
  // u8 output from RGB24: the +0.5 of R16's floor(v + 0.5) is folded into the
  // horizontal lerps (m - (2^23 - 0.5) = byte + 0.5 exactly; lerps of offset
  // values are offset lerps), so the rounding below is one packed add
  constexpr bool kHalf = FMT == MP_OUT_U8_NHWC && SRC == kSrcRGB24;
  const float2 M2 = kHalf ? make_float2(8388607.5f, 8388607.5f) : make_float2(8388608.0f, 8388608.0f);
  unsigned int ba[NP], bb[NP];
  unsigned int ca[NP], cb[NP], da[NP], db[NP];   // NV12: chroma byte of the left tap, +0/+2 to the right tap
  unsigned long long lx[NP];   // (lambda of column A, lambda of column B) as one b64 pair
#pragma unroll
  for (int p = 0; p < NP; p++) {
    const int cA = lane + 64 * p, cB = cA + 32;
    const int2 xa = xt[min(cA, cols - 1)];
    const int2 xb = xt[min(cB, cols - 1)];
    if (SRC == kSrcNV12) {
      // luma column a = x + i0 at staged byte a - b0; its chroma pair (U,V) at
      // 2(a>>1) - b0 = (a - b0) - (a & 1) of the chroma box; the right tap's
      // pair is 2 bytes further iff a is odd (R23 siting)
      ba[p] = doff + x0 + xa.x;
      bb[p] = doff + x0 + xb.x;
      const unsigned int pa = (unsigned int)(hdr->x + xa.x) & 1u, pb = (unsigned int)(hdr->x + xb.x) & 1u;
      ca[p] = ba[p] + (unsigned int)A.uv_off[q] - pa;
      cb[p] = bb[p] + (unsigned int)A.uv_off[q] - pb;
      da[p] = 2u * pa;
      db[p] = 2u * pb;
    } else {
      ba[p] = doff + x0 + 3 * xa.x;
      bb[p] = doff + x0 + 3 * xb.x;
    }
    lx[p] = pk2(make_float2(__int_as_float(xa.y), __int_as_float(xb.y)));
  }
#ifdef MP_LAM_SMEM
  // the (lambda_A, lambda_B) pairs go to this warp's shared scratch and are
  // re-loaded (LDS.64 into an aligned register pair) at every use, instead of
  // being copied into an aligned pair before every FFMA2 (IMAD.MOV / MOV were
  // 12 % of the u8 kernel's instructions)
  const unsigned int lam_base = smem_u32(smem + A.lam_off) + (unsigned int)(wid * kMaxNP * 32 + lane) * 8u;
#pragma unroll
  for (int p = 0; p < NP; p++) {
    const unsigned long long v = lx[p];
    asm volatile("st.shared.b64 [%0], %1;" ::"r"(lam_base + (unsigned int)p * 256u), "l"(v) : "memory");
  }
  __syncwarp();
#define MP_LX(p) lds64(lam_base + (unsigned int)(p) * 256u)
#else
#define MP_LX(p) lx[p]
#endif
  float2 P[NP][3], N[NP][3];   // ping-pong horizontal lerps (3 channels x column pair)
#define MP_HL(H, CH, A0, B0, A1, B1)                                                           \
  {                                                                                             \
    const float2 m_ = make_float2(u8m(smem[A0]), u8m(smem[B0]));                                \
    const float2 n_ = make_float2(u8m(smem[A1]), u8m(smem[B1]));                                \
    H[p][CH] = ffma2_w(fsub2(n_, m_), MP_LX(p), fsub2(m_, M2));                                  \
  }
  // NV12 chroma: one 16-bit load per tap fetches the (U, V) pair; bytes are
  // placed into the 2^23 fp32 pattern with one byte-permute each
#define MP_HC(H, QA, QB)                                                                        \
  {                                                                                             \
    const uint32_t la_ = *reinterpret_cast<const uint16_t*>(&smem[QA]);                         \
    const uint32_t ra_ = *reinterpret_cast<const uint16_t*>(&smem[(QA) + da[p]]);                \
    const uint32_t lb_ = *reinterpret_cast<const uint16_t*>(&smem[QB]);                         \
    const uint32_t rb_ = *reinterpret_cast<const uint16_t*>(&smem[(QB) + db[p]]);                \
    const float2 mu_ = make_float2(uvf(la_, 0x7540), uvf(lb_, 0x7540));                         \
    const float2 nu_ = make_float2(uvf(ra_, 0x7540), uvf(rb_, 0x7540));                         \
    const float2 mv_ = make_float2(uvf(la_, 0x7541), uvf(lb_, 0x7541));                         \
    const float2 nv_ = make_float2(uvf(ra_, 0x7541), uvf(rb_, 0x7541));                         \
    H[p][1] = ffma2_w(fsub2(nu_, mu_), lx[p], fsub2(mu_, M2));                                   \
    H[p][2] = ffma2_w(fsub2(nv_, mv_), lx[p], fsub2(mv_, M2));                                   \
  }
  // NV12 luma only (the chroma lerps are copied from PREV: same chroma row)
#define MP_HY(O_, H, PREV)                                                                      \
  {                                                                                             \
    const unsigned int o_ = (O_);                                                               \
    _Pragma("unroll") for (int p = 0; p < NP; p++) {                                            \
      const unsigned int pa_ = ba[p] + o_, pb_ = bb[p] + o_;                                    \
      MP_HL(H, 0, pa_, pb_, pa_ + 1, pb_ + 1)                                                   \
      H[p][1] = PREV[p][1];                                                                     \
      H[p][2] = PREV[p][2];                                                                     \
    }                                                                                           \
  }
  // RGB taps, two ways (measured, c2/c3/c4 gather alone, same box):
  //  * bytes: 6 LDS.U8 + 6 IADD (2^23 + byte) per column — f32 output
  //    (word taps there: 1.36 -> 1.43 ms at c2);
  //  * words (u8 output, kWordTaps): a column's 6 tap bytes [a, a+6) lie in
  //    the three aligned words from a & ~3 (the alignment of a is the same in
  //    every staged row: rows are 16-B multiples apart); two funnel shifts
  //    align them and one PRMT per byte builds the 2^23 + byte pattern:
  //    3 LDS.32 + 2 SHF + 6 PRMT per column, half the shared-memory
  //    wavefronts of the consumer-bound u8 kernel (c2 1.105 -> 1.089 ms,
  //    c3 4.93 -> 4.87, c4 3.13 -> 3.09).
#ifdef MP_WORD_TAPS
  constexpr bool kWordTaps = SRC == kSrcRGB24;
#else
  constexpr bool kWordTaps = SRC == kSrcRGB24 && FMT == MP_OUT_U8_NHWC;
#endif
  unsigned int wa[NP], wb[NP], sa[NP], sb[NP];
#pragma unroll
  for (int p = 0; p < NP; p++) {
    wa[p] = ba[p] & ~3u;
    wb[p] = bb[p] & ~3u;
    sa[p] = (ba[p] & 3u) * 8u;
    sb[p] = (bb[p] & 3u) * 8u;
  }
#define MP_W6(WB, SH, LO, HI)                                                                   \
  {                                                                                             \
    const uint32_t w0_ = *reinterpret_cast<const uint32_t*>(&smem[WB]);                         \
    const uint32_t w1_ = *reinterpret_cast<const uint32_t*>(&smem[(WB) + 4]);                   \
    const uint32_t w2_ = *reinterpret_cast<const uint32_t*>(&smem[(WB) + 8]);                   \
    LO = __funnelshift_r(w0_, w1_, SH);                                                         \
    HI = __funnelshift_r(w1_, w2_, SH);                                                         \
  }
#define MP_MB(W, K) __int_as_float(__byte_perm((W), 0x4B000000u, 0x7440u | (K)))
#define MP_HRGB(O_, H)                                                                          \
  if (kWordTaps) {                                                                              \
    _Pragma("unroll") for (int p = 0; p < NP; p++) {                                            \
      uint32_t la_, ha_, lb_, hb_;                                                              \
      MP_W6(wa[p] + (O_), sa[p], la_, ha_)                                                      \
      MP_W6(wb[p] + (O_), sb[p], lb_, hb_)                                                      \
      {                                                                                         \
        const float2 m_ = make_float2(MP_MB(la_, 0), MP_MB(lb_, 0));                            \
        const float2 n_ = make_float2(MP_MB(la_, 3), MP_MB(lb_, 3));                            \
        H[p][0] = ffma2_w(fsub2(n_, m_), MP_LX(p), fsub2(m_, M2));                              \
      }                                                                                         \
      {                                                                                         \
        const float2 m_ = make_float2(MP_MB(la_, 1), MP_MB(lb_, 1));                            \
        const float2 n_ = make_float2(MP_MB(ha_, 0), MP_MB(hb_, 0));                            \
        H[p][1] = ffma2_w(fsub2(n_, m_), MP_LX(p), fsub2(m_, M2));                              \
      }                                                                                         \
      {                                                                                         \
        const float2 m_ = make_float2(MP_MB(la_, 2), MP_MB(lb_, 2));                            \
        const float2 n_ = make_float2(MP_MB(ha_, 1), MP_MB(hb_, 1));                            \
        H[p][2] = ffma2_w(fsub2(n_, m_), MP_LX(p), fsub2(m_, M2));                              \
      }                                                                                         \
    }                                                                                           \
  } else {                                                                                      \
    _Pragma("unroll") for (int p = 0; p < NP; p++) {                                            \
      const unsigned int pa_ = ba[p] + (O_), pb_ = bb[p] + (O_);                                \
      _Pragma("unroll") for (int ch = 0; ch < 3; ch++)                                          \
          MP_HL(H, ch, pa_ + ch, pb_ + ch, pa_ + 3 + ch, pb_ + 3 + ch)                          \
    }                                                                                           \
  }
  // horizontal lerps of one staged source row: luma/RGB row at byte offset
  // O_, its chroma row (NV12) at OC_ (both relative to the staged boxes)
#define MP_H(O_, OC_, H)                                                                        \
  {                                                                                             \
    const unsigned int o_ = (O_);                                                               \
    if (SRC == kSrcNV12) {                                                                      \
      const unsigned int oc_ = (OC_);                                                           \
      _Pragma("unroll") for (int p = 0; p < NP; p++) {                                          \
        const unsigned int pa_ = ba[p] + o_, pb_ = bb[p] + o_;                                  \
        MP_HL(H, 0, pa_, pb_, pa_ + 1, pb_ + 1)                                                 \
        MP_HC(H, ca[p] + oc_, cb[p] + oc_)                                                      \
      }                                                                                         \
    } else {                                                                                    \
      MP_HRGB(o_, H)                                                                            \
    }                                                                                           \
  }
  // dense staging: source row r of the box (rows r_lo..); its chroma row is
  // ((ya + r) >> 1) - (ya >> 1) of the chroma box (ya = first staged luma row)
  const int ya = hdr->ya;
#define MP_HD(ROW, H) \
  MP_H((unsigned int)(ROW) * stride, (unsigned int)(((ya + (ROW)) >> 1) - (ya >> 1)) * stride, H)
  // row ROW after row ROW-1 (held in PREV): NV12 rows with odd ya + ROW share
  // their chroma row with the previous one -> only the luma is lerped
#define MP_HD2(ROW, H, PREV)                                                                    \
  if (SRC == kSrcNV12 && ((ya + (ROW)) & 1)) {                                                  \
    MP_HY((unsigned int)(ROW) * stride, H, PREV)                                                \
  } else {                                                                                      \
    MP_HD(ROW, H)                                                                               \
  }
  // vertical lerp of column pair p -> v0, v1, v2 (RGB); NV12: the lerped
  // Y, U, V are converted to R'G'B' and clamped to [0, 255] (R23)
  const float2 CY = make_float2(A.cvt[0], A.cvt[0]), CYO = make_float2(A.cvt[1], A.cvt[1]);
  const float2 CRV = make_float2(A.cvt[2], A.cvt[2]), CGU = make_float2(A.cvt[3], A.cvt[3]);
  const float2 CGV = make_float2(A.cvt[4], A.cvt[4]), CBU = make_float2(A.cvt[5], A.cvt[5]);
  const float2 C128 = make_float2(-128.0f, -128.0f);
#define MP_V(T, B)                                                                              \
  float2 v0 = __ffma2_rn(ly, fsub2(B[p][0], T[p][0]), T[p][0]);                                  \
  float2 v1 = __ffma2_rn(ly, fsub2(B[p][1], T[p][1]), T[p][1]);                                  \
  float2 v2 = __ffma2_rn(ly, fsub2(B[p][2], T[p][2]), T[p][2]);                                  \
  if (SRC == kSrcNV12) {                                                                        \
    const float2 yy_ = __ffma2_rn(CY, v0, CYO);                                                 \
    const float2 uu_ = __fadd2_rn(v1, C128), vv_ = __fadd2_rn(v2, C128);                         \
    v0 = __ffma2_rn(CRV, vv_, yy_);                                                             \
    v1 = __ffma2_rn(CGU, uu_, __ffma2_rn(CGV, vv_, yy_));                                       \
    v2 = __ffma2_rn(CBU, uu_, yy_);                                                             \
    v0 = make_float2(clamp255(v0.x), clamp255(v0.y));                                           \
    v1 = make_float2(clamp255(v1.x), clamp255(v1.y));                                           \
    v2 = make_float2(clamp255(v2.x), clamp255(v2.y));                                           \
  }
  const int ow = A.ow[q], oh = A.oh[q];
  const bool sparse = A.sparse[q] != 0;
  const unsigned int pair = (unsigned int)A.pair_bytes[q];
  const int wy = hdr->wy;
  bool ok[NCOL];
#pragma unroll
  for (int j = 0; j < NCOL; j++) ok[j] = lane + 32 * j < cols;
  // one output row from top/bottom horizontal lerps T, B with weight y.y
  if (FMT == MP_OUT_F32_NCHW) {
    const size_t plane = (size_t)oh * ow;
    float* o0 = reinterpret_cast<float*>(A.out[q]) + (size_t)hdr->slot * 3 * plane +
                (size_t)(hdr->oy0 + rb0) * ow + hdr->ox0 + lane;
    float* o1 = o0 + plane;
    float* o2 = o1 + plane;
#define MP_ROW(T, B)                                                                            \
  {                                                                                             \
    const float2 ly = make_float2(__int_as_float(y.y), __int_as_float(y.y));                    \
    _Pragma("unroll") for (int p = 0; p < NP; p++) {                                            \
      MP_V(T, B)                                                                                \
      if (ok[2 * p]) {                                                                          \
        __stcs(o0 + 64 * p, v0.x);                                                              \
        __stcs(o1 + 64 * p, v1.x);                                                              \
        __stcs(o2 + 64 * p, v2.x);                                                              \
      }                                                                                         \
      if (ok[2 * p + 1]) {                                                                      \
        __stcs(o0 + 64 * p + 32, v0.y);                                                         \
        __stcs(o1 + 64 * p + 32, v1.y);                                                         \
        __stcs(o2 + 64 * p + 32, v2.y);                                                         \
      }                                                                                         \
    }                                                                                           \
    o0 += ow;                                                                                   \
    o1 += ow;                                                                                   \
    o2 += ow;                                                                                   \
  }
#include "mp_gather_rows.inc"
#undef MP_ROW
  } else {
    uint8_t* o = reinterpret_cast<uint8_t*>(A.out[q]) +
                 (((size_t)hdr->slot * oh + hdr->oy0 + rb0) * ow + hdr->ox0 + lane) * 3;
#define MP_ROW(T, B)                                                                            \
  {                                                                                             \
    const float2 ly = make_float2(__int_as_float(y.y), __int_as_float(y.y));                    \
    _Pragma("unroll") for (int p = 0; p < NP; p++) {                                            \
      MP_V(T, B)                                                                                \
      const float2 r0 = kHalf ? u8_floor2(v0) : u8_round2(v0);                                  \
      const float2 r1 = kHalf ? u8_floor2(v1) : u8_round2(v1);                                  \
      const float2 r2 = kHalf ? u8_floor2(v2) : u8_round2(v2);                                  \
      if (ok[2 * p]) {                                                                          \
        o[192 * p + 0] = (uint8_t)__float_as_uint(r0.x);                                        \
        o[192 * p + 1] = (uint8_t)__float_as_uint(r1.x);                                        \
        o[192 * p + 2] = (uint8_t)__float_as_uint(r2.x);                                        \
      }                                                                                         \
      if (ok[2 * p + 1]) {                                                                      \
        o[192 * p + 96 + 0] = (uint8_t)__float_as_uint(r0.y);                                   \
        o[192 * p + 96 + 1] = (uint8_t)__float_as_uint(r1.y);                                   \
        o[192 * p + 96 + 2] = (uint8_t)__float_as_uint(r2.y);                                   \
      }                                                                                         \
    }                                                                                           \
    o += (size_t)ow * 3;                                                                        \
  }
#include "mp_gather_rows.inc"
#undef MP_ROW
  }
#undef MP_V
#undef MP_HD2
#undef MP_HD
#undef MP_H
#undef MP_HY
#undef MP_HC
#undef MP_HL
#undef MP_HRGB
#undef MP_W6
#undef MP_MB
#undef MP_LX
}

// ---------------------------------------------------------------------------
// u8 NHWC output from RGB24 frames at any scale (round 2b; the exact 4:3
// classes of windows on the 16-px grid take consume_tile_r43 below).
//
// The u8 gather is bound by its consumer, not by HBM: the
// generic consume_tile spent ~50 warp instructions per output pixel, a
// quarter of them register copies of per-column weight PAIRS into the
// aligned pair an FFMA2 reads.  This consumer (657 M instead of 774 M warp
// instructions at c2; gather alone 1.091 -> 1.059 ms) pairs values
// that share one weight instead, so every horizontal FFMA2 but one per
// column pair takes its lambda as a broadcast scalar (SASS `R.F32`, no
// copy), and carries the bytes with a bias that needs no unbiasing:
//
//  * a byte b is placed in bits 8..15 of 1.0f (one PRMT): 1 + b * 2^-15,
//    exact.  Lerps of biased values are biased lerps (the weights sum to 1),
//    so h = m + lambda (n - m) is one FADD2 + one FFMA2 per value pair (the
//    generic path also subtracts 2^23);
//  * R16's floor(v + 0.5) of a value held as 1 + v 2^-15 is the low byte of
//    RD(that + (255 + 2^-16)) = 256 + (v + 0.5) 2^-15 on the 2^-15 grid of
//    [256, 512): one packed add; STG.U8 stores the low byte.
//  * precision: every rounding is on the 2^-23 grid of [1, 2), i.e. 2^-9 of
//    an output LSB (generic path: 2^-17).  Four roundings bound the error by
//    ~0.004 LSB, far inside the 1-LSB bar; an output differs from the exact
//    rounding only where v + 0.5 lies within that of an integer.
//
// Value pairs per column pair (A = lane + 64 p, B = A + 32) and staged row:
// (R, G) of A and (R, G) of B with their own scalar lambda, (B_A, B_B) with
// the (lambda_A, lambda_B) pair; the vertical lerp takes the row weight as a
// broadcast scalar for all three.
__device__ __forceinline__ float2 ffma2_s(float2 a, float s, float2 c) {   // a * (s, s) + c
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(make_float2(s, s))), "l"(pk2(c)));
  return upk2(r);
}
// Bounds-checked dev builds (-DMP_BOUNDS_CHECK; the GPU suite runs through
// one — the pool's compute-sanitizer is closed): every shared-memory access
// of the round-2b consumers stays inside its stage's staged box / its warp's
// row buffer, and every global store inside its class's output tensor;
// a violation prints and traps.
#ifdef MP_BOUNDS_CHECK
__device__ __noinline__ void mp_bounds_fail(const char* what, long long a, long long lo, long long hi) {
  printf("MP_BOUNDS_CHECK %s: [%lld] not in [%lld, %lld) block %d thread %d\n", what, a, lo, hi, (int)blockIdx.x,
         (int)threadIdx.x);
  __trap();
}
#define MP_BCHK(WHAT, A_, N_, LO_, HI_)                                                         \
  {                                                                                             \
    const long long a__ = (long long)(A_), lo__ = (long long)(LO_), hi__ = (long long)(HI_);    \
    if ((long long)(N_) > 0 && (a__ < lo__ || a__ + (long long)(N_) > hi__))                    \
      mp_bounds_fail(WHAT, a__, lo__, hi__);                                                    \
  }
#else
#define MP_BCHK(WHAT, A_, N_, LO_, HI_) {}   /* a statement: "if (c) MP_BCHK(...)" stays an if */
#endif
// output tensor of class q in bytes (fmt: u8 NHWC or f32 NCHW)
__device__ __forceinline__ long long out_bytes(const GatherArgs& A, int q) {
  return (long long)A.cap[q] * A.oh[q] * A.ow[q] * (A.fmt == MP_OUT_U8_NHWC ? 3 : 12);
}

// byte K of W -> 1 + byte * 2^-15 (bits 8..15 of 1.0f = 0x3F800000)
#define MP_B1(W, K) __int_as_float(__byte_perm((W), 0x3F800000u, 0x7604u | ((K) << 4)))

// lane pixels A (column lane + 64 p) and B (+ 32): three bytes each
#define MP_U8_STORE(o, p, u0, u1, u2)                                                             \
  if (ok[2 * p]) {                                                                                \
    o[192 * p + 0] = (uint8_t)__float_as_uint(u0.x);                                              \
    o[192 * p + 1] = (uint8_t)__float_as_uint(u0.y);                                              \
    o[192 * p + 2] = (uint8_t)__float_as_uint(u2.x);                                              \
  }                                                                                               \
  if (ok[2 * p + 1]) {                                                                            \
    o[192 * p + 96 + 0] = (uint8_t)__float_as_uint(u1.x);                                         \
    o[192 * p + 96 + 1] = (uint8_t)__float_as_uint(u1.y);                                         \
    o[192 * p + 96 + 2] = (uint8_t)__float_as_uint(u2.y);                                         \
  }
template <int NCOL>
__device__ __forceinline__ void consume_tile_u8rgb(const GatherArgs& A, const TileHdr* hdr, unsigned int soff,
                                                   int wid, int lane) {
  constexpr int kCW = cw_of(MP_OUT_U8_NHWC, kSrcRGB24);
  constexpr int SRC = kSrcRGB24;
  constexpr int NP = NCOL / 2;
  const int2* xt = reinterpret_cast<const int2*>(&smem[soff + kHdrBytes]) + hdr->xs;
  const int2* yt = reinterpret_cast<const int2*>(&smem[soff + kHdrBytes + kXtapBytes]) + hdr->ys;
  const unsigned int doff = soff + kDataOff;
  const int q = hdr->k, rows = hdr->rows, cols = hdr->cols;
  const int x0 = 3 * hdr->x - hdr->b0, r_lo = hdr->r_lo;
  const unsigned int stride = (unsigned int)hdr->stride;
  const int R = (rows + kCW - 1) / kCW;
  const int rb0 = wid * R, rb1 = min(rows, rb0 + R);
  if (rb0 >= rb1 || lane >= cols) return;
  // a column's 6 tap bytes [a, a+6) lie in the three aligned words from
  // a & ~3 (rows are 16-B multiples apart: the same alignment in every row)
  unsigned int wa[NP], wb[NP], sa[NP], sb[NP];
  unsigned long long lp[NP];   // (lambda_A, lambda_B): the scalars are read from the pair's halves
#pragma unroll
  for (int p = 0; p < NP; p++) {
    const int cA = lane + 64 * p, cB = cA + 32;
    const int2 xa = xt[min(cA, cols - 1)];
    const int2 xb = xt[min(cB, cols - 1)];
    const unsigned int ba = doff + x0 + 3 * xa.x, bb = doff + x0 + 3 * xb.x;
    wa[p] = ba & ~3u;
    wb[p] = bb & ~3u;
    sa[p] = (ba & 3u) * 8u;
    sb[p] = (bb & 3u) * 8u;
    lp[p] = pk2(make_float2(__int_as_float(xa.y), __int_as_float(xb.y)));
  }
  float2 P[NP][3], N[NP][3];   // [0] (R, G) of A, [1] (R, G) of B, [2] (B of A, B of B)
#define MP_W6(WB, SH, LO, HI)                                                                   \
  {                                                                                             \
    MP_BCHK("u8rgb lds", WB, 12, doff, soff + A.stage_bytes)                                    \
    const uint32_t w0_ = *reinterpret_cast<const uint32_t*>(&smem[WB]);                         \
    const uint32_t w1_ = *reinterpret_cast<const uint32_t*>(&smem[(WB) + 4]);                   \
    const uint32_t w2_ = *reinterpret_cast<const uint32_t*>(&smem[(WB) + 8]);                   \
    LO = __funnelshift_r(w0_, w1_, SH);                                                         \
    HI = __funnelshift_r(w1_, w2_, SH);                                                         \
  }
  // horizontal lerps of the staged row at byte offset O_ (LO = R0 G0 B0 R1, HI = G1 B1 . .)
#define MP_H(O_, OC_, H)                                                                        \
  {                                                                                             \
    const unsigned int o_ = (O_);                                                               \
    _Pragma("unroll") for (int p = 0; p < NP; p++) {                                            \
      uint32_t l0_, h0_, l1_, h1_;                                                              \
      MP_W6(wa[p] + o_, sa[p], l0_, h0_)                                                        \
      MP_W6(wb[p] + o_, sb[p], l1_, h1_)                                                        \
      {                                                                                         \
        const float2 m_ = make_float2(MP_B1(l0_, 0), MP_B1(l0_, 1));                            \
        const float2 n_ = make_float2(MP_B1(l0_, 3), MP_B1(h0_, 0));                            \
        H[p][0] = ffma2_s(fsub2(n_, m_), upk2(lp[p]).x, m_);                                            \
      }                                                                                         \
      {                                                                                         \
        const float2 m_ = make_float2(MP_B1(l1_, 0), MP_B1(l1_, 1));                            \
        const float2 n_ = make_float2(MP_B1(l1_, 3), MP_B1(h1_, 0));                            \
        H[p][1] = ffma2_s(fsub2(n_, m_), upk2(lp[p]).y, m_);                                            \
      }                                                                                         \
      {                                                                                         \
        const float2 m_ = make_float2(MP_B1(l0_, 2), MP_B1(l1_, 2));                            \
        const float2 n_ = make_float2(MP_B1(h0_, 1), MP_B1(h1_, 1));                            \
        H[p][2] = ffma2_w(fsub2(n_, m_), lp[p], m_);                                            \
      }                                                                                         \
    }                                                                                           \
  }
#define MP_HD(ROW, H) MP_H((unsigned int)(ROW) * stride, 0u, H)
#define MP_HD2(ROW, H, PREV) MP_HD(ROW, H)
#define MP_HY(O_, H, PREV) {}
  const int ow = A.ow[q], oh = A.oh[q];
  const bool sparse = A.sparse[q] != 0;
  const unsigned int pair = (unsigned int)A.pair_bytes[q];
  const int wy = hdr->wy;
  (void)wy;
  (void)oh;
  bool ok[NCOL];
#pragma unroll
  for (int j = 0; j < NCOL; j++) ok[j] = lane + 32 * j < cols;
  uint8_t* o = reinterpret_cast<uint8_t*>(A.out[q]) +
               (((size_t)hdr->slot * A.oh[q] + hdr->oy0 + rb0) * ow + hdr->ox0) * 3;
  constexpr float kRnd = 255.0f + 1.52587890625e-05f;   // 255 + 2^-16 (exact in fp32)
  // one output row from the horizontal lerps T (top tap row) and B (bottom)
#define MP_U8V(T, B)                                                                            \
  const float2 u0 = __fadd2_rd(ffma2_s(fsub2(B[p][0], T[p][0]), ly, T[p][0]), make_float2(kRnd, kRnd)); \
  const float2 u1 = __fadd2_rd(ffma2_s(fsub2(B[p][1], T[p][1]), ly, T[p][1]), make_float2(kRnd, kRnd)); \
  const float2 u2 = __fadd2_rd(ffma2_s(fsub2(B[p][2], T[p][2]), ly, T[p][2]), make_float2(kRnd, kRnd));
#define MP_ROW(T, B)                                                                            \
  {                                                                                             \
    const float ly = __int_as_float(y.y);                                                       \
    uint8_t* const ol_ = o + 3 * lane;                                                          \
    _Pragma("unroll") for (int p = 0; p < NP; p++) {                                            \
      MP_U8V(T, B)                                                                              \
      MP_BCHK("u8rgb stg", ol_ + 192 * p - (uint8_t*)A.out[q], ok[2 * p + 1] ? 99 : (ok[2 * p] ? 3 : 0), 0, out_bytes(A, q)) \
      MP_U8_STORE(ol_, p, u0, u1, u2)                                                           \
    }                                                                                           \
    o += (size_t)ow * 3;                                                                        \
  }
  // downscale, dense staging: i0 strictly increases with the output row
  // (consecutive n differ by 2 in >= 2 out), so a staged row is the top tap
  // of at most one output row and the last output row ends the loop.  One
  // fixed body per staged row keeps P / N in place (no register rotation at
  // the back edge, unlike the generic multi-row loop).
#define MP_DOWN_LOOP                                                                            \
  {                                                                                             \
    int orow = rb0;                                                                             \
    int2 y = yt[orow];                                                                          \
    y.x -= r_lo;                                                                                \
    int r = y.x;                                                                                \
    unsigned int ro = (unsigned int)r * stride; /* byte offset of staged row r */               \
    MP_H(ro, 0u, P)                                                                             \
    for (;;) {                                                                                  \
      ro += stride;                                                                             \
      MP_H(ro, 0u, N)                                                                           \
      if (y.x == r) {                                                                           \
        MP_ROW(P, N)                                                                            \
        if (++orow >= rb1) break;                                                               \
        y = yt[orow];                                                                           \
        y.x -= r_lo;                                                                            \
      }                                                                                         \
      r++;                                                                                      \
      ro += stride;                                                                             \
      MP_H(ro, 0u, P)                                                                           \
      if (y.x == r) {                                                                           \
        MP_ROW(N, P)                                                                            \
        if (++orow >= rb1) break;                                                               \
        y = yt[orow];                                                                           \
        y.x -= r_lo;                                                                            \
      }                                                                                         \
      r++;                                                                                      \
    }                                                                                           \
  }
  if (!sparse && A.h[q] >= oh) {
    MP_DOWN_LOOP
  } else {
#include "mp_gather_rows.inc"
  }
#undef MP_DOWN_LOOP
#undef MP_ROW
#undef MP_U8V
#undef MP_HY
#undef MP_HD2
#undef MP_HD
#undef MP_H
#undef MP_W6
}

// ---------------------------------------------------------------------------
// u8 NHWC from RGB24 at an exact 4:3 downscale on both axes: a fixed-tap
// consumer (every BASELINE size class is 4:3: 256 -> 192, 512 -> 384,
// 128 -> 96 and the full-frame 1920x1080 -> 1440x810, 3840x2160 ->
// 2880x1620, 960x540 -> 720x405).
//
// R15 for in = 4u, out = 3u and output d = 3k + j (j = 0, 1, 2):
// n = (2d + 1) 4u - 3u, so n / 2out = 4k + (8j + 1) / 6: i0 = 4k + j and
// lambda = fp32((n mod 2out) / 2out) = fp32(u {1, 3, 5}[j] / 6u) = fp32(1/6),
// fp32(1/2), fp32(5/6) (the generic tap table holds exactly these: one
// correctly rounded division of exact integers), and i0 + 1 <= 4k + 3 <= in - 1
// (no clamp).  So output columns 3k..3k+2 read exactly source pixels
// 4k..4k+3, output rows 3m..3m+2 exactly source rows 4m..4m+3, with three
// fixed weights — no tap tables, no halo rows.
//
// Why a consumer of its own: the u8 gather is bound by the SM's LSU issue
// rate (~1.8 cycles per shared/global memory instruction per SM, B300
// microarch notes).  The per-column consumer issued 3 LDS.32 per column per
// staged row and 3 STG.U8 per pixel: ~7.4 LSU instructions per output pixel
// = 0.73 ms of LSU issue on c2 for a 0.62-ms HBM floor.  Here a task of 12
// output columns x 3 output rows reads its 48-byte source runs (16 pixels x 4
// rows, 16-B aligned when the window x is a multiple of 16 — always, for
// windows on the 32-px proxy grid) with 3 LDS.128 per row and writes 36-byte
// output rows with 9 STG.32: ~1.1 LSU instructions per pixel.  Each source
// byte is converted once (48 PRMT per row: 1 + b 2^-15, see consume_tile_u8rgb)
// and every lerp takes its weight as an immediate broadcast.
constexpr float kR43L0 = 1.0f / 6.0f, kR43L1 = 0.5f, kR43L2 = 5.0f / 6.0f;
constexpr int kR43Buf = 32 * 36;   // one warp output row: 32 tasks x 12 pixels x 3 bytes
constexpr int kR43BufBytes = MP_KCW_U8 * kR43Buf;   // one row buffer per u8 consumer warp
constexpr int kR43FBuf = 32 * 48;  // one warp plane row (f32): 32 tasks x 12 floats
constexpr int kR43FBufBytes = MP_KCW * kR43FBuf;   // one plane-row buffer per f32 consumer warp

// horizontal lerps of one 48-byte source run at shared byte address A_:
// H[j][c][kp] = (value of column 3(2kp) + j, column 3(2kp+1) + j), channel c
#define MP_R43_LD(A_, Q)                                                                        \
  MP_BCHK("r43 lds", A_, 48, soff + kDataOff, soff + A.stage_bytes)                              \
  uint4 Q[3];                                                                                   \
  Q[0] = *reinterpret_cast<const uint4*>(&smem[(A_)]);                                          \
  Q[1] = *reinterpret_cast<const uint4*>(&smem[(A_) + 16]);                                     \
  Q[2] = *reinterpret_cast<const uint4*>(&smem[(A_) + 32]);
#define MP_R43_H(A_, H)                                                                         \
  {                                                                                             \
    MP_R43_LD(A_, q_)                                                                           \
    const uint32_t w_[12] = {q_[0].x, q_[0].y, q_[0].z, q_[0].w, q_[1].x, q_[1].y, q_[1].z, q_[1].w, \
                             q_[2].x, q_[2].y, q_[2].z, q_[2].w};                               \
    _Pragma("unroll") for (int j = 0; j < 3; j++) {                                             \
      const float lam_ = j == 0 ? kR43L0 : (j == 1 ? kR43L1 : kR43L2);                          \
      _Pragma("unroll") for (int c = 0; c < 3; c++) {                                           \
        _Pragma("unroll") for (int kp = 0; kp < 2; kp++) {                                      \
          const int i_ = 24 * kp + 3 * j + c; /* byte of the left tap, column 3(2kp) + j */     \
          const float2 m_ = make_float2(MP_B1(w_[i_ >> 2], i_ & 3), MP_B1(w_[(i_ + 12) >> 2], (i_ + 12) & 3)); \
          const float2 n_ = make_float2(MP_B1(w_[(i_ + 3) >> 2], (i_ + 3) & 3),                 \
                                        MP_B1(w_[(i_ + 15) >> 2], (i_ + 15) & 3));              \
          /* lambda = 1/2 (j = 1): the unscaled sum m + n (exact); the 1/2 is  \
             applied in the rounding of MP_R43_ROW (a power of two: exact) */   \
          H[j][c][kp] = j == 1 ? __fadd2_rn(m_, n_) : ffma2_s(fsub2(n_, m_), lam_, m_);         \
        }                                                                                       \
      }                                                                                         \
    }                                                                                           \
  }
// one output row (12 pixels, 36 bytes) from tap rows T, B with weight LY:
// R16 rounding as in consume_tile_u8rgb, bytes packed 4 per word into this
// lane's 36-byte slot of the warp's row buffer at shared byte address BUF_
// HALF: the row weight is 1/2 (output row 3m + 1) — V = T + B, the 1/2
// joins the j = 1 columns' 1/2 in the rounding's exact power-of-two scale
#define MP_R43_ROW(T, B, LY, HALF, BUF_)                                                        \
  {                                                                                             \
    constexpr float kRnd_ = 255.0f + 1.52587890625e-05f;                                        \
    float2 u_[3][3][2];                                                                         \
    _Pragma("unroll") for (int j = 0; j < 3; j++)                                               \
      _Pragma("unroll") for (int c = 0; c < 3; c++)                                             \
        _Pragma("unroll") for (int kp = 0; kp < 2; kp++)                                        \
        {                                                                                       \
          const float sc_ = (j == 1 ? 0.5f : 1.0f) * ((HALF) ? 0.5f : 1.0f);                    \
          const float2 v_ = (HALF) ? __fadd2_rn(T[j][c][kp], B[j][c][kp])                       \
                                   : ffma2_s(fsub2(B[j][c][kp], T[j][c][kp]), (LY), T[j][c][kp]); \
          u_[j][c][kp] = __ffma2_rd(v_, make_float2(sc_, sc_), make_float2(kRnd_, kRnd_));      \
        }                                                                                       \
    _Pragma("unroll") for (int wi = 0; wi < 9; wi++) {                                          \
      uint32_t b_[4];                                                                           \
      _Pragma("unroll") for (int e = 0; e < 4; e++) {                                           \
        const int bi = 4 * wi + e, k = bi / 9, j = (bi % 9) / 3, c = bi % 3;                    \
        b_[e] = __float_as_uint((k & 1) ? u_[j][c][k >> 1].y : u_[j][c][k >> 1].x);             \
      }                                                                                         \
      const uint32_t lo_ = __byte_perm(b_[0], b_[1], 0x0040u), hi_ = __byte_perm(b_[2], b_[3], 0x0040u); \
      MP_BCHK("r43 sts", (BUF_) + 4 * wi, 4, buf0, buf0 + kR43Buf)                               \
      *reinterpret_cast<uint32_t*>(&smem[(BUF_) + 4 * wi]) = __byte_perm(lo_, hi_, 0x5410u);    \
    }                                                                                           \
  }

// ctid: consumer thread 0 .. kCW*32-1.  Tasks (row group rg of 3 output rows,
// column group cg of 12 output columns), t = rg * ncg + cg; warp w of pass
// p takes tasks 256 p + 32 w + lane.  ncg divides 32 and is a multiple of 4
// (host), so a warp's 32 tasks are 32/ncg whole row groups: per output row
// its 32 x 36 = 1152 bytes are 32/ncg tile-wide runs of ncg x 36 bytes
// (16-B multiples, 16-B aligned in the output).  The lanes pack their bytes
// into the warp's row buffer (9 STS.32, conflict-free: lane stride 9 words)
// and the warp writes the runs as 72 16-B chunks (LDS.128 + STG.128): every
// 32-B sector is written once, whole.  (Each lane storing its 36 bytes with
// 9 STG.32 directly measured 1.58 ms at c2: 287 M partial L2 sector writes.)
__device__ __forceinline__ void consume_tile_r43(const GatherArgs& A, const TileHdr* hdr, unsigned int soff,
                                                 int wid, int lane) {
  constexpr int kCW = cw_of(MP_OUT_U8_NHWC, kSrcRGB24);
  const int2* xt = reinterpret_cast<const int2*>(&smem[soff + kHdrBytes]) + hdr->xs;
  const int q = hdr->k, rows = hdr->rows, cols = hdr->cols;
  const int ncg = cols / 12, nrg = rows / 3, ntask = ncg * nrg, lg = __ffs(ncg) - 1;
  const int ow = A.ow[q];
  const size_t row3 = (size_t)ow * 3;
  const unsigned int stride = (unsigned int)hdr->stride;
  // staged byte of the tile's first source pixel (16-B aligned, see above)
  const unsigned int a0 = soff + kDataOff + (unsigned int)(3 * hdr->x - hdr->b0 + 3 * xt[0].x);
  uint8_t* const out0 = reinterpret_cast<uint8_t*>(A.out[q]) +
                        (((size_t)hdr->slot * A.oh[q] + hdr->oy0) * ow + hdr->ox0) * 3;
  // this lane's 16-B copy-out chunks of a warp row (72 per row: lanes take
  // chunks lane, lane + 32 and, lanes < 8, lane + 64): run (row group offset
  // seg) and chunk within the run; byte offset in the output relative to the
  // warp's first row, and the run's row group for the ragged last tile
  const int cps = 9 * ncg / 4;
  size_t coff[3];
  int cseg[3];
#pragma unroll
  for (int k = 0; k < 3; k++) {
    const int c = min(lane + 32 * k, 71);
    cseg[k] = c / cps;
    coff[k] = (size_t)(3 * cseg[k]) * row3 + 16 * (c - cseg[k] * cps);
  }
  const bool third = lane < 8;   // chunk lane + 64 exists
  const unsigned int buf0 = (unsigned int)A.obuf_off + (unsigned int)wid * kR43Buf;
  const unsigned int bl = buf0 + 16u * (unsigned int)lane;
  const int rpw = 32 / ncg;   // row groups per warp
  for (int base = 32 * wid; base < ntask; base += kCW * 32) {
    const int rgw = base >> lg;                           // first row group of this warp's tasks
    const int t = min(base + lane, ntask - 1);            // lanes past the tile redo its last task
    const int rg = t >> lg, cg = t & (ncg - 1);   // ncg is 4, 8 or 16 (host)
    const unsigned int a = a0 + (unsigned int)(4 * rg) * stride + 48u * (unsigned int)cg;
    MP_BCHK("r43 box rows", 4 * rg, 4, 0, A.box_h[q])
    MP_BCHK("r43 box cols", a0 - (soff + kDataOff) + 48u * cg, 48, 0, stride)
    uint8_t* const orow = out0 + (size_t)(3 * rgw) * row3;
    const bool full = rgw + rpw <= nrg;   // every run of the warp lies in the tile (all but a ragged last tile)
    float2 X[3][3][2], Y[3][3][2];
#define MP_R43_OUT(RR, BUFI)                                                                    \
  {                                                                                             \
    __syncwarp();                                                                               \
    uint8_t* const o_ = orow + (size_t)(RR) * row3;                                             \
    const unsigned int s_ = bl + (BUFI) * kR43Buf;                                              \
    if (full) {                                                                                 \
      MP_BCHK("r43 stg", o_ + coff[0] - (uint8_t*)A.out[q], 16, 0, out_bytes(A, q))             \
      MP_BCHK("r43 stg", o_ + coff[1] - (uint8_t*)A.out[q], 16, 0, out_bytes(A, q))             \
      MP_BCHK("r43 lds.128", s_ + (third ? 1024 : 512), 16, buf0, buf0 + kR43Buf)                \
      if (third) MP_BCHK("r43 stg", o_ + coff[2] - (uint8_t*)A.out[q], 16, 0, out_bytes(A, q))  \
      __stcs(reinterpret_cast<int4*>(o_ + coff[0]), *reinterpret_cast<const int4*>(&smem[s_])); \
      __stcs(reinterpret_cast<int4*>(o_ + coff[1]), *reinterpret_cast<const int4*>(&smem[s_ + 512])); \
      if (third)                                                                                \
        __stcs(reinterpret_cast<int4*>(o_ + coff[2]), *reinterpret_cast<const int4*>(&smem[s_ + 1024])); \
    } else {                                                                                    \
      _Pragma("unroll") for (int k = 0; k < 3; k++)                                             \
        if ((k < 2 || third) && rgw + cseg[k] < nrg) {                                          \
          MP_BCHK("r43 stg", o_ + coff[k] - (uint8_t*)A.out[q], 16, 0, out_bytes(A, q))         \
          __stcs(reinterpret_cast<int4*>(o_ + coff[k]), *reinterpret_cast<const int4*>(&smem[s_ + 512 * k])); \
        }                                                                                       \
    }                                                                                           \
  }
    // one row buffer per warp (shared memory beside the 12-warp ring): a
    // __syncwarp after each copy-out orders its reads before the next row's
    // writes
    MP_R43_H(a, X)
    MP_R43_H(a + stride, Y)
    MP_R43_ROW(X, Y, kR43L0, false, buf0 + 36u * (unsigned int)lane)
    MP_R43_OUT(0, 0)
    __syncwarp();
    MP_R43_H(a + 2 * stride, X)
    MP_R43_ROW(Y, X, kR43L1, true, buf0 + 36u * (unsigned int)lane)
    MP_R43_OUT(1, 0)
    __syncwarp();
    MP_R43_H(a + 3 * stride, Y)
    MP_R43_ROW(X, Y, kR43L2, false, buf0 + 36u * (unsigned int)lane)
    MP_R43_OUT(2, 0)
    __syncwarp();
#undef MP_R43_OUT
  }
}
#undef MP_R43_H
#undef MP_R43_ROW
#undef MP_B1

// f32 NCHW from RGB24 at an exact 4:3 downscale: the same fixed-tap tasks
// (12 output columns x 3 output rows per consumer thread, LDS.128 source
// runs), f32 arithmetic on the unbiased 0-255 scale (the 1e-3 bar is tighter
// than the u8 path's 1 + b 2^-15 representation allows).  Value pairs are
// output-ADJACENT columns (2i, 2i+1) so each plane row of a task leaves as
// three 16-B stores (12 floats, 48 B) — the per-column consumer issued 6
// LDS.U8 per column per staged row and 3 STG.32 per pixel (~12 LSU
// instructions per pixel against ~1.1 here); the lambda of a pair is then a
// constant pair: (L0, L1), (L2, L0), (L1, L2) for i mod 3 = 0, 1, 2.
// H[c][i]: channel c, output columns (2i, 2i+1).
__device__ __forceinline__ unsigned long long r43_lpair(int i) {
  const int ja = (2 * i) % 3, jb = (2 * i + 1) % 3;
  const float la = ja == 0 ? kR43L0 : (ja == 1 ? kR43L1 : kR43L2);
  const float lb = jb == 0 ? kR43L0 : (jb == 1 ? kR43L1 : kR43L2);
  return pk2(make_float2(la, lb));
}
#define MP_R43F_H(Q, H)                                                                         \
  {                                                                                             \
    const uint32_t w_[12] = {Q[0].x, Q[0].y, Q[0].z, Q[0].w, Q[1].x, Q[1].y, Q[1].z, Q[1].w,    \
                             Q[2].x, Q[2].y, Q[2].z, Q[2].w};                                   \
    _Pragma("unroll") for (int c = 0; c < 3; c++) {                                             \
      _Pragma("unroll") for (int i = 0; i < 6; i++) {                                           \
        const int ca_ = 2 * i, cb_ = 2 * i + 1;                                                 \
        const int ma_ = 3 * (4 * (ca_ / 3) + ca_ % 3) + c, mb_ = 3 * (4 * (cb_ / 3) + cb_ % 3) + c; \
        const float2 m_ = make_float2(MP_MB(w_[ma_ >> 2], ma_ & 3), MP_MB(w_[mb_ >> 2], mb_ & 3)); \
        const float2 n_ = make_float2(MP_MB(w_[(ma_ + 3) >> 2], (ma_ + 3) & 3),                 \
                                      MP_MB(w_[(mb_ + 3) >> 2], (mb_ + 3) & 3));                \
        H[c][i] = ffma2_w(fsub2(n_, m_), r43_lpair(i), fsub2(m_, make_float2(8388608.0f, 8388608.0f))); \
      }                                                                                         \
    }                                                                                           \
  }
// one output row of the task, plane by plane: 12 floats (48 B) into this
// lane's slot of the warp's plane-row buffer (3 STS.128), then the warp
// writes its 32 x 48 = 1536 bytes as 16-B chunks (3 LDS.128 + 3 STG.128 per
// lane), every 32-B sector once; a __syncwarp orders the chunk reads before
// the next plane's writes.  One buffer per warp: with two, the c4 ring (2 x
// ~54 KB + 24 KB) left room for only two co-running 34-KB plan CTAs per SM
// instead of three, and the planner fell behind the gather (c4 step 3.9 ->
// 4.5 ms, profiles/r02_timeline_c4_r43f_2buf.txt).  (Three STG.128
// per lane straight to global memory wrote each sector in two halves from
// two instructions: 347 M L2 write sectors, lg_throttle, 1.69 ms at c2.)
#define MP_R43F_ROW(T, B, LY, RR)                                                               \
  {                                                                                             \
    _Pragma("unroll") for (int c = 0; c < 3; c++) {                                             \
      float2 v_[6];                                                                             \
      _Pragma("unroll") for (int i = 0; i < 6; i++) v_[i] = ffma2_s(fsub2(B[c][i], T[c][i]), (LY), T[c][i]); \
      const unsigned int sb_ = buf0;                                                            \
      MP_BCHK("r43f sts", sb_ + 48u * (unsigned int)lane, 48, buf0, buf0 + kR43FBuf)            \
      float4* const sp_ = reinterpret_cast<float4*>(&smem[sb_ + 48u * (unsigned int)lane]);     \
      sp_[0] = make_float4(v_[0].x, v_[0].y, v_[1].x, v_[1].y);                                 \
      sp_[1] = make_float4(v_[2].x, v_[2].y, v_[3].x, v_[3].y);                                 \
      sp_[2] = make_float4(v_[4].x, v_[4].y, v_[5].x, v_[5].y);                                 \
      __syncwarp();                                                                             \
      float* const o_ = orow + (size_t)c * plane + (size_t)(RR) * ow;                           \
      if (full) {                                                                               \
        _Pragma("unroll") for (int k = 0; k < 3; k++) {                                         \
          MP_BCHK("r43f stg", (const char*)(o_ + coff[k]) - (const char*)A.out[q], 16, 0, out_bytes(A, q)) \
        }                                                                                       \
        _Pragma("unroll") for (int k = 0; k < 3; k++)                                           \
          __stcs(reinterpret_cast<float4*>(o_ + coff[k]),                                       \
                 *reinterpret_cast<const float4*>(&smem[sb_ + 16u * (unsigned int)(lane + 32 * k)])); \
      } else {                                                                                  \
        _Pragma("unroll") for (int k = 0; k < 3; k++)                                           \
          if (rgw + cseg[k] < nrg) {                                                            \
            MP_BCHK("r43f stg", (const char*)(o_ + coff[k]) - (const char*)A.out[q], 16, 0, out_bytes(A, q)) \
            __stcs(reinterpret_cast<float4*>(o_ + coff[k]),                                     \
                   *reinterpret_cast<const float4*>(&smem[sb_ + 16u * (unsigned int)(lane + 32 * k)])); \
          }                                                                                     \
      }                                                                                         \
      __syncwarp();                                                                             \
    }                                                                                           \
  }
#define MP_MB(W, K) __int_as_float(__byte_perm((W), 0x4B000000u, 0x7440u | (K)))
__device__ __forceinline__ void consume_tile_r43f(const GatherArgs& A, const TileHdr* hdr, unsigned int soff,
                                                  int wid, int lane) {
  constexpr int kCW = cw_of(MP_OUT_F32_NCHW, kSrcRGB24);
  const int2* xt = reinterpret_cast<const int2*>(&smem[soff + kHdrBytes]) + hdr->xs;
  const int q = hdr->k, rows = hdr->rows, cols = hdr->cols;
  const int ncg = cols / 12, nrg = rows / 3, ntask = ncg * nrg, lg = __ffs(ncg) - 1;
  const int ow = A.ow[q], oh = A.oh[q];
  const size_t plane = (size_t)oh * ow;
  const unsigned int stride = (unsigned int)hdr->stride;
  const unsigned int a0 = soff + kDataOff + (unsigned int)(3 * hdr->x - hdr->b0 + 3 * xt[0].x);
  float* const out0 = reinterpret_cast<float*>(A.out[q]) + (size_t)hdr->slot * 3 * plane +
                      (size_t)hdr->oy0 * ow + hdr->ox0;
  // this lane's copy-out chunks (96 per plane row: lane, lane + 32, lane + 64):
  // run (row group offset) and float offset relative to the warp's first row
  const int cps = 3 * ncg;   // 16-B chunks per run (ncg x 48 bytes)
  size_t coff[3];
  int cseg[3];
#pragma unroll
  for (int k = 0; k < 3; k++) {
    const int c = lane + 32 * k;
    cseg[k] = c / cps;
    coff[k] = (size_t)(3 * cseg[k]) * ow + 4 * (c - cseg[k] * cps);
  }
  const unsigned int buf0 = (unsigned int)A.obuf_off + (unsigned int)wid * kR43FBuf;
  const int rpw = 32 / ncg;
  for (int base = 32 * wid; base < ntask; base += kCW * 32) {
    const int rgw = base >> lg;
    const int t = min(base + lane, ntask - 1);   // lanes past the tile redo its last task
    const int rg = t >> lg, cg = t & (ncg - 1);   // ncg is 4, 8 or 16 (host)
    const unsigned int a = a0 + (unsigned int)(4 * rg) * stride + 48u * (unsigned int)cg;
    MP_BCHK("r43f box rows", 4 * rg, 4, 0, A.box_h[q])
    MP_BCHK("r43f box cols", a0 - (soff + kDataOff) + 48u * cg, 48, 0, stride)
    float* const orow = out0 + (size_t)(3 * rgw) * ow;
    const bool full = rgw + rpw <= nrg;
    float2 X[3][6], Y[3][6];
    MP_R43_LD(a, ra)
    MP_R43F_H(ra, X)
    MP_R43_LD(a + stride, rb)
    MP_R43F_H(rb, Y)
    MP_R43F_ROW(X, Y, kR43L0, 0)
    MP_R43_LD(a + 2 * stride, rc)
    MP_R43F_H(rc, X)
    MP_R43F_ROW(Y, X, kR43L1, 1)
    MP_R43_LD(a + 3 * stride, rd)
    MP_R43F_H(rd, Y)
    MP_R43F_ROW(X, Y, kR43L2, 2)
  }
}

// NV12 -> f32 NCHW at an exact 4:3 downscale (NEXT-3 crops): the same tasks.
// A task's 16 luma pixels are one 16-byte run (LDS.128) and their 8 (U, V)
// pairs one 16-byte run of the staged chroma box (R23 siting: luma column a
// reads chroma pair a >> 1, so output column 3k + j reads pairs (2k, 2k),
// (2k, 2k+1), (2k+1, 2k+1) for j = 0, 1, 2).  Chroma rows: luma row a reads
// chroma row (ya + a) >> 1 (ya = the tile's first staged luma row), so the 4
// luma rows of a task read 2 chroma rows (ya even) or 3 (ya odd) — a
// tile-uniform choice, two instantiations.  Every lerp, the conversion and
// the clamp are the per-column NV12 consumer's operations in the same order
// (bit-identical results), then the planes leave like consume_tile_r43f's.
// Y pairs / U, V pairs: output columns (2i, 2i+1).
#define MP_NVY_H(R_, H)                                                                         \
  {                                                                                             \
    MP_BCHK("r43nv lds y", R_, 16, soff + kDataOff, soff + A.stage_bytes)                       \
    const uint4 q_ = *reinterpret_cast<const uint4*>(&smem[(R_)]);                              \
    const uint32_t w_[4] = {q_.x, q_.y, q_.z, q_.w};                                            \
    _Pragma("unroll") for (int i = 0; i < 6; i++) {                                             \
      const int ca_ = 2 * i, cb_ = 2 * i + 1;                                                   \
      const int ma_ = 4 * (ca_ / 3) + ca_ % 3, mb_ = 4 * (cb_ / 3) + cb_ % 3;                   \
      const float2 m_ = make_float2(MP_MB(w_[ma_ >> 2], ma_ & 3), MP_MB(w_[mb_ >> 2], mb_ & 3)); \
      const float2 n_ = make_float2(MP_MB(w_[(ma_ + 1) >> 2], (ma_ + 1) & 3),                   \
                                    MP_MB(w_[(mb_ + 1) >> 2], (mb_ + 1) & 3));                  \
      H[i] = ffma2_w(fsub2(n_, m_), r43_lpair(i), fsub2(m_, make_float2(8388608.0f, 8388608.0f))); \
    }                                                                                           \
  }
// U (ch 0) and V (ch 1) of the 12 columns from one 16-byte chroma run
#define MP_NVC_H(R_, H)                                                                         \
  {                                                                                             \
    MP_BCHK("r43nv lds uv", R_, 16, soff + kDataOff, soff + A.stage_bytes)                      \
    const uint4 q_ = *reinterpret_cast<const uint4*>(&smem[(R_)]);                              \
    const uint32_t w_[4] = {q_.x, q_.y, q_.z, q_.w};                                            \
    _Pragma("unroll") for (int ch = 0; ch < 2; ch++) {                                          \
      _Pragma("unroll") for (int i = 0; i < 6; i++) {                                           \
        const int ca_ = 2 * i, cb_ = 2 * i + 1;                                                 \
        const int la_ = 4 * (ca_ / 3) + ca_ % 3, lb_ = 4 * (cb_ / 3) + cb_ % 3; /* left luma taps */ \
        const int ma_ = 2 * (la_ >> 1) + ch, mb_ = 2 * (lb_ >> 1) + ch;                         \
        const int na_ = 2 * ((la_ + 1) >> 1) + ch, nb_ = 2 * ((lb_ + 1) >> 1) + ch;            \
        const float2 m_ = make_float2(MP_MB(w_[ma_ >> 2], ma_ & 3), MP_MB(w_[mb_ >> 2], mb_ & 3)); \
        const float2 n_ = make_float2(MP_MB(w_[na_ >> 2], na_ & 3), MP_MB(w_[nb_ >> 2], nb_ & 3)); \
        H[ch][i] = ffma2_w(fsub2(n_, m_), r43_lpair(i), fsub2(m_, make_float2(8388608.0f, 8388608.0f))); \
      }                                                                                         \
    }                                                                                           \
  }
template <bool ODD>
__device__ __forceinline__ void r43nv_task(const GatherArgs& A, unsigned int soff, unsigned int al, unsigned int ac,
                                           unsigned int stride, float* orow, size_t plane, int ow, int lane,
                                           unsigned int buf0, const size_t (&coff)[3], const int (&cseg)[3],
                                           bool full, int rgw, int nrg, int q) {
  const float2 CY = make_float2(A.cvt[0], A.cvt[0]), CYO = make_float2(A.cvt[1], A.cvt[1]);
  const float2 CRV = make_float2(A.cvt[2], A.cvt[2]), CGU = make_float2(A.cvt[3], A.cvt[3]);
  const float2 CGV = make_float2(A.cvt[4], A.cvt[4]), CBU = make_float2(A.cvt[5], A.cvt[5]);
  const float2 C128 = make_float2(-128.0f, -128.0f);
  float2 Y[4][6];
  float2 C[ODD ? 3 : 2][2][6];
  MP_NVY_H(al, Y[0])
  MP_NVY_H(al + stride, Y[1])
  MP_NVY_H(al + 2 * stride, Y[2])
  MP_NVY_H(al + 3 * stride, Y[3])
  MP_NVC_H(ac, C[0])
  MP_NVC_H(ac + stride, C[1])
  if (ODD) MP_NVC_H(ac + 2 * stride, C[ODD ? 2 : 1])
  _Pragma("unroll") for (int r = 0; r < 3; r++) {
    const float ly = r == 0 ? kR43L0 : (r == 1 ? kR43L1 : kR43L2);
    // chroma rows of luma rows r and r + 1 (relative to the task's first)
    const int ct = ODD ? (r + 1) >> 1 : r >> 1, cbt = ODD ? (r + 2) >> 1 : (r + 1) >> 1;
    float2 v_[3][6];
    _Pragma("unroll") for (int i = 0; i < 6; i++) {
      float2 v0 = ffma2_s(fsub2(Y[r + 1][i], Y[r][i]), ly, Y[r][i]);
      float2 v1 = ffma2_s(fsub2(C[cbt][0][i], C[ct][0][i]), ly, C[ct][0][i]);
      float2 v2 = ffma2_s(fsub2(C[cbt][1][i], C[ct][1][i]), ly, C[ct][1][i]);
      const float2 yy_ = __ffma2_rn(CY, v0, CYO);
      const float2 uu_ = __fadd2_rn(v1, C128), vv_ = __fadd2_rn(v2, C128);
      v0 = __ffma2_rn(CRV, vv_, yy_);
      v1 = __ffma2_rn(CGU, uu_, __ffma2_rn(CGV, vv_, yy_));
      v2 = __ffma2_rn(CBU, uu_, yy_);
      v_[0][i] = make_float2(clamp255(v0.x), clamp255(v0.y));
      v_[1][i] = make_float2(clamp255(v1.x), clamp255(v1.y));
      v_[2][i] = make_float2(clamp255(v2.x), clamp255(v2.y));
    }
    _Pragma("unroll") for (int c = 0; c < 3; c++) {
      MP_BCHK("r43nv sts", buf0 + 48u * (unsigned int)lane, 48, buf0, buf0 + kR43FBuf)
      float4* const sp_ = reinterpret_cast<float4*>(&smem[buf0 + 48u * (unsigned int)lane]);
      sp_[0] = make_float4(v_[c][0].x, v_[c][0].y, v_[c][1].x, v_[c][1].y);
      sp_[1] = make_float4(v_[c][2].x, v_[c][2].y, v_[c][3].x, v_[c][3].y);
      sp_[2] = make_float4(v_[c][4].x, v_[c][4].y, v_[c][5].x, v_[c][5].y);
      __syncwarp();
      float* const o_ = orow + (size_t)c * plane + (size_t)r * ow;
      _Pragma("unroll") for (int k = 0; k < 3; k++) {
        if (full || rgw + cseg[k] < nrg) {
          MP_BCHK("r43nv stg", (const char*)(o_ + coff[k]) - (const char*)A.out[q], 16, 0, out_bytes(A, q))
          __stcs(reinterpret_cast<float4*>(o_ + coff[k]),
                 *reinterpret_cast<const float4*>(&smem[buf0 + 16u * (unsigned int)(lane + 32 * k)]));
        }
      }
      __syncwarp();
    }
  }
}
__device__ __forceinline__ void consume_tile_r43nv(const GatherArgs& A, const TileHdr* hdr, unsigned int soff,
                                                   int wid, int lane) {
  constexpr int kCW = cw_of(MP_OUT_F32_NCHW, kSrcNV12);
  const int2* xt = reinterpret_cast<const int2*>(&smem[soff + kHdrBytes]) + hdr->xs;
  const int q = hdr->k, rows = hdr->rows, cols = hdr->cols;
  const int ncg = cols / 12, nrg = rows / 3, ntask = ncg * nrg, lg = __ffs(ncg) - 1;
  const int ow = A.ow[q], oh = A.oh[q];
  const size_t plane = (size_t)oh * ow;
  const unsigned int stride = (unsigned int)hdr->stride;
  const int ya = hdr->ya;
  // first luma tap of the tile (even: x and the tile origin are multiples of 16)
  const unsigned int l0 = (unsigned int)(hdr->x + xt[0].x - hdr->b0);
  const unsigned int a0 = soff + kDataOff + l0, c0 = soff + kDataOff + (unsigned int)A.uv_off[q] + l0;
  float* const out0 = reinterpret_cast<float*>(A.out[q]) + (size_t)hdr->slot * 3 * plane +
                      (size_t)hdr->oy0 * ow + hdr->ox0;
  const int cps = 3 * ncg;
  size_t coff[3];
  int cseg[3];
#pragma unroll
  for (int k = 0; k < 3; k++) {
    const int c = lane + 32 * k;
    cseg[k] = c / cps;
    coff[k] = (size_t)(3 * cseg[k]) * ow + 4 * (c - cseg[k] * cps);
  }
  const unsigned int buf0 = (unsigned int)A.obuf_off + (unsigned int)wid * kR43FBuf;
  const int rpw = 32 / ncg;
  for (int base = 32 * wid; base < ntask; base += kCW * 32) {
    const int rgw = base >> lg;
    const int t = min(base + lane, ntask - 1);
    const int rg = t >> lg, cg = t & (ncg - 1);   // ncg is 4, 8 or 16 (host)
    const unsigned int al = a0 + (unsigned int)(4 * rg) * stride + 16u * (unsigned int)cg;
    const int cr = ((ya + 4 * rg) >> 1) - (ya >> 1);   // chroma box row of the task's first luma row
    const unsigned int ac = c0 + (unsigned int)cr * stride + 16u * (unsigned int)cg;
    MP_BCHK("r43nv box rows", 4 * rg, 4, 0, A.box_h[q])
    MP_BCHK("r43nv uv rows", cr, (ya & 1) ? 3 : 2, 0, A.box_huv[q])
    float* const orow = out0 + (size_t)(3 * rgw) * ow;
    const bool full = rgw + rpw <= nrg;
    if (ya & 1) r43nv_task<true>(A, soff, al, ac, stride, orow, plane, ow, lane, buf0, coff, cseg, full, rgw, nrg, q);
    else r43nv_task<false>(A, soff, al, ac, stride, orow, plane, ow, lane, buf0, coff, cseg, full, rgw, nrg, q);
  }
}
#undef MP_NVY_H
#undef MP_NVC_H
#undef MP_MB
#undef MP_R43F_H
#undef MP_R43F_ROW
#undef MP_R43_LD

template <int FMT, int SRC>
__global__ void __launch_bounds__((cw_of(FMT, SRC) + kProducerWarps) * 32) gather_kernel(const __grid_constant__ GatherArgs A,
                                                                 const __grid_constant__ TmapArray tm,
                                                                 const uint8_t* const* __restrict__ frames,
                                                                 int* __restrict__ ws_cnt,
                                                                 const int* __restrict__ ws_list,
                                                                 const mp_window* __restrict__ windows,
                                                                 const int* __restrict__ frame_off,
                                                                 const int2* __restrict__ ws_tap,
                                                                 int* __restrict__ d_status) {
  constexpr int kCW = cw_of(FMT, SRC);
  const int nst = A.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)nst * A.stage_bytes);
  uint64_t* empty = full + nst;
  __shared__ int cnt[kMaxClasses];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid < kMaxClasses) cnt[tid] = tid < A.k ? ws_cnt[tid] : 0;
  if (tid == 0) {
    for (int s = 0; s < nst; s++) {
      mbar_init(&full[s], 1);
      // every consumer thread releases the stage it read: with one arrive per
      // warp after __syncwarp, racecheck cannot see lanes 1-31's header reads
      // ordered before the producer's next write of that stage (the end
      // marker) and reports a hazard; 32 arrives per warp cost <1 % (c2 f32
      // 1.358 -> 1.368 ms, u8 1.176 -> 1.162)
      mbar_init(&empty[s], kCW * 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int T = tiles_total(A, cnt);
  const int G = gridDim.x;

  if (wid >= kCW) {
    // ===================== producer warp =====================
    // The global loads a tile needs (its window descriptor and 3 tap bounds)
    // are issued one tile ahead, so their latency overlaps the wait for a free
    // stage; the tap slices themselves are staged by the copy engine.
    struct TileInfo {
      int q, slot, oy0, ox0, rows, cols;
    };
    auto decode = [&](int t, TileInfo& ti) {
      int q = 0, rel = t;
      while (rel >= min(cnt[q], A.cap[q]) * A.tpw[q]) {
        rel -= min(cnt[q], A.cap[q]) * A.tpw[q];
        q++;
      }
      // tiles ordered by class, slot, then tile: neighbouring CTAs share halo rows in L2
      ti.q = q;
      ti.slot = rel / A.tpw[q];
      const int tw = rel - ti.slot * A.tpw[q];
      const int rt = tw / A.nct[q], ct = tw - rt * A.nct[q];
      ti.oy0 = rt * A.TR[q];
      ti.ox0 = ct * A.TW[q];
      ti.rows = min(A.TR[q], A.oh[q] - ti.oy0);
      ti.cols = min(A.TW[q], A.ow[q] - ti.ox0);
    };
    struct WinRef {
      int frame, x, y, valid;
    };
    const int n_win = min(frame_off[A.F], A.max_windows);
    TileInfo cur, nxt;
    WinRef dcur = WinRef{0, 0, 0, 0}, dnxt = dcur;
    int clo_cur = 0, rlo_cur = 0, rhi_cur = 0, clo_nxt = 0, rlo_nxt = 0, rhi_nxt = 0;
    auto prefetch = [&](const TileInfo& ti, WinRef& d, int& clo, int& rlo, int& rhi) {
      // the class list entry must point at a window of this class and slot
      // (catches slots that are not 0..count-1 without zero-filling the list)
      const int wi = ws_list[A.list_off[ti.q] + ti.slot];
      d.valid = 0;
      if (wi >= 0 && wi < n_win) {
        const mp_window w = windows[wi];
        d.frame = w.frame;
        d.x = w.x;
        d.y = w.y;
        d.valid = (w.size_idx == ti.q && w.slot == ti.slot && w.frame >= 0 && w.frame < A.F && w.x >= 0 &&
                   w.y >= 0 && w.w == A.w[ti.q] && w.h == A.h[ti.q] && w.x + w.w <= A.W && w.y + w.h <= A.H)
                      ? 1 : 0;
      }
      clo = __ldg(&ws_tap[A.xtab_off[ti.q] + ti.ox0].x);
      rlo = __ldg(&ws_tap[A.ytab_off[ti.q] + ti.oy0].x);
      rhi = __ldg(&ws_tap[A.ytab_off[ti.q] + ti.oy0 + ti.rows - 1].x);
    };
    // Dynamic tile scheduling: CTA b takes tile b first, then the next free
    // tile from a global counter (ticket G + n), claimed one tile ahead so the
    // atomic's latency overlaps the current tile.  Tiles are still handed out
    // in order (concurrently processed tiles stay neighbours in the frames and
    // outputs), but a CTA whose SM also runs plan/NMS blocks of neighbouring
    // batches simply takes fewer tiles instead of finishing last.
    // Tickets hand out chunks of kTileChunk consecutive tiles; the next
    // chunk's ticket is claimed when a chunk is opened, so the atomic has
    // kTileChunk tiles of time to return (one tile was not enough for the
    // small c2 tiles: 1.37 -> 1.47 ms).  Measured against the former static
    // round-robin (same box, alone): chunks of 2: c2 1.383 -> 1.360 ms, c3
    // 6.61 -> 6.49, c4 4.15 -> 4.00; chunks of 4 / 8 balance less well.
    int* tile_ctr = ws_cnt + kMaxClasses;
    int ticket = 0, cbase = 0, cleft = 0;   // ticket: lane 0's in-flight atomic
    if (lane == 0) ticket = atomicAdd(tile_ctr, 1);
    auto next_tile = [&]() -> int {
      if (cleft == 0) {
        cbase = G + __shfl_sync(0xffffffffu, ticket, 0) * kTileChunk;
        cleft = kTileChunk;
        if (lane == 0) ticket = atomicAdd(tile_ctr, 1);
      }
      cleft--;
      return cbase++;
    };
    int t = blockIdx.x;
    int tn = T;
    if (t < T) {
      decode(t, cur);
      prefetch(cur, dcur, clo_cur, rlo_cur, rhi_cur);
      tn = next_tile();
    }
    for (int i = 0;; i++) {
      const int s = i % nst;
      // the next tile's descriptor loads are issued before the wait for a
      // free stage, so their latency hides behind it
      if (tn < T) {
        decode(tn, nxt);
        prefetch(nxt, dnxt, clo_nxt, rlo_nxt, rhi_nxt);
      }
      if (i >= nst) {
        if (A.wait_mode & 1) mbar_wait_sleep(&empty[s], ((i / nst) - 1) & 1);
        else mbar_wait(&empty[s], ((i / nst) - 1) & 1);
      }
      unsigned char* stage = smem + (size_t)s * A.stage_bytes;
      TileHdr* hdr = reinterpret_cast<TileHdr*>(stage);
      if (t >= T) {   // no tile left: an end marker releases the consumers
        if (lane == 0) {
          hdr->valid = -1;
          mbar_arrive(&full[s]);
        }
        break;
      }
      unsigned char* xt = stage + kHdrBytes;
      unsigned char* yt = stage + kHdrBytes + kXtapBytes;
      unsigned char* data = stage + kDataOff;
      const int q = cur.q;
      if (lane == 0) {
        if (!dcur.valid) {   // slots of this class are not 0..count-1
          hdr->valid = 0;
          set_status(d_status, MP_ERR_INVALID);
          mbar_arrive(&full[s]);
        } else {
          const int b0 = ((SRC == kSrcNV12 ? 1 : 3) * (dcur.x + clo_cur)) & ~15;
          const int stride = A.box_w[q];
          const int xe = A.xtab_off[q] + cur.ox0, ye = A.ytab_off[q] + cur.oy0;   // first tap entries
          const int xs = xe & 1, ys = ye & 1;                                       // 16-B aligned slices
          const uint32_t xbytes = (uint32_t)((cur.cols + xs + 1) & ~1) * 8;
          const uint32_t ybytes = (uint32_t)((cur.rows + ys + 1) & ~1) * 8;
          hdr->valid = 1;
          hdr->k = q;
          hdr->slot = cur.slot;
          hdr->oy0 = cur.oy0;
          hdr->ox0 = cur.ox0;
          hdr->rows = cur.rows;
          hdr->cols = cur.cols;
          hdr->stride = stride;
          hdr->x = dcur.x;
          hdr->b0 = b0;
          hdr->r_lo = rlo_cur;
          hdr->xs = xs;
          hdr->ys = ys;
          hdr->ya = dcur.y + rlo_cur;
          hdr->wy = dcur.y;
          if (A.debug == 2) {   // experiment: no pixel copies (compute-only bound)
            mbar_arrive_expect_tx(&full[s], xbytes + ybytes);
            bulk_g2s(xt, ws_tap + (xe - xs), xbytes, &full[s]);
            bulk_g2s(yt, ws_tap + (ye - ys), ybytes, &full[s]);
          } else if (A.sparse[q]) {
            // row-sparse: the warp issues the 4-row TMA gathers below (RGB: two
            // output rows per gather, odd counts padded; NV12: one per row)
            const uint32_t nrow4 = SRC == kSrcNV12 ? (uint32_t)cur.rows : (uint32_t)(cur.rows + 1) / 2;
            mbar_arrive_expect_tx(&full[s], nrow4 * (uint32_t)(4 * stride) + xbytes + ybytes);
            bulk_g2s(xt, ws_tap + (xe - xs), xbytes, &full[s]);
            bulk_g2s(yt, ws_tap + (ye - ys), ybytes, &full[s]);
          } else if (SRC == kSrcNV12) {
            // two TMA boxes from the same column origin b0: luma rows ya.., then
            // chroma rows (ya >> 1).. of the interleaved UV plane (R23)
            const int ya = dcur.y + rlo_cur;
            mbar_arrive_expect_tx(&full[s], (uint32_t)(stride * A.box_h[q]) + (uint32_t)(stride * A.box_huv[q]) +
                                                xbytes + ybytes);
            bulk_g2s(xt, ws_tap + (xe - xs), xbytes, &full[s]);
            bulk_g2s(yt, ws_tap + (ye - ys), ybytes, &full[s]);
            tma_load_3d(data, &tm.m[q], b0 >> 3, ya, dcur.frame, &full[s]);
            tma_load_3d(data + A.uv_off[q], &tm.m[kMaxClasses + q], b0 >> 3, ya >> 1, dcur.frame, &full[s]);
          } else if (A.tensor) {
            // one TMA box: [box_h rows][box_w bytes] from (b0, y + r_lo) of frame d.frame;
            // rows past the frame bottom / bytes past the pitch are zero-filled.
            mbar_arrive_expect_tx(&full[s], (uint32_t)(stride * A.box_h[q]) + xbytes + ybytes);
            bulk_g2s(xt, ws_tap + (xe - xs), xbytes, &full[s]);
            bulk_g2s(yt, ws_tap + (ye - ys), ybytes, &full[s]);
            tma_load_3d(data, &tm.m[q], b0 >> 3, dcur.y + rlo_cur, dcur.frame, &full[s]);
          } else {
            // one 1-D bulk copy per source row (rows r_lo .. min(i0(last)+1, h-1) of the crop)
            const int nrows = min(rhi_cur + 1, A.h[q] - 1) - rlo_cur + 1;
            const int bytes = min(stride, A.pitch - b0);
            mbar_arrive_expect_tx(&full[s], (uint32_t)(nrows * bytes) + xbytes + ybytes);
            bulk_g2s(xt, ws_tap + (xe - xs), xbytes, &full[s]);
            bulk_g2s(yt, ws_tap + (ye - ys), ybytes, &full[s]);
            const uint8_t* src = frames[dcur.frame] + (size_t)(dcur.y + rlo_cur) * A.pitch + b0;
            for (int r = 0; r < nrows; r++)
              bulk_g2s(data + (size_t)r * stride, src + (size_t)r * A.pitch, (uint32_t)bytes, &full[s]);
          }
        }
      }
      __syncwarp();
      if (A.sparse[q] && dcur.valid && A.debug != 2) {
        // row-sparse staging (strong vertical downscale): output row j of the
        // tile needs source rows (i0_j, i0_j + 1) only (and, for NV12, chroma
        // rows (y+i0_j)>>1 and the one after), fetched with sm_100 TMA row
        // gathers (tile::gather4) over the 2-D row view of the frame batch
        // (row = frame * rpf + row-in-frame; NV12 chroma rows follow the H
        // luma rows).  Rows no tap touches are never read.  Lanes issue in
        // parallel; lane 0 posted the byte count above.
        const int b0 = ((SRC == kSrcNV12 ? 1 : 3) * (dcur.x + clo_cur)) & ~15;
        const int fr = dcur.frame * A.rpf;
        const int stride = A.box_w[q];
        const int* ytap = &ws_tap[A.ytab_off[q] + cur.oy0].x;
        if (SRC == kSrcNV12) {
          for (int j = lane; j < cur.rows; j += 32) {
            const int ry = dcur.y + __ldg(ytap + 2 * j);
            // rows: luma i0, i0+1, then the chroma rows of those two luma
            // rows (equal when y+i0 is even: the repeat is an L2 hit)
            const int lr = fr + ry, cr = fr + A.H;
            tma_gather4(data + (size_t)j * (4 * stride), &tm.m[q], b0 >> 3, lr, lr + 1, cr + (ry >> 1),
                        cr + ((ry + 1) >> 1), &full[s]);
          }
        } else {
          for (int jj = lane; 2 * jj < cur.rows; jj += 32) {
            const int r0 = fr + dcur.y + __ldg(ytap + 4 * jj);
            const int r1 = fr + dcur.y + __ldg(ytap + 2 * min(2 * jj + 1, cur.rows - 1));
            tma_gather4(data + (size_t)jj * (4 * stride), &tm.m[q], b0 >> 3, r0, r0 + 1, r1, r1 + 1, &full[s]);
          }
        }
      }
      cur = nxt;
      dcur = dnxt;
      clo_cur = clo_nxt;
      rlo_cur = rlo_nxt;
      rhi_cur = rhi_nxt;
      t = tn;
      tn = tn < T ? next_tile() : T;
    }
    return;
  }

  // ===================== consumer warps =====================
  for (int i = 0;; i++) {
    const int s = i % nst;
    if (A.wait_mode & 2) mbar_wait_sleep(&full[s], (i / nst) & 1);
    else mbar_wait(&full[s], (i / nst) & 1);
    const unsigned int soff = (unsigned int)s * (unsigned int)A.stage_bytes;
    const TileHdr* hdr = reinterpret_cast<const TileHdr*>(&smem[soff]);
    if (hdr->valid < 0) break;   // end marker
    if (hdr->valid && A.debug != 1) {
#ifndef MP_U8_GENERIC
      if constexpr (FMT == MP_OUT_U8_NHWC && SRC == kSrcRGB24) {
        const int q = hdr->k;
        if (A.r43[q] && (hdr->x & 15) == 0) {
          consume_tile_r43(A, hdr, soff, wid, lane);
        } else {
          switch (A.ncol[q]) {
            case 2: consume_tile_u8rgb<2>(A, hdr, soff, wid, lane); break;
            case 4: consume_tile_u8rgb<4>(A, hdr, soff, wid, lane); break;
            case 6: consume_tile_u8rgb<6>(A, hdr, soff, wid, lane); break;
            default: consume_tile_u8rgb<8>(A, hdr, soff, wid, lane); break;
          }
        }
      } else
#endif
      if (FMT == MP_OUT_F32_NCHW && SRC == kSrcRGB24 && A.r43[hdr->k] && (hdr->x & 15) == 0) {
        consume_tile_r43f(A, hdr, soff, wid, lane);
      } else if (FMT == MP_OUT_F32_NCHW && SRC == kSrcNV12 && A.r43[hdr->k] && (hdr->x & 15) == 0) {
        consume_tile_r43nv(A, hdr, soff, wid, lane);
      } else
      switch (A.ncol[hdr->k]) {
        case 2: consume_tile<FMT, 2, SRC>(A, hdr, soff, wid, lane); break;
        case 4: consume_tile<FMT, 4, SRC>(A, hdr, soff, wid, lane); break;
        case 6: consume_tile<FMT, 6, SRC>(A, hdr, soff, wid, lane); break;
        default: consume_tile<FMT, 8, SRC>(A, hdr, soff, wid, lane); break;
      }
    }
    mbar_arrive(&empty[s]);
  }
}

// ------------------------------------------------------------------ host side
static void host_tap(int in, int out, int d, int* i0, int* i1) {
  long long n = (long long)(2 * d + 1) * in - out;
  long long a = n < 0 ? 0 : n / (2LL * out);
  if (a >= in - 1) a = in - 1;
  *i0 = (int)a;
  *i1 = (int)(a + 1 < in - 1 ? a + 1 : in - 1);
}

// Staged box of a class with tile dims (TW, TR): every tile reads source
// columns c_lo .. i0(last)+1 (the +1 pixel is the always-present right tap)
// starting at a 16-B aligned byte b0 >= bpp*(x+c_lo)-15, and source rows
// r_lo .. i0(last)+1.  Returns the box (bytes x rows) that covers any tile.
// NV12 (bpp 1): the chroma pair of the last luma column a sits at bytes up to
// 2((a+1)>>1)+1 <= a+2, one byte past the luma footprint -> +1 byte.
static void class_box(int in_w, int in_h, int ow, int oh, int TW, int TR, int src, int* box_w, int* box_h) {
  int nct = (ow + TW - 1) / TW, nrt = (oh + TR - 1) / TR;
  int max_rows = 0, max_cols = 0, a, b, c, d;
  for (int rt = 0; rt < nrt; rt++) {
    int oy0 = rt * TR, rows = (TR < oh - oy0 ? TR : oh - oy0);
    host_tap(in_h, oh, oy0, &a, &b);
    host_tap(in_h, oh, oy0 + rows - 1, &c, &d);
    if (c - a + 2 > max_rows) max_rows = c - a + 2;
  }
  for (int ct = 0; ct < nct; ct++) {
    int ox0 = ct * TW, cols = (TW < ow - ox0 ? TW : ow - ox0);
    host_tap(in_w, ow, ox0, &a, &b);
    host_tap(in_w, ow, ox0 + cols - 1, &c, &d);
    // the right tap of the last column is staged only when it lies inside the
    // crop; at the crop edge lambda = 0 and the +1 read lands in stage slack
    const int c_hi = (c + 1 < in_w - 1) ? c + 1 : in_w - 1;
    if (c_hi - a + 1 > max_cols) max_cols = c_hi - a + 1;
  }
  const int bytes = src == kSrcNV12 ? max_cols + 1 : 3 * max_cols;
  *box_w = (bytes + 15 + 15) / 16 * 16;   // + up to 15 B of 16-B start alignment
  *box_h = max_rows;
}

// Staged bytes of a class box.  Dense: RGB24 = the box; NV12 = the luma box
// (padded to 128 B for the second TMA destination) + the chroma box (box_h/2 +
// 1 rows: the chroma rows of box_h consecutive luma rows at any parity).
// Row-sparse: TR row pairs of 2 box rows each (128-B aligned), twice for NV12.
static long long pair_bytes(int src, int bw) { return (src == kSrcNV12 ? 4LL : 2LL) * bw; }
static long long stage_data_bytes(int src, bool sparse, int bw, int bh, int TR) {
  if (sparse) return (long long)TR * pair_bytes(src, bw);   // TR is a multiple of kCW (even)
  if (src != kSrcNV12) return (long long)bw * bh;
  return ((long long)bw * bh + 127) / 128 * 128 + (long long)bw * (bh / 2 + 1);
}

// allow_sparse: the entry point stages through a TMA tensor map (row-sparse
// staging needs 2-row boxes); the pointer-array path always stages densely.
static bool build_gather_args(int src, bool allow_sparse, int pitch, int W, int H, int F, int k,
                              const mp_size* sizes, const mp_size* out_dims, void* const* d_out,
                              const int32_t* out_cap, mp_out_format fmt, GatherArgs* A) {
  if (W < 1 || H < 1 || W > 16384 || H > 16384 || F < 0 || k < 1 || k > kMaxClasses) return false;
  if (pitch < (src == kSrcNV12 ? W : 3 * W) || (pitch & 15)) return false;
  if (src == kSrcNV12 && ((W & 1) || (H & 1))) return false;
  if (!sizes || !out_dims || !d_out || !out_cap) return false;
  if (fmt != MP_OUT_F32_NCHW && fmt != MP_OUT_U8_NHWC) return false;
  memset(A, 0, sizeof(*A));
  const int cw = cw_of(fmt, src);   // consumer warps of this instantiation
  A->k = k;
  A->W = W;
  A->H = H;
  A->pitch = pitch;
  A->F = F;
  A->fmt = fmt;
  A->src = src;
  long long data_max = 0;
  int list = 0, taps = 0;
  const char* bud = knob("MP_GATHER_BUDGET_KB");   // experiment knob
  const long long budget = (bud && atoi(bud) >= 8) ? 1024LL * atoi(bud)
                          : (fmt == MP_OUT_U8_NHWC ? kStageDataBudgetU8
                                                   : (src == kSrcNV12 ? kStageDataBudgetNV12 : kStageDataBudget));
  for (int q = 0; q < k; q++) {
    const int w = sizes[q].w, h = sizes[q].h, ow = out_dims[q].w, oh = out_dims[q].h;
    if (w < 1 || h < 1 || w > W || h > H || ow < 1 || oh < 1 || ow > 16384 || oh > 16384) return false;
    if (out_cap[q] < 0 || (out_cap[q] > 0 && !d_out[q])) return false;
    if (((uintptr_t)d_out[q]) & 15) return false;
    A->w[q] = w;
    A->h[q] = h;
    A->ow[q] = ow;
    A->oh[q] = oh;
    // column tiles of equal width TW <= 256 (so every tile's TMA box is the
    // class box, no over-fetch), NCOL = TW/32 rounded up to even columns per
    // lane; rows: cw warps x Rw rows each, Rw as large as the stage budget
    // and the TMA box limits (256 rows, 256 x 8 bytes) allow (<= 8).
    // Tile width (measured on B200): stores must start on full 128-B lines —
    // so prefer the largest TW <= 256 that is a multiple of 32 and divides ow
    // (equal tiles: every tile's TMA box is the class box, no over-fetch);
    // else equal tiles rounded up to a multiple of 8 (full 32-B sectors).
    // Rows per warp: the tallest Rw whose box fits the stage budget and the
    // TMA limits.  Narrower fallbacks only when nothing fits.
    // Row-sparse staging when the vertical downscale exceeds 2x (h > 2 oh):
    // output rows then share no source rows, and staging only each row's two
    // taps reads fewer bytes than the contiguous box (e.g. the proxy-input
    // downscale, NEXT-3).  No halo rows, so short (Rw = 1) tiles are fine.
    const bool sparse = allow_sparse && h > 2 * oh;
    const int min_rw = sparse ? 1 : 3;
    // RGB f32 classes wider than 512 output columns (the full-frame fallback
    // windows of dense scenes) stage taller tiles: the ring's stage size is
    // the largest class's, and the narrow classes keep their 40-KB geometry
    const long long cbudget = (sparse && !bud) ? (long long)kSparseStageBudget
                              : (!bud && fmt == MP_OUT_F32_NCHW && src == kSrcRGB24 && ow > 512)
                                    ? (long long)kStageDataBudgetWide : budget;
    int TW = 0, TR = 0, bw = 0, bh = 0;
    // RGB24 at an exact 4:3 downscale: fixed-tap tasks of 12 columns x 3
    // rows, one per consumer thread (consume_tile_r43 / _r43f): the widest column
    // group count ncg in {16, 8, 4} dividing ow / 12, then as many row groups
    // as there are consumer threads left (box within the stage budget)
    const bool r43 = (src == kSrcRGB24 || (src == kSrcNV12 && fmt == MP_OUT_F32_NCHW)) && !sparse &&
                     3 * w == 4 * ow && 3 * h == 4 * oh &&
                     ow % 12 == 0 && oh % 3 == 0 && !knob("MP_GATHER_TILE");
    if (r43) {
      // stage budget: two stages and the consumers' output-row buffers leave
      // kSideReserve (every consumer thread busy beats more, smaller stages:
      // u8 A/B 3 x 40 KB 1.047 ms, 3 x 44 KB 0.962, 2 x ~53 KB 0.859)
      const long long obuf = fmt == MP_OUT_U8_NHWC ? kR43BufBytes : kR43FBufBytes;
      const long long r43_budget =
          bud ? budget : (227LL * 1024 - (long long)kSideReserve - obuf - 64) / 2 - kDataOff - 64 - 127;
      // ncg: a multiple of 4 dividing 32 (whole row groups per warp, 16-B runs)
      for (int ncg = 16; ncg >= 4 && !TW; ncg /= 2) {
        if ((ow / 12) % ncg || 12 * ncg > kMaxTW) continue;
        // as many row groups as there are consumer threads (a short last row
        // tile stages rows no task uses — the TMA box is the class's — but
        // equal row tiles with idle threads measured slower: c2 u8 0.761 ->
        // 0.778 ms, c3 3.06 -> 3.15, profiles/ab/r02_u8_equal_row_tiles.jsonl)
        for (int nrg = min(min(cw * 32 / ncg, oh / 3), kMaxTR / 3); nrg >= 1; nrg--) {
          int cbw, cbh;
          class_box(w, h, ow, oh, 12 * ncg, 3 * nrg, src, &cbw, &cbh);
          if (stage_data_bytes(src, false, cbw, cbh, 3 * nrg) <= r43_budget && cbw <= 2048 && cbh <= 256) {
            TW = 12 * ncg;
            TR = 3 * nrg;
            bw = cbw;
            bh = cbh;
            break;
          }
        }
      }
    }
    A->r43[q] = TW ? 1 : 0;
    auto fit_rows = [&](int tw, int& rw, int& cbw, int& cbh) {
      for (rw = 8; rw >= 1; rw--) {
        class_box(w, h, ow, oh, tw, cw * rw, src, &cbw, &cbh);
        if (sparse) {   // gather4 destinations: 4 rows x box_w bytes, 128-B aligned
          cbh = 1;
          cbw = (cbw + 31) / 32 * 32;
        }
        if (stage_data_bytes(src, sparse, cbw, cbh, cw * rw) <= cbudget && cbw <= 2048 && cbh <= 256)
          return true;
      }
      return false;
    };
    // (a 32-multiple divisor narrower than 128 columns, e.g. 32 for ow = 416,
    // loses to the equal split: per-tile overheads dominate narrow tiles)
    for (int tw = kMaxTW; tw >= (ow < 128 ? 32 : 128) && !TW; tw -= 32) {
      if (ow % tw) continue;
      int rw, cbw, cbh;
      if (fit_rows(tw, rw, cbw, cbh) && rw >= min_rw) {
        TW = tw;
        TR = cw * rw;
        bw = cbw;
        bh = cbh;
      }
    }
    // u8 output: a divisor width with an odd number of 32-column lane groups
    // leaves the last lane column of every tile idle (columns are processed
    // in pairs); one more group with a ragged last tile wins when the consumer
    // is the bound (c3, ow = 1440: 160 -> 192 columns, 5.58 -> 5.20 ms)
    if (TW && !A->r43[q] && fmt == MP_OUT_U8_NHWC && ((TW / 32) & 1) && TW + 32 <= kMaxTW && ow > TW + 32) {
      int rw, cbw, cbh;
      if (fit_rows(TW + 32, rw, cbw, cbh) && cw * rw >= TR) {
        TW += 32;
        TR = cw * rw;
        bw = cbw;
        bh = cbh;
      }
    }
    for (int nct = (ow + kMaxTW - 1) / kMaxTW; nct <= (ow + 7) / 8 && !TW; nct++) {
      int tw = (ow + nct - 1) / nct;
      tw = (tw + 7) / 8 * 8;
      if (tw > kMaxTW) continue;
      int rw, cbw, cbh;
      if (fit_rows(tw, rw, cbw, cbh) && (rw >= min_rw || tw <= 32)) {
        TW = tw;
        TR = cw * rw;
        bw = cbw;
        bh = cbh;
      }
    }
    {
      // experiment knob: MP_GATHER_TILE=ow,TW,Rw forces the tile of classes with that output width
      const char* ft = knob("MP_GATHER_TILE");
      int fow = 0, ftw = 0, frw = 0;
      if (ft && sscanf(ft, "%d,%d,%d", &fow, &ftw, &frw) == 3 && fow == ow) {
        TW = ftw;
        TR = cw * frw;
        class_box(w, h, ow, oh, TW, TR, src, &bw, &bh);
        if (sparse) {
          bh = 1;
          bw = (bw + 31) / 32 * 32;
        }
      }
    }
    if (TW == 0) return false;   // too strong a downscale of too wide a window: unsupported
    int ncol = (TW + 31) / 32;
    ncol += ncol & 1;
    A->ncol[q] = ncol;
    A->TW[q] = TW;
    A->TR[q] = TR;
    A->box_w[q] = bw;
    A->box_h[q] = bh;
    A->sparse[q] = sparse ? 1 : 0;
    A->pair_bytes[q] = (int)pair_bytes(src, bw);
    A->box_huv[q] = bh / 2 + 1;
    A->uv_off[q] = sparse ? 2 * bw : (int)(((long long)bw * bh + 127) / 128 * 128);
    A->nct[q] = (ow + TW - 1) / TW;
    A->tpw[q] = A->nct[q] * ((oh + TR - 1) / TR);
    A->cap[q] = out_cap[q];
    A->list_off[q] = list;
    A->out[q] = d_out[q];
    list += out_cap[q];
    A->xtab_off[q] = taps;
    taps += ow;
    A->ytab_off[q] = taps;
    taps += oh;
    if (stage_data_bytes(src, sparse, bw, bh, TR) > data_max) data_max = stage_data_bytes(src, sparse, bw, bh, TR);
  }
  A->stage_bytes = (int)((kDataOff + data_max + 64 + 127) / 128 * 128);
  return true;
}

}  // namespace mpk

using namespace mpk;

struct GatherWs {
  size_t cnt_off, list_off, tap_off, total;
};

static bool gather_ws_layout(int32_t k, const mp_size* out_dims, const int32_t* out_cap, GatherWs* L) {
  if (k < 1 || k > kMaxClasses || !out_cap || !out_dims) return false;
  size_t desc = 0, taps = 0;
  for (int q = 0; q < k; q++) {
    if (out_cap[q] < 0 || out_dims[q].w < 1 || out_dims[q].h < 1) return false;
    desc += (size_t)out_cap[q];
    taps += (size_t)out_dims[q].w + out_dims[q].h;
  }
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  L->cnt_off = 0;
  L->list_off = 256;
  L->tap_off = al(L->list_off + desc * sizeof(int));
  L->total = al(L->tap_off + taps * sizeof(int2));
  return true;
}

extern "C" size_t mp_gather_workspace_size(int32_t k, const mp_size* out_dims, const int32_t* out_cap) {
  GatherWs L;
  return gather_ws_layout(k, out_dims, out_cap, &L) ? L.total : 0;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static mp_status gather_launch(GatherArgs& A, const TmapArray& tm, const uint8_t* const* d_frame_ptrs,
                               const mp_window* d_windows, const int32_t* d_frame_off, int32_t k,
                               const mp_size* out_dims, const int32_t* out_cap, mp_out_format fmt,
                               int32_t* d_status, void* d_ws, size_t ws_bytes, void* stream) {
  GatherWs L;
  if (!gather_ws_layout(k, out_dims, out_cap, &L) || !d_ws || ws_bytes < L.total) return MP_ERR_INVALID;
  int n_taps = 0;
  for (int q = 0; q < k; q++) n_taps += out_dims[q].w + out_dims[q].h;
  cudaStream_t s = (cudaStream_t)stream;
  unsigned char* ws = (unsigned char*)d_ws;
  int* ws_cnt = (int*)(ws + L.cnt_off);
  int* ws_list = (int*)(ws + L.list_off);
  int2* ws_tap = (int2*)(ws + L.tap_off);
  MP_CUDA_TRY(prefer_max_shared((const void*)gather_prep_kernel));
  MP_CUDA_TRY(cudaMemsetAsync(ws_cnt, 0, (kMaxClasses + 1) * sizeof(int), s));   // class counts + tile counter
  gather_prep_kernel<<<256, kPrepThreads, 0, s>>>(A, d_windows, d_frame_off, ws_cnt, ws_list, ws_tap, n_taps, d_status);
  MP_CUDA_TRY(cudaGetLastError());
  if (A.F == 0) return MP_OK;
  const char* wm = knob("MP_GATHER_WAIT");   // experiment knob
  // default: plain try_wait loops (no suspend hint) — same-box A/B against
  // sleeping waits: c2 f32 alone 1.387 -> 1.374 ms, pipelined step 1.547 ->
  // 1.533 ms; u8 1.182 -> 1.175 ms; c4 unchanged
  A.wait_mode = wm ? atoi(wm) : 0;
  const char* stg = knob("MP_GATHER_STAGES");   // experiment knob
  // RGB24: three stages where they fit beside kSideReserve (f32 3 x 40 KB;
  // larger stages fall back to two below).  NV12: three when every class is
  // a fixed-tap class (~30-KB stages; c2 crops alone 1.247 -> 1.192 ms,
  // profiles/ab/r02_nv12_r43.jsonl), else two (3 x 40 KB measured slower for
  // the per-column NV12 consumer)
  bool all_r43 = true;
  for (int q = 0; q < A.k; q++) all_r43 = all_r43 && A.r43[q];
  A.stages = stg ? atoi(stg) : ((A.src == kSrcRGB24 || all_r43) ? kStagesF32 : kStages);
  if (A.stages < 2 || A.stages > kMaxStages) A.stages = kStages;
  // fewer stages when the ring would not leave kSideReserve of the SM's shared
  // memory to the latency-bound plan / remap-NMS CTAs of neighbouring batches
  // (they must co-run beside this persistent kernel, or they queue behind it
  // and serialise the pipeline), or when it does not fit at all (row-sparse
  // classes stage 96 KB: the proxy-input downscale keeps its 2 x 96 KB ring)
  bool any_r43 = false;   // fixed-tap classes stage their output rows per warp
  for (int q = 0; q < A.k; q++) any_r43 = any_r43 || A.r43[q];
  const size_t obuf_bytes = !any_r43 ? 0 : (fmt == MP_OUT_U8_NHWC ? (size_t)kR43BufBytes : (size_t)kR43FBufBytes);
  const size_t ring_cap = (2 * (size_t)A.stage_bytes + 4 * sizeof(uint64_t) + obuf_bytes <= 227 * 1024 - kSideReserve)
                              ? 227 * 1024 - kSideReserve : 227 * 1024;
#ifdef MP_LAM_SMEM
  const size_t lam_bytes = (size_t)cw_of(fmt, A.src) * kMaxNP * 32 * 8;
#else
  const size_t lam_bytes = 0;
#endif
  while (A.stages > 2 &&
         (size_t)A.stages * A.stage_bytes + 2 * A.stages * sizeof(uint64_t) + lam_bytes + obuf_bytes > ring_cap)
    A.stages--;
  A.lam_off = (int)(((size_t)A.stages * A.stage_bytes + 2 * A.stages * sizeof(uint64_t) + 15) & ~size_t(15));
  A.obuf_off = any_r43 ? (int)((A.lam_off + lam_bytes + 127) & ~size_t(127)) : 0;
  const size_t smem = any_r43 ? (size_t)A.obuf_off + obuf_bytes : (size_t)A.lam_off + lam_bytes;
  if (smem > 227 * 1024) return MP_ERR_UNSUPPORTED;
  int dev = 0, sms = 0, per_sm = 0;
  MP_CUDA_TRY(cudaGetDevice(&dev));
  // per-device SM count and per-(kernel, device) attribute/occupancy results
  // are cached: a steady-state call issues only the memset and two launches
  static std::atomic<int> sm_cache[64];
  if (dev >= 0 && dev < 64 && sm_cache[dev].load() > 0) {
    sms = sm_cache[dev].load();
  } else {
    MP_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (dev >= 0 && dev < 64) sm_cache[dev].store(sms);
  }
  // Diagnostic only (profiling the two halves of the pipeline): MP_GATHER_DEBUG=1
  // skips the consumer math, =2 skips the pixel copies.  Unset in production.
  const char* dbg = knob("MP_GATHER_DEBUG");
  A.debug = dbg ? atoi(dbg) : 0;
  const int threads = (cw_of(fmt, A.src) + kProducerWarps) * 32;
  auto launch = [&](auto kern) -> mp_status {
    // cache key: kernel instance x device x dynamic shared memory
    struct Occ {
      const void* fn;
      int dev;
      size_t smem;
      int per_sm;
    };
    static Occ occ_cache[32];
    static int occ_n = 0;
    static size_t attr_max[64][4];   // largest MaxDynamicSharedMemorySize set per (device, instance)
    static std::mutex mu;            // callers may enqueue from several host threads
    std::lock_guard<std::mutex> lock(mu);
    const int inst = (A.src == kSrcNV12 ? 2 : 0) + (fmt == MP_OUT_F32_NCHW ? 0 : 1);
    per_sm = 0;
    for (int i = 0; i < occ_n; i++)
      if (occ_cache[i].fn == (const void*)kern && occ_cache[i].dev == dev && occ_cache[i].smem == smem)
        per_sm = occ_cache[i].per_sm;
    MP_CUDA_TRY(prefer_max_shared((const void*)kern));
    if (dev < 0 || dev >= 64 || attr_max[dev][inst] < smem) {
      MP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      if (dev >= 0 && dev < 64) attr_max[dev][inst] = smem;
    }
    if (per_sm == 0) {
      MP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
      if (per_sm < 1) per_sm = 1;
      if (occ_n < 32) occ_cache[occ_n++] = Occ{(const void*)kern, dev, smem, per_sm};
    }
    // mp_gather_set_sm_reserve: SMs left to the co-running planner
    const int rsv = g_sm_reserve.load(std::memory_order_relaxed);
    const int gsms = rsv < sms ? sms - rsv : 1;
    kern<<<gsms * per_sm, threads, smem, s>>>(A, tm, d_frame_ptrs, ws_cnt, ws_list, d_windows, d_frame_off, ws_tap,
                                             d_status);
    MP_CUDA_TRY(cudaGetLastError());
    return MP_OK;
  };
  if (A.src == kSrcNV12)
    return fmt == MP_OUT_F32_NCHW ? launch(gather_kernel<MP_OUT_F32_NCHW, kSrcNV12>)
                                  : launch(gather_kernel<MP_OUT_U8_NHWC, kSrcNV12>);
  return fmt == MP_OUT_F32_NCHW ? launch(gather_kernel<MP_OUT_F32_NCHW, kSrcRGB24>)
                                : launch(gather_kernel<MP_OUT_U8_NHWC, kSrcRGB24>);
}

extern "C" mp_status mp_gather_resize(const uint8_t* const* d_frame_ptrs, int32_t pitch, int32_t W, int32_t H,
                                      int32_t F, const mp_window* d_windows, const int32_t* d_frame_off,
                                      int32_t max_windows, int32_t k, const mp_size* sizes, const mp_size* out_dims,
                                      void* const* d_out, const int32_t* out_cap, mp_out_format fmt,
                                      int32_t* d_status, void* d_ws, size_t ws_bytes, void* stream) {
  GatherArgs A;
  if (!build_gather_args(kSrcRGB24, false, pitch, W, H, F, k, sizes, out_dims, d_out, out_cap, fmt, &A))
    return MP_ERR_INVALID;
  if (!d_frame_off || !d_status || (F > 0 && (!d_frame_ptrs || (max_windows > 0 && !d_windows))))
    return MP_ERR_INVALID;
  if (max_windows < 0) return MP_ERR_INVALID;
  A.max_windows = max_windows;
  TmapArray tm;
  memset(&tm, 0, sizeof(tm));
  A.tensor = 0;
  return gather_launch(A, tm, d_frame_ptrs, d_windows, d_frame_off, k, out_dims, out_cap, fmt, d_status, d_ws,
                       ws_bytes, stream);
}

static EncodeTiledFn get_encode() {
  static std::atomic<EncodeTiledFn> cached{nullptr};   // the driver entry point does not change
  if (EncodeTiledFn c = cached.load()) return c;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) != cudaSuccess ||
      qr != cudaDriverEntryPointSuccess || !fn) {
    (void)cudaGetLastError();
    return nullptr;
  }
  cached.store((EncodeTiledFn)fn);
  return (EncodeTiledFn)fn;
}

// A plane batch as a 3-D tensor of 8-byte elements [F][rows][pitch/8]; box =
// one class's staged footprint.  Rows past the plane bottom and bytes past the
// pitch are zero-filled by the copy engine.
static bool encode_plane(EncodeTiledFn encode, CUtensorMap* m, const void* base, int pitch, int rows, int F,
                         int64_t frame_stride, int box_w, int box_h) {
  const cuuint64_t gdim[3] = {(cuuint64_t)(pitch / 8), (cuuint64_t)rows, (cuuint64_t)F};
  const cuuint64_t gstride[2] = {(cuuint64_t)pitch, (cuuint64_t)frame_stride};
  const cuuint32_t box[3] = {(cuuint32_t)(box_w / 8), (cuuint32_t)box_h, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  // measured on B200: 64-B L2 promotion beats none / 128 B / 256 B for these ~0.8 KB box rows
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<void*>(base), gdim, gstride, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The frame batch as a 2-D tensor of rows [F * rpf][pitch/8] (rpf = rows per
// frame = frame_stride / pitch) with a one-row box of box_w bytes: the view
// the tile::gather4 row gathers of row-sparse classes index.
static bool encode_rows(EncodeTiledFn encode, CUtensorMap* m, const void* base, int pitch, int64_t total_rows,
                        int box_w) {
  const cuuint64_t gdim[2] = {(cuuint64_t)(pitch / 8), (cuuint64_t)total_rows};
  const cuuint64_t gstride[1] = {(cuuint64_t)pitch};
  const cuuint32_t box[2] = {(cuuint32_t)(box_w / 8), 1};
  const cuuint32_t estr[2] = {1, 1};
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void*>(base), gdim, gstride, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Row-sparse staging needs the 2-D row view: frame_stride a multiple of pitch.
static bool row_view_ok(int64_t frame_stride, int pitch, int F) {
  return pitch > 0 && frame_stride > 0 && frame_stride % pitch == 0 &&
         (int64_t)F * (frame_stride / pitch) < (int64_t(1) << 31);
}

extern "C" mp_status mp_gather_resize_strided(const uint8_t* d_frames, int64_t frame_stride, int32_t pitch,
                                              int32_t W, int32_t H, int32_t F, const mp_window* d_windows,
                                              const int32_t* d_frame_off, int32_t max_windows, int32_t k,
                                              const mp_size* sizes,
                                              const mp_size* out_dims, void* const* d_out, const int32_t* out_cap,
                                              mp_out_format fmt, int32_t* d_status, void* d_ws, size_t ws_bytes,
                                              void* stream) {
  GatherArgs A;
  const bool rows = row_view_ok(frame_stride, pitch, F);
  if (!build_gather_args(kSrcRGB24, rows, pitch, W, H, F, k, sizes, out_dims, d_out, out_cap, fmt, &A))
    return MP_ERR_INVALID;
  A.rpf = rows ? (int)(frame_stride / pitch) : 0;
  if (!d_frame_off || !d_status || (F > 0 && (!d_frames || (max_windows > 0 && !d_windows))))
    return MP_ERR_INVALID;
  if (max_windows < 0) return MP_ERR_INVALID;
  A.max_windows = max_windows;
  if (F > 0 && (((uintptr_t)d_frames) & 15)) return MP_ERR_INVALID;
  if (frame_stride < (int64_t)H * pitch || (frame_stride & 15) || frame_stride >= (int64_t(1) << 40))
    return MP_ERR_INVALID;
  TmapArray tm;
  memset(&tm, 0, sizeof(tm));
  A.tensor = 1;
  if (F > 0) {
    EncodeTiledFn encode = get_encode();
    if (!encode) return MP_ERR_CUDA;
    for (int q = 0; q < k; q++) {
      const bool ok = A.sparse[q]
                          ? encode_rows(encode, &tm.m[q], d_frames, pitch, (int64_t)F * A.rpf, A.box_w[q])
                          : encode_plane(encode, &tm.m[q], d_frames, pitch, H, F, frame_stride, A.box_w[q],
                                         A.box_h[q]);
      if (!ok) return MP_ERR_UNSUPPORTED;
    }
  }
  return gather_launch(A, tm, nullptr, d_windows, d_frame_off, k, out_dims, out_cap, fmt, d_status, d_ws,
                       ws_bytes, stream);
}

// R23 conversion coefficients from the BT.601 / BT.709 definitions (computed in
// fp64, rounded once to fp32): out = cy*Y - cy*yo + {crv*(V-128); cgu*(U-128)
// + cgv*(V-128); cbu*(U-128)}.
static bool nv12_coefficients(int matrix, float* c) {
  if (matrix < MP_BT709_LIMITED || matrix > MP_BT601_FULL) return false;
  const bool bt601 = matrix == MP_BT601_LIMITED || matrix == MP_BT601_FULL;
  const bool full = matrix == MP_BT709_FULL || matrix == MP_BT601_FULL;
  const double Kr = bt601 ? 0.299 : 0.2126, Kb = bt601 ? 0.114 : 0.0722, Kg = 1.0 - Kr - Kb;
  const double yo = full ? 0.0 : 16.0, ys = full ? 255.0 : 219.0, cs = full ? 255.0 : 224.0;
  const double cy = 255.0 / ys;
  c[0] = (float)cy;
  c[1] = (float)(-cy * yo);
  c[2] = (float)(255.0 * 2.0 * (1.0 - Kr) / cs);
  c[3] = (float)(-255.0 * 2.0 * Kb * (1.0 - Kb) / (Kg * cs));
  c[4] = (float)(-255.0 * 2.0 * Kr * (1.0 - Kr) / (Kg * cs));
  c[5] = (float)(255.0 * 2.0 * (1.0 - Kb) / cs);
  return true;
}

extern "C" mp_status mp_gather_resize_nv12(const uint8_t* d_frames, int64_t frame_stride, int32_t pitch, int32_t W,
                                           int32_t H, int32_t F, const mp_window* d_windows,
                                           const int32_t* d_frame_off, int32_t max_windows, int32_t k,
                                           const mp_size* sizes,
                                           const mp_size* out_dims, void* const* d_out, const int32_t* out_cap,
                                           mp_out_format fmt, mp_color_matrix matrix, int32_t* d_status,
                                           void* d_ws, size_t ws_bytes, void* stream) {
  GatherArgs A;
  const bool rows = row_view_ok(frame_stride, pitch, F);
  if (!build_gather_args(kSrcNV12, rows, pitch, W, H, F, k, sizes, out_dims, d_out, out_cap, fmt, &A))
    return MP_ERR_INVALID;
  A.rpf = rows ? (int)(frame_stride / pitch) : 0;
  if (!nv12_coefficients((int)matrix, A.cvt)) return MP_ERR_INVALID;
  if (!d_frame_off || !d_status || (F > 0 && (!d_frames || (max_windows > 0 && !d_windows))))
    return MP_ERR_INVALID;
  if (max_windows < 0) return MP_ERR_INVALID;
  A.max_windows = max_windows;
  if (F > 0 && (((uintptr_t)d_frames) & 15)) return MP_ERR_INVALID;
  if (frame_stride < (int64_t)(H + H / 2) * pitch || (frame_stride & 15) || frame_stride >= (int64_t(1) << 40))
    return MP_ERR_INVALID;
  TmapArray tm;
  memset(&tm, 0, sizeof(tm));
  A.tensor = 1;
  if (F > 0) {
    EncodeTiledFn encode = get_encode();
    if (!encode) return MP_ERR_CUDA;
    const uint8_t* uv = d_frames + (size_t)H * pitch;
    for (int q = 0; q < k; q++) {
      const bool ok =
          A.sparse[q] ? encode_rows(encode, &tm.m[q], d_frames, pitch, (int64_t)F * A.rpf, A.box_w[q])
                      : (encode_plane(encode, &tm.m[q], d_frames, pitch, H, F, frame_stride, A.box_w[q],
                                      A.box_h[q]) &&
                         encode_plane(encode, &tm.m[kMaxClasses + q], uv, pitch, H / 2, F, frame_stride,
                                      A.box_w[q], A.box_huv[q]));
      if (!ok) return MP_ERR_UNSUPPORTED;
    }
  }
  return gather_launch(A, tm, nullptr, d_windows, d_frame_off, k, out_dims, out_cap, fmt, d_status, d_ws,
                       ws_bytes, stream);
}
