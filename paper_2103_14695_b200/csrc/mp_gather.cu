// mp_gather.cu — step a5: gather every window's crop from its full-resolution
// RGB24 frame and bilinearly resample it to its size class's detector-input
// dims (PAPER.md:152 — the detector runs batched "at each of those sizes";
// resampling convention R15/R16 in DESIGN.md §3).  HBM-bound: this kernel
// carries ~99% of the path's bytes.
//
// Launches:
//   gather_prep_kernel   one CTA: validate windows (n_win read on device),
//                        count windows per class, build per-class slot ->
//                        window descriptors (crop origin pointer, x), and the
//                        per-class exact integer tap tables (i0, lambda) for
//                        both axes (R15).
//   gather_kernel<fmt>   persistent, warp-specialised, Grid = SMs x resident
//                        CTAs.  Warps 8-9 = producers (alternate tiles): one
//                        descriptor + 4 tap loads per tile, copy the tile's tap
//                        slices into the stage header, then 1-D bulk copies
//                        (TMA engine, cp.async.bulk) of the tile's source rows
//                        into a 4-deep shared-memory stage ring completing on an
//                        mbarrier (complete_tx).  Warps 0-7 = consumers: two
//                        output columns per thread (packed f32x2 math),
//                        separable lerps reusing staged rows, streaming stores.
#include "mp_internal.cuh"

namespace mpk {

constexpr int kConsumerWarps = 8;
constexpr int kProducerWarps = 2;
constexpr int kGatherThreads = (kConsumerWarps + kProducerWarps) * 32;
constexpr int kStages = 4;
constexpr int kHdrBytes = 64;
constexpr int kMaxTW = 256;
constexpr int kMaxTR = 64;
constexpr int kTapBytes = kMaxTW * 8 + kMaxTR * 16;
constexpr int kStageDataBudget = 24 * 1024;

struct GatherArgs {
  int k, W, H, pitch, F, fmt, stage_bytes;
  int w[kMaxClasses], h[kMaxClasses], ow[kMaxClasses], oh[kMaxClasses];
  int TW[kMaxClasses], TR[kMaxClasses], nct[kMaxClasses], tpw[kMaxClasses];
  int cap[kMaxClasses], list_off[kMaxClasses], xtab_off[kMaxClasses], ytab_off[kMaxClasses];
  void* out[kMaxClasses];
};

// Per listed window: pointer to the crop's first row (frame + y*pitch), x, slot.
struct WinDesc {
  const uint8_t* row0;
  int x, valid;
};
static_assert(sizeof(WinDesc) == 16, "desc");

struct TileHdr {
  int valid, k, slot, oy0, ox0, rows, cols, stride;
  int pad[8];
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

__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {   // packed a - b (FADD2 with negated operand)
  return __fadd2_rn(a, make_float2(-b.x, -b.y));
}

// u8 -> (2^23 + u8) as an fp32 bit pattern; subtracting 2^23 afterwards is exact.
__device__ __forceinline__ float u8m(uint32_t b) { return __int_as_float(0x4B000000u + b); }

__device__ __forceinline__ uint8_t u8_round(float v) {   // R16: floor(v + 0.5), clamped
  const int r = __float2int_rd(v + 0.5f);
  return (uint8_t)min(max(r, 0), 255);
}

__device__ __forceinline__ int tiles_total(const GatherArgs& A, const int* cnt) {
  int T = 0;
  for (int q = 0; q < A.k; q++) T += min(cnt[q], A.cap[q]) * A.tpw[q];
  return T;
}

__global__ void __launch_bounds__(1024) gather_prep_kernel(GatherArgs A, const uint8_t* const* __restrict__ frames,
                                                           const mp_window* __restrict__ win,
                                                           const int* __restrict__ frame_off,
                                                           int* __restrict__ ws_cnt, WinDesc* __restrict__ ws_desc,
                                                           int2* __restrict__ ws_tap, int desc_total,
                                                           int* __restrict__ d_status) {
  __shared__ int cnt[kMaxClasses];
  if (threadIdx.x < kMaxClasses) cnt[threadIdx.x] = 0;
  for (int i = threadIdx.x; i < desc_total; i += blockDim.x) ws_desc[i] = WinDesc{nullptr, 0, 0};
  // tap tables: x taps of class q at xtab_off[q] (ow entries), y taps at ytab_off[q]
  for (int q = 0; q < A.k; q++) {
    for (int d = threadIdx.x; d < A.ow[q]; d += blockDim.x) {
      int i0; float lam;
      tap(A.w[q], A.ow[q], d, i0, lam);
      ws_tap[A.xtab_off[q] + d] = make_int2(i0, __float_as_int(lam));
    }
    for (int d = threadIdx.x; d < A.oh[q]; d += blockDim.x) {
      int i0; float lam;
      tap(A.h[q], A.oh[q], d, i0, lam);
      ws_tap[A.ytab_off[q] + d] = make_int2(i0, __float_as_int(lam));
    }
  }
  __syncthreads();
  const int n_win = frame_off[A.F];
  for (int i = threadIdx.x; i < n_win; i += blockDim.x) {
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
    ws_desc[A.list_off[q] + w.slot] = WinDesc{frames[w.frame] + (size_t)w.y * A.pitch, w.x, 1};
  }
  __syncthreads();
  if (threadIdx.x < kMaxClasses) ws_cnt[threadIdx.x] = cnt[threadIdx.x];
}

template <int FMT>
__global__ void __launch_bounds__(kGatherThreads) gather_kernel(GatherArgs A, const int* __restrict__ ws_cnt,
                                                                 const WinDesc* __restrict__ ws_desc,
                                                                 const int2* __restrict__ ws_tap,
                                                                 int* __restrict__ d_status) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)kStages * A.stage_bytes);
  uint64_t* empty = full + kStages;
  __shared__ int cnt[kMaxClasses];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid < kMaxClasses) cnt[tid] = tid < A.k ? ws_cnt[tid] : 0;
  if (tid == 0) {
    for (int s = 0; s < kStages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int T = tiles_total(A, cnt);
  const int G = gridDim.x;

  if (wid >= kConsumerWarps) {
    // ===================== producer warps (tiles i = p, p+2, ...) =====================
    const int p = wid - kConsumerWarps;
    for (int i = p;; i += kProducerWarps) {
      const int t = blockIdx.x + i * G;
      if (t >= T) break;
      const int s = i % kStages;
      if (i >= kStages) mbar_wait(&empty[s], ((i / kStages) - 1) & 1);
      unsigned char* stage = smem + (size_t)s * A.stage_bytes;
      TileHdr* hdr = reinterpret_cast<TileHdr*>(stage);
      int2* xt = reinterpret_cast<int2*>(stage + kHdrBytes);
      int4* yt = reinterpret_cast<int4*>(stage + kHdrBytes + kMaxTW * 8);
      unsigned char* data = stage + kHdrBytes + kTapBytes;
      // decode t -> (class, slot, row tile, col tile); tiles ordered by class,
      // slot, then tile, so neighbouring CTAs share halo rows in L2.
      int q = 0, rel = t;
      while (rel >= min(cnt[q], A.cap[q]) * A.tpw[q]) {
        rel -= min(cnt[q], A.cap[q]) * A.tpw[q];
        q++;
      }
      const int slot = rel / A.tpw[q];
      const int tw = rel - slot * A.tpw[q];
      const int rt = tw / A.nct[q], ct = tw - rt * A.nct[q];
      const int in_w = A.w[q], in_h = A.h[q];
      const int oy0 = rt * A.TR[q], ox0 = ct * A.TW[q];
      const int rows = min(A.TR[q], A.oh[q] - oy0), cols = min(A.TW[q], A.ow[q] - ox0);
      const int2* xtab = ws_tap + A.xtab_off[q];
      const int2* ytab = ws_tap + A.ytab_off[q];
      const WinDesc d = ws_desc[A.list_off[q] + slot];
      const int c_lo = __ldg(&xtab[ox0].x), c_hi = min(__ldg(&xtab[ox0 + cols - 1].x) + 1, in_w - 1);
      const int r_lo = __ldg(&ytab[oy0].x), r_hi = min(__ldg(&ytab[oy0 + rows - 1].x) + 1, in_h - 1);
      if (!d.valid) {   // slots of this class are not 0..count-1
        if (lane == 0) {
          hdr->valid = 0;
          set_status(d_status, MP_ERR_INVALID);
          mbar_arrive(&full[s]);
        }
        __syncwarp();
        continue;
      }
      const int b0 = (3 * (d.x + c_lo)) & ~15;
      const int b1 = (3 * (d.x + c_hi + 1) + 15) & ~15;
      const int stride = b1 - b0;
      const int nrows = r_hi - r_lo + 1;
      for (int c = lane; c < cols; c += 32) {
        const int2 e = __ldg(&xtab[ox0 + c]);
        const int di = (e.x < in_w - 1) ? 3 : 0;
        xt[c] = make_int2((3 * (d.x + e.x) - b0) | (di << 20), e.y);
      }
      for (int r = lane; r < rows; r += 32) {
        const int2 e = __ldg(&ytab[oy0 + r]);
        const int i1 = min(e.x + 1, in_h - 1);
        yt[r] = make_int4((e.x - r_lo) * stride, (i1 - r_lo) * stride, e.y, 0);
      }
      if (lane == 0) {
        hdr->valid = 1;
        hdr->k = q;
        hdr->slot = slot;
        hdr->oy0 = oy0;
        hdr->ox0 = ox0;
        hdr->rows = rows;
        hdr->cols = cols;
        hdr->stride = stride;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&full[s], (uint32_t)(nrows * stride));
      __syncwarp();
      const uint8_t* src = d.row0 + (size_t)r_lo * A.pitch + b0;
      for (int r = lane; r < nrows; r += 32)
        bulk_g2s(data + (size_t)r * stride, src + (size_t)r * A.pitch, (uint32_t)stride, &full[s]);
    }
    return;
  }

  // ===================== consumer warps =====================
  // Thread <-> two output columns of the tile, c and c + half (consecutive
  // lanes = consecutive columns: conflict-free byte loads, coalesced stores;
  // the pair shares one packed f32x2 datapath), and a contiguous block of rows.
  // Separable evaluation: the horizontal lerp of a staged source row is
  // computed once and reused by the next output row that taps the same row.
  const int ctid = tid;   // 0 .. 32*kConsumerWarps-1
  const float2 M2 = make_float2(8388608.0f, 8388608.0f);
  for (int i = 0;; i++) {
    const int t = blockIdx.x + i * G;
    if (t >= T) break;
    const int s = i % kStages;
    mbar_wait(&full[s], (i / kStages) & 1);
    const unsigned int soff = (unsigned int)s * (unsigned int)A.stage_bytes;
    const TileHdr* hdr = reinterpret_cast<const TileHdr*>(&smem[soff]);
    if (hdr->valid) {
      const int2* xt = reinterpret_cast<const int2*>(&smem[soff + kHdrBytes]);
      const int4* yt = reinterpret_cast<const int4*>(&smem[soff + kHdrBytes + kMaxTW * 8]);
      const unsigned int doff = soff + kHdrBytes + kTapBytes;
      const int q = hdr->k, rows = hdr->rows, cols = hdr->cols;
      const int half = (cols + 1) >> 1;
      const int nph = max(1, (32 * kConsumerWarps) / half);
      const int ph = ctid / half, c = ctid - ph * half;
      if (ph < nph) {
        const int rpp = (rows + nph - 1) / nph;
        const int rb0 = ph * rpp, rb1 = min(rows, rb0 + rpp);
        const bool two = (c + half) < cols;
        const int2 xa = xt[c];
        const int2 xb = two ? xt[c + half] : xa;
        const unsigned int ba = doff + (xa.x & 0xFFFFF), bb = doff + (xb.x & 0xFFFFF);
        const unsigned int da = ba + (xa.x >> 20), db = bb + (xb.x >> 20);
        const float2 lx = make_float2(__int_as_float(xa.y), __int_as_float(xb.y));
        const int ow = A.ow[q], oh = A.oh[q];
        int ra = -1, rb = -1;
        float2 ha0, ha1, ha2, hb0, hb1, hb2;
#define MP_HLERP(ROWOFF, H0, H1, H2)                                                          \
  {                                                                                           \
    const unsigned int o_ = (unsigned int)(ROWOFF);                                           \
    float2 m_, n_;                                                                            \
    m_ = make_float2(u8m(smem[ba + o_ + 0]), u8m(smem[bb + o_ + 0]));                          \
    n_ = make_float2(u8m(smem[da + o_ + 0]), u8m(smem[db + o_ + 0]));                          \
    H0 = __ffma2_rn(lx, fsub2(n_, m_), fsub2(m_, M2));                               \
    m_ = make_float2(u8m(smem[ba + o_ + 1]), u8m(smem[bb + o_ + 1]));                          \
    n_ = make_float2(u8m(smem[da + o_ + 1]), u8m(smem[db + o_ + 1]));                          \
    H1 = __ffma2_rn(lx, fsub2(n_, m_), fsub2(m_, M2));                               \
    m_ = make_float2(u8m(smem[ba + o_ + 2]), u8m(smem[bb + o_ + 2]));                          \
    n_ = make_float2(u8m(smem[da + o_ + 2]), u8m(smem[db + o_ + 2]));                          \
    H2 = __ffma2_rn(lx, fsub2(n_, m_), fsub2(m_, M2));                               \
  }
        if (FMT == MP_OUT_F32_NCHW) {
          const int plane = oh * ow;
          float* o = reinterpret_cast<float*>(A.out[q]) + (size_t)hdr->slot * 3 * plane +
                     (size_t)(hdr->oy0 + rb0) * ow + hdr->ox0 + c;
          for (int r = rb0; r < rb1; r++) {
            const int4 y = yt[r];
            if (y.x != ra) {
              if (y.x == rb) { ha0 = hb0; ha1 = hb1; ha2 = hb2; }
              else MP_HLERP(y.x, ha0, ha1, ha2)
              ra = y.x;
            }
            if (y.y != rb) {
              if (y.y == ra) { hb0 = ha0; hb1 = ha1; hb2 = ha2; }
              else MP_HLERP(y.y, hb0, hb1, hb2)
              rb = y.y;
            }
            const float2 ly = make_float2(__int_as_float(y.z), __int_as_float(y.z));
            const float2 v0 = __ffma2_rn(ly, fsub2(hb0, ha0), ha0);
            const float2 v1 = __ffma2_rn(ly, fsub2(hb1, ha1), ha1);
            const float2 v2 = __ffma2_rn(ly, fsub2(hb2, ha2), ha2);
            __stcs(o, v0.x);
            __stcs(o + plane, v1.x);
            __stcs(o + 2 * plane, v2.x);
            if (two) {
              __stcs(o + half, v0.y);
              __stcs(o + plane + half, v1.y);
              __stcs(o + 2 * plane + half, v2.y);
            }
            o += ow;
          }
        } else {
          uint8_t* o = reinterpret_cast<uint8_t*>(A.out[q]) +
                       (((size_t)hdr->slot * oh + hdr->oy0 + rb0) * ow + hdr->ox0 + c) * 3;
          for (int r = rb0; r < rb1; r++) {
            const int4 y = yt[r];
            if (y.x != ra) {
              if (y.x == rb) { ha0 = hb0; ha1 = hb1; ha2 = hb2; }
              else MP_HLERP(y.x, ha0, ha1, ha2)
              ra = y.x;
            }
            if (y.y != rb) {
              if (y.y == ra) { hb0 = ha0; hb1 = ha1; hb2 = ha2; }
              else MP_HLERP(y.y, hb0, hb1, hb2)
              rb = y.y;
            }
            const float2 ly = make_float2(__int_as_float(y.z), __int_as_float(y.z));
            const float2 v0 = __ffma2_rn(ly, fsub2(hb0, ha0), ha0);
            const float2 v1 = __ffma2_rn(ly, fsub2(hb1, ha1), ha1);
            const float2 v2 = __ffma2_rn(ly, fsub2(hb2, ha2), ha2);
            o[0] = u8_round(v0.x);   // R16 round half up, clamp
            o[1] = u8_round(v1.x);
            o[2] = u8_round(v2.x);
            if (two) {
              o[3 * half + 0] = u8_round(v0.y);
              o[3 * half + 1] = u8_round(v1.y);
              o[3 * half + 2] = u8_round(v2.y);
            }
            o += (size_t)ow * 3;
          }
        }
#undef MP_HLERP
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
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

// Largest staged footprint (bytes) of any tile of a class with tile dims (TW, TR).
static long long class_stage_data(int in_w, int in_h, int ow, int oh, int TW, int TR) {
  long long best = 0;
  int nct = (ow + TW - 1) / TW, nrt = (oh + TR - 1) / TR;
  int max_rows = 0, max_cols = 0, a, b, c, d;
  for (int rt = 0; rt < nrt; rt++) {
    int oy0 = rt * TR, rows = (TR < oh - oy0 ? TR : oh - oy0);
    host_tap(in_h, oh, oy0, &a, &b);
    host_tap(in_h, oh, oy0 + rows - 1, &c, &d);
    if (d - a + 1 > max_rows) max_rows = d - a + 1;
  }
  for (int ct = 0; ct < nct; ct++) {
    int ox0 = ct * TW, cols = (TW < ow - ox0 ? TW : ow - ox0);
    host_tap(in_w, ow, ox0, &a, &b);
    host_tap(in_w, ow, ox0 + cols - 1, &c, &d);
    if (d - a + 1 > max_cols) max_cols = d - a + 1;
  }
  long long stride = ((3LL * max_cols + 30) + 15) / 16 * 16;
  best = stride * max_rows;
  return best;
}

static bool build_gather_args(int pitch, int W, int H, int F, int k, const mp_size* sizes,
                              const mp_size* out_dims, void* const* d_out, const int32_t* out_cap,
                              mp_out_format fmt, GatherArgs* A) {
  if (W < 1 || H < 1 || W > 16384 || H > 16384 || F < 0 || k < 1 || k > kMaxClasses) return false;
  if (pitch < 3 * W || (pitch & 15)) return false;
  if (!sizes || !out_dims || !d_out || !out_cap) return false;
  if (fmt != MP_OUT_F32_NCHW && fmt != MP_OUT_U8_NHWC) return false;
  memset(A, 0, sizeof(*A));
  A->k = k;
  A->W = W;
  A->H = H;
  A->pitch = pitch;
  A->F = F;
  A->fmt = fmt;
  long long data_max = 0;
  int list = 0, taps = 0;
  for (int q = 0; q < k; q++) {
    const int w = sizes[q].w, h = sizes[q].h, ow = out_dims[q].w, oh = out_dims[q].h;
    if (w < 1 || h < 1 || w > W || h > H || ow < 1 || oh < 1 || ow > 16384 || oh > 16384) return false;
    if (out_cap[q] < 0 || (out_cap[q] > 0 && !d_out[q])) return false;
    if (((uintptr_t)d_out[q]) & 15) return false;
    A->w[q] = w;
    A->h[q] = h;
    A->ow[q] = ow;
    A->oh[q] = oh;
    // tile width: a power of two <= 256 (so 256 consumer threads split into
    // whole column phases), height so a tile is ~4K output pixels
    int TW = 256;
    while (TW > 32 && TW > ow) TW >>= 1;
    int TR = 4096 / TW;
    if (TR > kMaxTR) TR = kMaxTR;
    long long dat = class_stage_data(w, h, ow, oh, TW, TR);
    while (dat > kStageDataBudget && TR > 1) {
      TR = TR - 1;
      dat = class_stage_data(w, h, ow, oh, TW, TR);
    }
    while (dat > kStageDataBudget && TW > 32) {
      TW >>= 1;
      dat = class_stage_data(w, h, ow, oh, TW, TR);
    }
    if (dat > 4 * kStageDataBudget) return false;   // > 32x downscale: unsupported
    A->TW[q] = TW;
    A->TR[q] = TR;
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
    if (dat > data_max) data_max = dat;
  }
  A->stage_bytes = (int)(((kHdrBytes + kTapBytes + data_max) + 127) / 128 * 128);
  return true;
}

}  // namespace mpk

using namespace mpk;

struct GatherWs {
  size_t cnt_off, desc_off, tap_off, total;
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
  L->desc_off = 256;
  L->tap_off = al(L->desc_off + desc * sizeof(WinDesc));
  L->total = al(L->tap_off + taps * sizeof(int2));
  return true;
}

extern "C" size_t mp_gather_workspace_size(int32_t k, const mp_size* out_dims, const int32_t* out_cap) {
  GatherWs L;
  return gather_ws_layout(k, out_dims, out_cap, &L) ? L.total : 0;
}

extern "C" mp_status mp_gather_resize(const uint8_t* const* d_frame_ptrs, int32_t pitch, int32_t W, int32_t H,
                                      int32_t F, const mp_window* d_windows, const int32_t* d_frame_off,
                                      int32_t k, const mp_size* sizes, const mp_size* out_dims,
                                      void* const* d_out, const int32_t* out_cap, mp_out_format fmt,
                                      int32_t* d_status, void* d_ws, size_t ws_bytes, void* stream) {
  GatherArgs A;
  if (!build_gather_args(pitch, W, H, F, k, sizes, out_dims, d_out, out_cap, fmt, &A)) return MP_ERR_INVALID;
  if (!d_frame_off || !d_status || (F > 0 && (!d_frame_ptrs || !d_windows))) return MP_ERR_INVALID;
  GatherWs L;
  if (!gather_ws_layout(k, out_dims, out_cap, &L) || !d_ws || ws_bytes < L.total) return MP_ERR_INVALID;
  int desc_total = 0;
  for (int q = 0; q < k; q++) desc_total += out_cap[q];
  cudaStream_t s = (cudaStream_t)stream;
  unsigned char* ws = (unsigned char*)d_ws;
  int* ws_cnt = (int*)(ws + L.cnt_off);
  WinDesc* ws_desc = (WinDesc*)(ws + L.desc_off);
  int2* ws_tap = (int2*)(ws + L.tap_off);
  gather_prep_kernel<<<1, 1024, 0, s>>>(A, d_frame_ptrs, d_windows, d_frame_off, ws_cnt, ws_desc, ws_tap, desc_total,
                                        d_status);
  MP_CUDA_TRY(cudaGetLastError());
  if (F == 0) return MP_OK;
  const size_t smem = (size_t)kStages * A.stage_bytes + 2 * kStages * sizeof(uint64_t);
  if (smem > 227 * 1024) return MP_ERR_UNSUPPORTED;
  int dev = 0, sms = 0, per_sm = 0;
  MP_CUDA_TRY(cudaGetDevice(&dev));
  MP_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  auto launch = [&](auto kern) -> mp_status {
    MP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    MP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kGatherThreads, smem));
    if (per_sm < 1) per_sm = 1;
    kern<<<sms * per_sm, kGatherThreads, smem, s>>>(A, ws_cnt, ws_desc, ws_tap, d_status);
    MP_CUDA_TRY(cudaGetLastError());
    return MP_OK;
  };
  return fmt == MP_OUT_F32_NCHW ? launch(gather_kernel<MP_OUT_F32_NCHW>) : launch(gather_kernel<MP_OUT_U8_NHWC>);
}
