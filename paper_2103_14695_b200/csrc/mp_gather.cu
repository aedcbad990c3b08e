// mp_gather.cu — step a5: gather every window's crop from its full-resolution
// RGB24 frame and bilinearly resample it to its size class's detector-input
// dims (PAPER.md:152 — the detector runs batched "at each of those sizes";
// resampling convention R15/R16 in DESIGN.md §3).  HBM-bound: this kernel
// carries ~99% of the path's bytes.
//
// Launches:
//   gather_prep_kernel   one CTA: validate windows, build per-class slot->window
//                        lists, count windows per class (reads n_win on device)
//   gather_kernel<fmt>   persistent, warp-specialised: warp 8 = producer
//                        (decodes tile, computes exact integer taps, issues 1-D
//                        bulk copies of the tile's source rows into a shared-
//                        memory stage ring, mbarrier complete_tx); warps 0-7 =
//                        consumers (bilinear taps from shared memory, streaming
//                        coalesced stores).  Grid = SMs x resident CTAs.
#include "mp_internal.cuh"

namespace mpk {

constexpr int kConsumerWarps = 8;
constexpr int kGatherThreads = (kConsumerWarps + 1) * 32;
constexpr int kStages = 3;
constexpr int kHdrBytes = 64;
constexpr int kMaxTW = 256;
constexpr int kMaxTR = 128;
constexpr int kTapBytes = kMaxTW * 8 + kMaxTR * 16;
constexpr int kStageDataBudget = 32 * 1024;

struct GatherArgs {
  int k, W, H, pitch, F, fmt, stage_bytes;
  int w[kMaxClasses], h[kMaxClasses], ow[kMaxClasses], oh[kMaxClasses];
  int TW[kMaxClasses], TR[kMaxClasses], nct[kMaxClasses], tpw[kMaxClasses];
  int cap[kMaxClasses], list_off[kMaxClasses];
  void* out[kMaxClasses];
};

struct TileHdr {
  const uint8_t* src;   // unused by consumers (debug)
  int valid, k, slot, oy0, ox0, rows, cols, stride;
  int pad[4];
};
static_assert(sizeof(TileHdr) <= kHdrBytes, "header");

// R15 exact integer taps: n = (2d+1)*in - out; i0 = floor(n / 2out) (n<0 -> 0),
// lambda = (n mod 2out) / 2out (fp32 of exact integers, one rounding);
// i0 >= in-1 -> (in-1, 0); i1 = min(i0+1, in-1).
__device__ __forceinline__ void tap(int in, int out, int d, int& i0, int& i1, float& lam) {
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
  i1 = min(a + 1, in - 1);
  lam = __fdiv_rn((float)rem, (float)(2 * out));
}

__device__ __forceinline__ float u8f(uint32_t b) {   // exact u8 -> f32 via the 2^23 magic
  return __int_as_float(0x4B000000u | b) - 8388608.0f;
}

__device__ __forceinline__ int tiles_total(const GatherArgs& A, const int* cnt) {
  int T = 0;
  for (int q = 0; q < A.k; q++) T += min(cnt[q], A.cap[q]) * A.tpw[q];
  return T;
}

__global__ void __launch_bounds__(1024) gather_prep_kernel(GatherArgs A, const mp_window* __restrict__ win,
                                                           const int* __restrict__ frame_off,
                                                           int* __restrict__ ws_cnt, int* __restrict__ ws_list,
                                                           int list_total, int* __restrict__ d_status) {
  __shared__ int cnt[kMaxClasses];
  if (threadIdx.x < kMaxClasses) cnt[threadIdx.x] = 0;
  for (int i = threadIdx.x; i < list_total; i += blockDim.x) ws_list[i] = -1;
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
    ws_list[A.list_off[q] + w.slot] = i;
  }
  __syncthreads();
  if (threadIdx.x < kMaxClasses) ws_cnt[threadIdx.x] = cnt[threadIdx.x];
}

template <int FMT>
__global__ void __launch_bounds__(kGatherThreads) gather_kernel(GatherArgs A, const uint8_t* const* __restrict__ frames,
                                                                 const mp_window* __restrict__ win,
                                                                 const int* __restrict__ ws_cnt,
                                                                 const int* __restrict__ ws_list,
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

  if (wid == kConsumerWarps) {
    // ===================== producer warp =====================
    for (int i = 0;; i++) {
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
      // slot, then tile -> neighbouring CTAs share halo rows in L2.
      int q = 0, rel = t;
      while (rel >= min(cnt[q], A.cap[q]) * A.tpw[q]) {
        rel -= min(cnt[q], A.cap[q]) * A.tpw[q];
        q++;
      }
      const int slot = rel / A.tpw[q];
      const int tw = rel - slot * A.tpw[q];
      const int rt = tw / A.nct[q], ct = tw - rt * A.nct[q];
      const int wi = ws_list[A.list_off[q] + slot];
      if (wi < 0) {   // slots of this class are not 0..count-1
        if (lane == 0) {
          hdr->valid = 0;
          set_status(d_status, MP_ERR_INVALID);
          mbar_arrive(&full[s]);
        }
        __syncwarp();
        continue;
      }
      const mp_window w = win[wi];
      const int in_w = A.w[q], in_h = A.h[q], ow = A.ow[q], oh = A.oh[q];
      const int oy0 = rt * A.TR[q], ox0 = ct * A.TW[q];
      const int rows = min(A.TR[q], oh - oy0), cols = min(A.TW[q], ow - ox0);
      int c_lo, c_hi, r_lo, r_hi, dummy;
      float fl;
      tap(in_w, ow, ox0, c_lo, dummy, fl);
      tap(in_w, ow, ox0 + cols - 1, dummy, c_hi, fl);
      tap(in_h, oh, oy0, r_lo, dummy, fl);
      tap(in_h, oh, oy0 + rows - 1, dummy, r_hi, fl);
      const int b0 = (3 * (w.x + c_lo)) & ~15;
      const int b1 = (3 * (w.x + c_hi + 1) + 15) & ~15;
      const int stride = b1 - b0;
      const int nrows = r_hi - r_lo + 1;
      // taps for this tile: byte offsets inside the staged rows
      for (int c = lane; c < cols; c += 32) {
        int i0, i1;
        float lam;
        tap(in_w, ow, ox0 + c, i0, i1, lam);
        const int off = 3 * (w.x + i0) - b0;
        xt[c] = make_int2(off | ((3 * (i1 - i0)) << 20), __float_as_int(lam));
      }
      for (int r = lane; r < rows; r += 32) {
        int i0, i1;
        float lam;
        tap(in_h, oh, oy0 + r, i0, i1, lam);
        yt[r] = make_int4((i0 - r_lo) * stride, (i1 - r_lo) * stride, __float_as_int(lam), 0);
      }
      const uint8_t* src = frames[w.frame] + (size_t)(w.y + r_lo) * A.pitch + b0;
      if (lane == 0) {
        hdr->src = src;
        hdr->valid = 1;
        hdr->k = q;
        hdr->slot = w.slot;
        hdr->oy0 = oy0;
        hdr->ox0 = ox0;
        hdr->rows = rows;
        hdr->cols = cols;
        hdr->stride = stride;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&full[s], (uint32_t)(nrows * stride));
      __syncwarp();
      for (int r = lane; r < nrows; r += 32)
        bulk_g2s(data + (size_t)r * stride, src + (size_t)r * A.pitch, (uint32_t)stride, &full[s]);
    }
    return;
  }

  // ===================== consumer warps =====================
  // Thread <-> one output column of the tile (consecutive lanes = consecutive
  // columns: conflict-free byte loads, coalesced stores) and a contiguous block
  // of rows.  Separable evaluation: the horizontal lerp of a staged source row
  // is computed once and reused by the next output row that taps it.
  const int ctid = tid;   // 0 .. 32*kConsumerWarps-1
  for (int i = 0;; i++) {
    const int t = blockIdx.x + i * G;
    if (t >= T) break;
    const int s = i % kStages;
    mbar_wait(&full[s], (i / kStages) & 1);
    const unsigned char* stage = smem + (size_t)s * A.stage_bytes;
    const TileHdr* hdr = reinterpret_cast<const TileHdr*>(stage);
    if (hdr->valid) {
      const int2* xt = reinterpret_cast<const int2*>(stage + kHdrBytes);
      const int4* yt = reinterpret_cast<const int4*>(stage + kHdrBytes + kMaxTW * 8);
      const unsigned char* data = stage + kHdrBytes + kTapBytes;
      const int q = hdr->k, rows = hdr->rows, cols = hdr->cols;
      const int nph = max(1, (32 * kConsumerWarps) / cols);
      const int ph = ctid / cols, c = ctid - ph * cols;
      if (ph < nph) {
        const int rpp = (rows + nph - 1) / nph;
        const int rb0 = ph * rpp, rb1 = min(rows, rb0 + rpp);
        const int2 x = xt[c];
        const unsigned char* base = data + (x.x & 0xFFFFF);
        const int dx = x.x >> 20;
        const float lx = __int_as_float(x.y);
        const int ow = A.ow[q], oh = A.oh[q];
        int ra = -1, rb = -1;
        float ha0 = 0.f, ha1 = 0.f, ha2 = 0.f, hb0 = 0.f, hb1 = 0.f, hb2 = 0.f;
        auto hlerp = [&](int rowoff, float& h0, float& h1, float& h2) {
          const unsigned char* p = base + rowoff;
          const float a0 = u8f(p[0]), a1 = u8f(p[1]), a2 = u8f(p[2]);
          const float b0 = u8f(p[dx]), b1 = u8f(p[dx + 1]), b2 = u8f(p[dx + 2]);
          h0 = fmaf(lx, b0 - a0, a0);
          h1 = fmaf(lx, b1 - a1, a1);
          h2 = fmaf(lx, b2 - a2, a2);
        };
        if (FMT == MP_OUT_F32_NCHW) {
          const size_t plane = (size_t)oh * ow;
          float* o = reinterpret_cast<float*>(A.out[q]) + (size_t)hdr->slot * 3 * plane +
                     (size_t)(hdr->oy0 + rb0) * ow + hdr->ox0 + c;
          for (int r = rb0; r < rb1; r++) {
            const int4 y = yt[r];
            if (y.x != ra) {
              if (y.x == rb) { ha0 = hb0; ha1 = hb1; ha2 = hb2; }
              else hlerp(y.x, ha0, ha1, ha2);
              ra = y.x;
            }
            if (y.y != rb) {
              if (y.y == ra) { hb0 = ha0; hb1 = ha1; hb2 = ha2; }
              else hlerp(y.y, hb0, hb1, hb2);
              rb = y.y;
            }
            const float ly = __int_as_float(y.z);
            __stcs(o, fmaf(ly, hb0 - ha0, ha0));
            __stcs(o + plane, fmaf(ly, hb1 - ha1, ha1));
            __stcs(o + 2 * plane, fmaf(ly, hb2 - ha2, ha2));
            o += ow;
          }
        } else {
          uint8_t* o = reinterpret_cast<uint8_t*>(A.out[q]) +
                       (((size_t)hdr->slot * oh + hdr->oy0 + rb0) * ow + hdr->ox0 + c) * 3;
          for (int r = rb0; r < rb1; r++) {
            const int4 y = yt[r];
            if (y.x != ra) {
              if (y.x == rb) { ha0 = hb0; ha1 = hb1; ha2 = hb2; }
              else hlerp(y.x, ha0, ha1, ha2);
              ra = y.x;
            }
            if (y.y != rb) {
              if (y.y == ra) { hb0 = ha0; hb1 = ha1; hb2 = ha2; }
              else hlerp(y.y, hb0, hb1, hb2);
              rb = y.y;
            }
            const float ly = __int_as_float(y.z);
            const float v[3] = {fmaf(ly, hb0 - ha0, ha0), fmaf(ly, hb1 - ha1, ha1), fmaf(ly, hb2 - ha2, ha2)};
#pragma unroll
            for (int ch = 0; ch < 3; ch++) {
              int rr = __float2int_rd(v[ch] + 0.5f);   // R16 round half up
              o[ch] = (uint8_t)min(max(rr, 0), 255);
            }
            o += (size_t)ow * 3;
          }
        }
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
  int list = 0;
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
      TR = TR / 2;
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
    if (dat > data_max) data_max = dat;
  }
  A->stage_bytes = (int)(((kHdrBytes + kTapBytes + data_max) + 127) / 128 * 128);
  return true;
}

}  // namespace mpk

using namespace mpk;

extern "C" size_t mp_gather_workspace_size(int32_t k, const int32_t* out_cap) {
  if (k < 1 || k > kMaxClasses || !out_cap) return 0;
  size_t list = 0;
  for (int q = 0; q < k; q++) {
    if (out_cap[q] < 0) return 0;
    list += (size_t)out_cap[q];
  }
  return 256 + ((list * sizeof(int) + 255) & ~size_t(255));
}

extern "C" mp_status mp_gather_resize(const uint8_t* const* d_frame_ptrs, int32_t pitch, int32_t W, int32_t H,
                                      int32_t F, const mp_window* d_windows, const int32_t* d_frame_off,
                                      int32_t k, const mp_size* sizes, const mp_size* out_dims,
                                      void* const* d_out, const int32_t* out_cap, mp_out_format fmt,
                                      int32_t* d_status, void* d_ws, size_t ws_bytes, void* stream) {
  GatherArgs A;
  if (!build_gather_args(pitch, W, H, F, k, sizes, out_dims, d_out, out_cap, fmt, &A)) {
    // distinguish "too strong a downscale" from bad parameters
    return MP_ERR_INVALID;
  }
  if (!d_frame_off || !d_status || (F > 0 && (!d_frame_ptrs || !d_windows))) return MP_ERR_INVALID;
  const size_t need = mp_gather_workspace_size(k, out_cap);
  if (!d_ws || ws_bytes < need) return MP_ERR_INVALID;
  int list_total = 0;
  for (int q = 0; q < k; q++) list_total += out_cap[q];
  cudaStream_t s = (cudaStream_t)stream;
  int* ws_cnt = (int*)d_ws;
  int* ws_list = (int*)((unsigned char*)d_ws + 256);
  gather_prep_kernel<<<1, 1024, 0, s>>>(A, d_windows, d_frame_off, ws_cnt, ws_list, list_total, d_status);
  MP_CUDA_TRY(cudaGetLastError());
  if (F == 0) return MP_OK;
  const size_t smem = (size_t)kStages * A.stage_bytes + 2 * kStages * sizeof(uint64_t);
  if (smem > 227 * 1024) return MP_ERR_UNSUPPORTED;
  int dev = 0, sms = 0, per_sm = 0;
  MP_CUDA_TRY(cudaGetDevice(&dev));
  MP_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (fmt == MP_OUT_F32_NCHW) {
    MP_CUDA_TRY(cudaFuncSetAttribute(gather_kernel<MP_OUT_F32_NCHW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    MP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gather_kernel<MP_OUT_F32_NCHW>,
                                                              kGatherThreads, smem));
    if (per_sm < 1) per_sm = 1;
    gather_kernel<MP_OUT_F32_NCHW><<<sms * per_sm, kGatherThreads, smem, s>>>(A, d_frame_ptrs, d_windows, ws_cnt,
                                                                              ws_list, d_status);
  } else {
    MP_CUDA_TRY(cudaFuncSetAttribute(gather_kernel<MP_OUT_U8_NHWC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    MP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gather_kernel<MP_OUT_U8_NHWC>,
                                                              kGatherThreads, smem));
    if (per_sm < 1) per_sm = 1;
    gather_kernel<MP_OUT_U8_NHWC><<<sms * per_sm, kGatherThreads, smem, s>>>(A, d_frame_ptrs, d_windows, ws_cnt,
                                                                             ws_list, d_status);
  }
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}
