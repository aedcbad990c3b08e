// mp_nms.cu — steps a6-a7 (not in the paper; readings R17-R20):
// remap window-local detector boxes to frame pixels (one fp64 rounding
// sequence, bit-identical to the reading) and merge the windows of a frame
// with class-aware greedy NMS over a shared-memory IoU bitmask.
//
// Launches:
//   memset                      tier queue counters
//   nms_tiny_kernel    F warps  one warp per frame with <= 64 raw boxes: remap,
//                               ballot compaction, rank sort of the (score
//                               desc, index) keys, 64-bit IoU row masks, greedy
//                               scan; larger frames are queued
//   nms_small_kernel   6/SM     queued frames with <= 512 raw boxes, one 128-thread CTA
//                               each (persistent): block compaction, bitonic sort,
//                               then above 96 candidates (iou_thr >= 0) a
//                               spatial-grid sparse adjacency + warp-0 greedy,
//                               else an n x ceil(n/64) IoU bitmask (<= 128
//                               candidates) or 64-candidate tiles
//   nms_large_kernel   2/SM     queued frames with <= 1024 raw boxes, the same
//                               steps (128 threads); frames with more raw boxes
//                               run the tiled greedy over global-memory scratch,
//                               with a merge sort of the keys — no per-frame limit
//   nms_scan_kernel    1 CTA    kept-box CSR per frame, capacity check
//   nms_scatter_kernel          compact kept boxes into the caller's buffers
#include "mp_internal.cuh"

namespace mpk {

struct NmsArgs {
  int F, k, max_out, max_boxes;
  int max_windows;   // capacity of the windows buffer (a plan may report more in frame_off)
  float score_thr, iou_thr;
  int ow[kMaxClasses], oh[kMaxClasses];
};

#ifndef MP_NMS_SMALL_CAP   // (dev A/B builds may override the small tier's geometry)
#define MP_NMS_SMALL_CAP 512
#endif
#ifndef MP_NMS_SMALL_MINB
#define MP_NMS_SMALL_MINB 1
#endif
constexpr int kSmallCap = MP_NMS_SMALL_CAP, kSmallMaskCap = 128, kSmallThreads = 128;
// Every tier's CTA fits in what the persistent gather CTA leaves of an SM
// (<= 54 KB of shared memory = kSideReserve in mp_gather.cu, <= 16K registers), so the
// remap/NMS of batch i-1 runs beside gather(i) instead of queueing behind it
// (the former 1024-thread, 207-KB large tier could not start on any SM until
// the gather ended: c4 step = gather + NMS/plan tail).
constexpr int kLargeCap = 1024, kLargeMaskCap = 128, kLargeThreads = 128;

struct NmsSmem {
  float4* bx;
  int* cls;
  float* score;
  int* src;
  int* order;
  int* keep;
  unsigned long long* key;    // sort keys, then reused for the IoU bitmask
  unsigned char* supp;        // tiled-path suppression flags (overlaps key/mask)
  int* tmp;
  unsigned long long* bmask;  // tiled path: one 64-candidate block's IoU masks
  int* bkeep;                 // tiled path: candidates kept in the current block
  unsigned int ubytes;        // bytes of the key region (grid path scratch)
};

__host__ __device__ inline int pow2_at_least(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

__host__ __device__ inline size_t nms_smem_bytes(int cap, int mask_cap, NmsSmem* S, unsigned char* base) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 15) & ~size_t(15);
    return base ? base + o : nullptr;
  };
  NmsSmem s;
  s.bx = (float4*)take(sizeof(float4) * cap);
  s.cls = (int*)take(sizeof(int) * cap);
  s.score = (float*)take(sizeof(float) * cap);
  s.src = (int*)take(sizeof(int) * cap);
  s.order = (int*)take(sizeof(int) * cap);
  s.keep = (int*)take(sizeof(int) * cap);
  s.tmp = (int*)take(sizeof(int) * 64);
  s.bmask = (unsigned long long*)take(sizeof(unsigned long long) * 64);
  s.bkeep = (int*)take(sizeof(int) * 64);
  const size_t keyb = sizeof(unsigned long long) * pow2_at_least(cap);
  const size_t maskb = sizeof(unsigned long long) * (size_t)mask_cap * ((mask_cap + 63) / 64);
  size_t u = keyb > maskb ? keyb : maskb;
  if ((size_t)cap > u) u = cap;
  const size_t permb = (size_t)cap * sizeof(float4);   // sorted-order permutation scratch (one array at a time)
  if (permb > u) u = permb;
  s.key = (unsigned long long*)take(u);
  s.supp = (unsigned char*)s.key;
  s.ubytes = (unsigned int)u;
  if (S) *S = s;
  return off;
}

// R18: clip to [0,ow]x[0,oh] (fmin/fmax: NaN -> bound), drop degenerate,
// X = fp32((x_l * w) / ow + x) with each fp64 operation rounded once.
__device__ __forceinline__ bool remap(const mp_box& b, const mp_window& w, int ow, int oh, float thr, float4& o) {
  if (!(b.score > thr)) return false;
  const float x1 = fminf(fmaxf(b.x1, 0.0f), (float)ow), x2 = fminf(fmaxf(b.x2, 0.0f), (float)ow);
  const float y1 = fminf(fmaxf(b.y1, 0.0f), (float)oh), y2 = fminf(fmaxf(b.y2, 0.0f), (float)oh);
  if (!(x2 > x1) || !(y2 > y1)) return false;
  const double W = (double)w.w, H = (double)w.h, OW = (double)ow, OH = (double)oh;
  const double X = (double)w.x, Y = (double)w.y;
  o.x = __double2float_rn(__dadd_rn(__ddiv_rn(__dmul_rn((double)x1, W), OW), X));
  o.y = __double2float_rn(__dadd_rn(__ddiv_rn(__dmul_rn((double)y1, H), OH), Y));
  o.z = __double2float_rn(__dadd_rn(__ddiv_rn(__dmul_rn((double)x2, W), OW), X));
  o.w = __double2float_rn(__dadd_rn(__ddiv_rn(__dmul_rn((double)y2, H), OH), Y));
  return true;
}

// R19: fp32 IoU, every operation individually rounded (no FMA contraction),
// torchvision's formula order: inter / ((area_a + area_b) - inter).
__device__ __forceinline__ float iou_rn(const float4 a, const float4 b) {
  const float area_a = __fmul_rn(__fsub_rn(a.z, a.x), __fsub_rn(a.w, a.y));
  const float area_b = __fmul_rn(__fsub_rn(b.z, b.x), __fsub_rn(b.w, b.y));
  const float iw = fmaxf(__fsub_rn(fminf(a.z, b.z), fmaxf(a.x, b.x)), 0.0f);
  const float ih = fmaxf(__fsub_rn(fminf(a.w, b.w), fmaxf(a.y, b.y)), 0.0f);
  const float inter = __fmul_rn(iw, ih);
  const float uni = __fsub_rn(__fadd_rn(area_a, area_b), inter);
  // disjoint boxes (most pairs): 0 / uni is exactly 0 for uni > 0 -- skip the
  // IEEE division, whose slow path (FCHK) a zero dividend always takes
  if (inter == 0.0f && uni > 0.0f) return 0.0f;
  return __fdiv_rn(inter, uni);
}

// The suppression predicate of every NMS path: iou_rn(a, b) > thr.  For
// thr >= 0 it needs a positive-area intersection (IoU > 0), so the exact
// test min(x2) > max(x1) && min(y2) > max(y1) rejects the (most) disjoint
// pairs before the areas and the division; thr < 0 suppresses every pair
// (IoU >= 0 > thr) and takes the plain predicate.
__device__ __forceinline__ bool suppresses(const float4 a, const float4 b, float thr) {
  if (thr >= 0.0f && (!(fminf(a.z, b.z) > fmaxf(a.x, b.x)) || !(fminf(a.w, b.w) > fmaxf(a.y, b.y)))) return false;
  return iou_rn(a, b) > thr;
}

__device__ __forceinline__ unsigned int score_desc_bits(float s) {
  if (s == 0.0f) s = 0.0f;   // -0.0 -> +0.0 (equal in fp32 value order)
  const unsigned int u = __float_as_uint(s);
  const unsigned int asc = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ~asc;
}

// Index of the window containing raw box b: largest wi in [lo,hi) with off[wi] <= b.
__device__ __forceinline__ int window_of(const int* __restrict__ off, int lo, int hi, int b) {
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(off + mid) <= b) lo = mid;
    else hi = mid;
  }
  return lo;
}

// ---- a7 over a spatial grid (iou_thr >= 0): a pair can only suppress if the
// boxes intersect with positive area (IoU > thr >= 0 needs inter > 0; remap
// drops degenerate boxes), so each candidate is tested only against the
// candidates whose top-left corner lies in its own or a neighbouring cell of a
// grid whose cells are wider / taller than every candidate box.  The tested
// pairs produce a sparse adjacency (j > i, same class, iou_rn > thr — the very
// predicate of the bitmask paths), and warp 0 runs the greedy over it in score
// order: the same keep list as the dense paths, with O(n) instead of O(n^2)
// IoUs for the spread-out boxes of traffic / drone frames (c4: ~880 raw boxes
// per frame).  Scratch = the key region (free after the permutation).
// Returns the kept count, or -1 if the adjacency does not fit (the caller
// then runs a dense path).
constexpr int kGridMaxCells = 1024;
constexpr int kRankSortMax = 256;   // candidates up to which nms_frame rank-sorts its keys
constexpr int kGridMin = 96;   // candidates above which the grid path runs (below: the bitmask)

__device__ int nms_grid(const NmsArgs& A, const NmsSmem& S, int n) {
  const int tid = threadIdx.x, lane = tid & 31, BS = blockDim.x;
  // cell table size: 1/16 of the scratch (cell ends are ints), <= kGridMaxCells
  const int Gmax = min(kGridMaxCells, (int)(S.ubytes / 16));
  const int G = Gmax;
  int* red = S.tmp + 40;   // fp32 bits of min x1, min y1, max x1, max y1, max w, max h (all >= 0)
  if (tid < 6) red[tid] = tid < 2 ? 0x7f7fffff : 0;
  __syncthreads();
  {
    float v[6] = {3.4e38f, 3.4e38f, 0.f, 0.f, 0.f, 0.f};
    for (int p = tid; p < n; p += BS) {
      const float4 b = S.bx[p];
      v[0] = fminf(v[0], b.x);
      v[1] = fminf(v[1], b.y);
      v[2] = fmaxf(v[2], b.x);
      v[3] = fmaxf(v[3], b.y);
      v[4] = fmaxf(v[4], __fsub_rn(b.z, b.x));
      v[5] = fmaxf(v[5], __fsub_rn(b.w, b.y));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      v[0] = fminf(v[0], __shfl_xor_sync(0xffffffffu, v[0], o));
      v[1] = fminf(v[1], __shfl_xor_sync(0xffffffffu, v[1], o));
#pragma unroll
      for (int t = 2; t < 6; t++) v[t] = fmaxf(v[t], __shfl_xor_sync(0xffffffffu, v[t], o));
    }
    if (lane == 0) {
      atomicMin(&red[0], __float_as_int(v[0]));
      atomicMin(&red[1], __float_as_int(v[1]));
#pragma unroll
      for (int t = 2; t < 6; t++) atomicMax(&red[t], __float_as_int(v[t]));
    }
  }
  __syncthreads();
  const float mnx = __int_as_float(red[0]), mny = __int_as_float(red[1]);
  const float spx = __int_as_float(red[2]) - mnx, spy = __int_as_float(red[3]) - mny;
  // cells strictly wider / taller than any box (margin for the rounding of
  // the widths and of the cell index): an intersecting j has its corner in
  // the cell of i's corner or a neighbour.  As many cells as fit the scratch
  // (<= Gmax, about one candidate per cell for spread-out boxes): the
  // minimal cells, scaled up evenly when there would be more.
  const float mwx = __int_as_float(red[4]) * 1.0625f + 1.0f, mwy = __int_as_float(red[5]) * 1.0625f + 1.0f;
  float fx = spx / mwx + 1.0f, fy = spy / mwy + 1.0f;
  if (fx * fy > (float)Gmax) {
    const float sc = sqrtf((float)Gmax / (fx * fy));
    fx = fmaxf(1.0f, fx * sc);
    fy = fmaxf(1.0f, fy * sc);
  }
  int gx = max(1, min((int)fx, Gmax));
  int gy = max(1, min((int)fy, Gmax / gx));
  const float cwx = fmaxf(mwx, spx / (float)gx), cwy = fmaxf(mwy, spy / (float)gy);
  gx = min(gx, (int)(spx / cwx) + 1);
  gy = min(gy, (int)(spy / cwy) + 1);
  auto cell_x = [&](float x) { return min(gx - 1, (int)((x - mnx) / cwx)); };
  auto cell_y = [&](float y) { return min(gy - 1, (int)((y - mny) / cwy)); };
  // key-region layout: cell ends [G], members u16 [n], adjacency offsets [n+1],
  // suppression flags u8 [n], adjacency u16 [rest]
  unsigned char* base = reinterpret_cast<unsigned char*>(S.key);
  int* cend = reinterpret_cast<int*>(base);
  unsigned short* cellm = reinterpret_cast<unsigned short*>(base + 4 * G);
  int* off = reinterpret_cast<int*>(base + ((4 * G + 2 * n + 15) & ~15));
  unsigned char* supp = reinterpret_cast<unsigned char*>(off) + (((n + 1) * 4 + 15) & ~15);
  unsigned short* adj = reinterpret_cast<unsigned short*>(supp + ((n + 15) & ~15));
  const int cap_adj = (int)(((long long)S.ubytes - (long long)(reinterpret_cast<unsigned char*>(adj) - base)) / 2);
  for (int c = tid; c < G; c += BS) cend[c] = 0;
  __syncthreads();
  for (int p = tid; p < n; p += BS) atomicAdd(&cend[cell_y(S.bx[p].y) * gx + cell_x(S.bx[p].x)], 1);
  __syncthreads();
  block_excl_scan_smem(cend, gx * gy, S.tmp);   // cend[c] = start of cell c
  for (int p = tid; p < n; p += BS) {
    const int c = cell_y(S.bx[p].y) * gx + cell_x(S.bx[p].x);
    cellm[atomicAdd(&cend[c], 1)] = (unsigned short)p;   // afterwards cend[c] = end of cell c
  }
  __syncthreads();
  const float thr = A.iou_thr;
  // each candidate i scans the three rows of its 3x3 neighbourhood (the
  // cells of a row are contiguous in cellm) in a fixed order; test k of the
  // scan records its outcome in bit k of `hits` (k < 64), so after
  // reserving popc(hits) adjacency slots with one shared atomic the scan is
  // replayed writing the hits without recomputing any IoU.  The exact
  // intersection test first skips the (most) pairs that cannot overlap:
  // iou_rn > thr >= 0 needs min(x2) > max(x1) and min(y2) > max(y1).
  int* nadj = S.tmp + 48;
  if (tid == 0) *nadj = 0;
  __syncthreads();
  for (int i = tid; i < n; i += BS) {
    const float4 bi = S.bx[i];
    const int ci = S.cls[i];
    const int cx = cell_x(bi.x), cy = cell_y(bi.y);
    const int x0 = max(cx - 1, 0), x1 = min(cx + 1, gx - 1);
    const int y0 = max(cy - 1, 0), y1 = min(cy + 1, gy - 1);
    auto test = [&](int j) -> bool {
      if (j <= i || S.cls[j] != ci) return false;
      return suppresses(bi, S.bx[j], thr);   // (thr >= 0 here)
    };
    unsigned long long hits = 0;
    int d = 0, k = 0;
    for (int yy = y0; yy <= y1; yy++) {
      const int c0 = yy * gx + x0, c1 = yy * gx + x1;
      for (int e = (c0 ? cend[c0 - 1] : 0); e < cend[c1]; e++, k++) {
        if (test(cellm[e])) {
          if (k < 64) hits |= 1ull << k;
          d++;
        }
      }
    }
    const int base = d ? atomicAdd(nadj, d) : 0;
    off[i] = (int)(((unsigned int)base << 16) | (unsigned int)d);   // (base, degree), both < 65536 when it fits
    if (base + d <= cap_adj && d) {
      int w = base;
      k = 0;
      for (int yy = y0; yy <= y1; yy++) {
        const int c0 = yy * gx + x0, c1 = yy * gx + x1;
        for (int e = (c0 ? cend[c0 - 1] : 0); e < cend[c1]; e++, k++) {
          const int j = cellm[e];
          if (k < 64 ? ((hits >> k) & 1ull) != 0 : test(j)) adj[w++] = (unsigned short)j;
        }
      }
    }
  }
  for (int p = tid; p < n; p += BS) supp[p] = 0;
  __syncthreads();
  if (*nadj > cap_adj) return -1;   // (uniform) the adjacency does not fit: dense path
  // greedy in score order (warp 0): per chunk of 32 candidates, repeatedly
  // take the first candidate neither suppressed nor already kept, keep it and
  // flag its suppressees (later chunk members included, re-read next round)
  if (threadIdx.x < 32) {
    int nk = 0;
    for (int b0 = 0; b0 < n; b0 += 32) {
      const int i = b0 + lane;
      uint32_t taken = 0;
      while (true) {
        const uint32_t free = __ballot_sync(0xffffffffu, i < n && !supp[i]) & ~taken;
        __syncwarp();   // every lane's supp read is ordered before this round's writes
        if (!free) break;
        const int b = __ffs(free) - 1;
        const int k = b0 + b;
        taken |= 1u << b;
        if (lane == 0) S.keep[nk] = k;
        nk++;
        const int ob = (int)((unsigned int)off[k] >> 16), od = off[k] & 0xffff;
        for (int e = lane; e < od; e += 32) supp[adj[ob + e]] = 1;
        __syncwarp();
      }
    }
    if (lane == 0) S.tmp[32] = nk;
  }
  __syncthreads();
  return S.tmp[32];
}

// Process one frame with the whole CTA.  Returns nothing; writes kept boxes to
// the frame's scratch region (raw-box offsets) and ws_kept[f].
__device__ void nms_frame(const NmsArgs& A, int f, int b_lo, int b_hi, int w_lo, int w_hi, const NmsSmem& S,
                          int cap, int mask_cap, const mp_box* __restrict__ boxes,
                          const int* __restrict__ win_box_off, const mp_window* __restrict__ windows,
                          mp_box* __restrict__ ws_box, int* __restrict__ ws_src, int* __restrict__ ws_kept) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  // ---- a6: remap + ordered compaction (candidate order = input order)
  int n = 0;
  for (int base = b_lo; base < b_hi; base += blockDim.x) {
    const int b = base + tid;
    bool ok = false;
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
    mp_box bb;
    if (b < b_hi) {
      const int wi = window_of(win_box_off, w_lo, w_hi, b);
      const mp_window w = windows[wi];
      bb = boxes[b];
      const int q = w.size_idx;
      ok = (q >= 0 && q < A.k) && remap(bb, w, A.ow[q], A.oh[q], A.score_thr, o);
    }
    const uint32_t m = __ballot_sync(0xffffffffu, ok);
    if (lane == 0) S.tmp[wid] = __popc(m);
    __syncthreads();
    int before = 0, tot = 0;
    for (int q = 0; q < nw; q++) {
      const int c = S.tmp[q];
      before += (q < wid) ? c : 0;
      tot += c;
    }
    if (ok) {
      const int p = n + before + __popc(m & lanemask_lt());
      S.bx[p] = o;
      S.cls[p] = bb.cls;
      S.score[p] = bb.score;
      S.src[p] = b;
      S.key[p] = ((unsigned long long)score_desc_bits(bb.score) << 32) | (unsigned)p;
    }
    n += tot;
    __syncthreads();
  }
  // ---- sort keys ascending = (score desc, candidate index asc)
  if (n <= kRankSortMax) {
    // rank sort (the keys are unique): one barrier instead of the bitonic
    // network's log^2 barriers — beside a persistent gather every barrier
    // phase is slow, and c3's 100-150-candidate frames would spend most of
    // their time in the network's ~36 phases
    for (int p = tid; p < n; p += blockDim.x) {
      const unsigned long long k = S.key[p];
      int r = 0;
      for (int q = 0; q < n; q++) r += S.key[q] < k ? 1 : 0;
      S.order[r] = p;
    }
    __syncthreads();
  } else {
    const int P = pow2_at_least(n < 1 ? 1 : n);
    for (int p = n + tid; p < P; p += blockDim.x) S.key[p] = ~0ull;
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int t = tid; t < (P >> 1); t += blockDim.x) {
          const int i = 2 * j * (t / j) + (t % j);
          const int l = i + j;
          const bool up = (i & k) == 0;
          const unsigned long long a = S.key[i], c = S.key[l];
          if ((a > c) == up) {
            S.key[i] = c;
            S.key[l] = a;
          }
        }
        __syncthreads();
      }
    }
    for (int p = tid; p < n; p += blockDim.x) S.order[p] = (int)(S.key[p] & 0xffffffffu);
    __syncthreads();
  }
  // physically permute the candidates into the sorted order (one array at a
  // time through the now free key region, 16 B per candidate) so the O(n^2)
  // IoU loops read consecutive entries instead of order[]-scattered ones;
  // order[] becomes the identity
  {
    float4* tb = reinterpret_cast<float4*>(S.key);
    for (int p = tid; p < n; p += blockDim.x) tb[p] = S.bx[S.order[p]];
    __syncthreads();
    for (int p = tid; p < n; p += blockDim.x) S.bx[p] = tb[p];
    __syncthreads();
    int* ti = reinterpret_cast<int*>(S.key);
    int* arrs[3] = {S.cls, reinterpret_cast<int*>(S.score), S.src};
#pragma unroll
    for (int a = 0; a < 3; a++) {
      int* v = arrs[a];
      for (int p = tid; p < n; p += blockDim.x) ti[p] = v[S.order[p]];
      __syncthreads();
      for (int p = tid; p < n; p += blockDim.x) v[p] = ti[p];
      __syncthreads();
    }
    for (int p = tid; p < n; p += blockDim.x) S.order[p] = p;
    __syncthreads();
  }

  // ---- a7: greedy class-aware NMS
  int nk = -1;
  if (n > kGridMin && A.iou_thr >= 0.0f) nk = nms_grid(A, S, n);
  if (nk >= 0) {
    // kept by the grid path
  } else if (n <= mask_cap) {
    nk = 0;
    const int words = (n + 63) >> 6;
    unsigned long long* mask = S.key;
    for (int idx = tid; idx < n * words; idx += blockDim.x) {
      // consecutive threads = consecutive rows of one 64-column word: the
      // (sorted, contiguous) column boxes are read as broadcasts
      const int wd = idx / n, i = idx - wd * n;
      const int qi = S.order[i];
      const float4 bi = S.bx[qi];
      const int ci = S.cls[qi];
      unsigned long long bits = 0;
      const int j0 = max(i + 1, wd * 64), j1 = min(n, wd * 64 + 64);
      for (int j = j0; j < j1; j++) {
        const int qj = S.order[j];
        if (S.cls[qj] == ci && suppresses(bi, S.bx[qj], A.iou_thr)) bits |= 1ull << (j - wd * 64);
      }
      mask[(size_t)i * words + wd] = bits;
    }
    __syncthreads();
    if (wid == 0) {
      unsigned long long r0 = 0, r1 = 0;
      for (int i = 0; i < n; i++) {
        const int wd = i >> 6;
        const unsigned long long mine = (wd >> 5) ? r1 : r0;
        const unsigned long long wv = __shfl_sync(0xffffffffu, mine, wd & 31);
        if (!((wv >> (i & 63)) & 1ull)) {
          if (lane == 0) S.keep[nk] = i;
          nk++;
          if (lane < words) r0 |= mask[(size_t)i * words + lane];
          if (lane + 32 < words) r1 |= mask[(size_t)i * words + lane + 32];
        }
      }
      if (lane == 0) S.tmp[32] = nk;
    }
    __syncthreads();
    nk = S.tmp[32];
  } else {
    nk = 0;
    // Tiled greedy for large frames (identical result to the sequential scan):
    // for each block of 64 sorted candidates, (a) the block's 64x64 IoU masks,
    // (b) one thread resolves the block sequentially against those masks and
    // the suppression flags left by earlier blocks, (c) the whole CTA
    // suppresses every later candidate overlapping a box kept in this block.
    for (int p = tid; p < n; p += blockDim.x) S.supp[p] = 0;
    __syncthreads();
    for (int b0 = 0; b0 < n; b0 += 64) {
      const int b1 = min(n, b0 + 64);
      for (int i = b0 + tid; i < b1; i += blockDim.x) {
        const int qi = S.order[i];
        const float4 bi = S.bx[qi];
        const int ci = S.cls[qi];
        unsigned long long bits = 0;
        for (int j = i + 1; j < b1; j++) {
          const int qj = S.order[j];
          if (S.cls[qj] == ci && suppresses(bi, S.bx[qj], A.iou_thr)) bits |= 1ull << (j - b0);
        }
        S.bmask[i - b0] = bits;
      }
      __syncthreads();
      if (tid == 0) {
        unsigned long long removed = 0;
        for (int i = b0; i < b1; i++)
          if (S.supp[i]) removed |= 1ull << (i - b0);
        int nb = 0;
        for (int i = b0; i < b1; i++) {
          if (!((removed >> (i - b0)) & 1ull)) {
            S.keep[nk + nb] = i;
            S.bkeep[nb++] = i;
            removed |= S.bmask[i - b0];
          }
        }
        S.tmp[33] = nb;
      }
      __syncthreads();
      const int nb = S.tmp[33];
      for (int j = b1 + tid; j < n; j += blockDim.x) {
        if (S.supp[j]) continue;
        const int qj = S.order[j];
        const float4 bj = S.bx[qj];
        const int cj = S.cls[qj];
        for (int r = 0; r < nb; r++) {
          const int qk = S.order[S.bkeep[r]];
          if (S.cls[qk] == cj && suppresses(S.bx[qk], bj, A.iou_thr)) {
            S.supp[j] = 1;
            break;
          }
        }
      }
      nk += nb;
      __syncthreads();
    }
  }
  // ---- output in keep order to the frame's scratch region
  for (int r = tid; r < nk; r += blockDim.x) {
    const int q = S.order[S.keep[r]];
    const float4 o = S.bx[q];
    mp_box ob;
    ob.x1 = o.x;
    ob.y1 = o.y;
    ob.x2 = o.z;
    ob.y2 = o.w;
    ob.score = S.score[q];
    ob.cls = S.cls[q];
    ws_box[b_lo + r] = ob;
    ws_src[b_lo + r] = S.src[q];
  }
  if (tid == 0) ws_kept[f] = nk;
}

// Global-memory scratch of the unbounded path, indexed by raw-box position
// (a frame's candidates live at its raw-box range [b_lo, b_hi)).
struct NmsGlobal {
  float4* bx;
  int* cls;
  float* score;
  int* src;
  unsigned long long* key;
  unsigned long long* key2;
  int* keep;
  unsigned char* supp;
};

// Number of keys in the ascending run k[lo, hi) that are < x.
__device__ __forceinline__ int count_less(const unsigned long long* __restrict__ k, int lo, int hi,
                                          unsigned long long x) {
  const int base = lo;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (k[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo - base;
}

// Frames with more raw boxes than fit in shared memory: the same steps and
// arithmetic as nms_frame (remap + ordered compaction, sort by the unique
// (score desc, index) keys, tiled greedy with 64-candidate blocks), with the
// candidates in global scratch and the keys sorted by a bottom-up merge sort
// (each key's output position = its offset in its run + its rank in the
// partner run).  Slow (O(n^2) IoUs over L2) but exact and unbounded.
__device__ void nms_frame_global(const NmsArgs& A, int f, int b_lo, int b_hi, int w_lo, int w_hi, const NmsSmem& S,
                                 const NmsGlobal& g, const mp_box* __restrict__ boxes,
                                 const int* __restrict__ win_box_off, const mp_window* __restrict__ windows,
                                 mp_box* __restrict__ ws_box, int* __restrict__ ws_src, int* __restrict__ ws_kept) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  float4* gbx = g.bx + b_lo;
  int* gcls = g.cls + b_lo;
  float* gscore = g.score + b_lo;
  int* gsrc = g.src + b_lo;
  unsigned char* supp = g.supp + b_lo;
  int* keep = g.keep + b_lo;
  // ---- a6: remap + ordered compaction (candidate order = input order)
  int n = 0;
  for (int base = b_lo; base < b_hi; base += blockDim.x) {
    const int b = base + tid;
    bool ok = false;
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
    mp_box bb;
    if (b < b_hi) {
      const int wi = window_of(win_box_off, w_lo, w_hi, b);
      const mp_window w = windows[wi];
      bb = boxes[b];
      const int q = w.size_idx;
      ok = (q >= 0 && q < A.k) && remap(bb, w, A.ow[q], A.oh[q], A.score_thr, o);
    }
    const uint32_t m = __ballot_sync(0xffffffffu, ok);
    if (lane == 0) S.tmp[wid] = __popc(m);
    __syncthreads();
    int before = 0, tot = 0;
    for (int q = 0; q < nw; q++) {
      const int c = S.tmp[q];
      before += (q < wid) ? c : 0;
      tot += c;
    }
    if (ok) {
      const int p = n + before + __popc(m & lanemask_lt());
      gbx[p] = o;
      gcls[p] = bb.cls;
      gscore[p] = bb.score;
      gsrc[p] = b;
      g.key[b_lo + p] = ((unsigned long long)score_desc_bits(bb.score) << 32) | (unsigned)p;
    }
    n += tot;
    __syncthreads();
  }
  // ---- merge sort of the unique keys (ascending = score desc, index asc)
  unsigned long long* ka = g.key + b_lo;
  unsigned long long* kb = g.key2 + b_lo;
  for (int w = 1; w < n; w <<= 1) {
    for (int i = tid; i < n; i += blockDim.x) {
      const int a = (i / (2 * w)) * (2 * w);
      const int mid = min(a + w, n), end = min(a + 2 * w, n);
      const unsigned long long x = ka[i];
      const int pos = i < mid ? i + count_less(ka, mid, end, x) : a + (i - mid) + count_less(ka, a, mid, x);
      kb[pos] = x;
    }
    __syncthreads();
    unsigned long long* t = ka;
    ka = kb;
    kb = t;
  }
  for (int p = tid; p < n; p += blockDim.x) supp[p] = 0;
  __syncthreads();
  // ---- a7: tiled greedy (identical result to the sequential scan)
  int nk = 0;
  for (int b0 = 0; b0 < n; b0 += 64) {
    const int b1 = min(n, b0 + 64);
    for (int i = b0 + tid; i < b1; i += blockDim.x) {
      const int qi = (int)(ka[i] & 0xffffffffu);
      const float4 bi = gbx[qi];
      const int ci = gcls[qi];
      unsigned long long bits = 0;
      for (int j = i + 1; j < b1; j++) {
        const int qj = (int)(ka[j] & 0xffffffffu);
        if (gcls[qj] == ci && suppresses(bi, gbx[qj], A.iou_thr)) bits |= 1ull << (j - b0);
      }
      S.bmask[i - b0] = bits;
    }
    __syncthreads();
    if (tid == 0) {
      unsigned long long removed = 0;
      for (int i = b0; i < b1; i++)
        if (supp[i]) removed |= 1ull << (i - b0);
      int nb = 0;
      for (int i = b0; i < b1; i++) {
        if (!((removed >> (i - b0)) & 1ull)) {
          keep[nk + nb] = i;
          S.bkeep[nb++] = i;
          removed |= S.bmask[i - b0];
        }
      }
      S.tmp[33] = nb;
    }
    __syncthreads();
    const int nb = S.tmp[33];
    for (int j = b1 + tid; j < n; j += blockDim.x) {
      if (supp[j]) continue;
      const int qj = (int)(ka[j] & 0xffffffffu);
      const float4 bj = gbx[qj];
      const int cj = gcls[qj];
      for (int r = 0; r < nb; r++) {
        const int qk = (int)(ka[S.bkeep[r]] & 0xffffffffu);
        if (gcls[qk] == cj && suppresses(gbx[qk], bj, A.iou_thr)) {
          supp[j] = 1;
          break;
        }
      }
    }
    nk += nb;
    __syncthreads();
  }
  // ---- output in keep order to the frame's scratch region
  for (int r = tid; r < nk; r += blockDim.x) {
    const int q = (int)(ka[keep[r]] & 0xffffffffu);
    const float4 o = gbx[q];
    mp_box ob;
    ob.x1 = o.x;
    ob.y1 = o.y;
    ob.x2 = o.z;
    ob.y2 = o.w;
    ob.score = gscore[q];
    ob.cls = gcls[q];
    ws_box[b_lo + r] = ob;
    ws_src[b_lo + r] = gsrc[q];
  }
  if (tid == 0) ws_kept[f] = nk;
}

__device__ __forceinline__ bool frame_range(const NmsArgs& A, int f, const int* frame_off, const int* win_box_off,
                                            int& w_lo, int& w_hi, int& b_lo, int& b_hi) {
  // windows past the buffer's capacity (a plan that overflowed it still
  // reports true offsets) do not exist: clamp, so no read leaves the buffers
  w_lo = min(max(frame_off[f], 0), A.max_windows);
  w_hi = min(max(frame_off[f + 1], 0), A.max_windows);
  if (w_hi < w_lo) {
    b_lo = b_hi = 0;
    return false;
  }
  b_lo = win_box_off[w_lo];
  b_hi = win_box_off[w_hi];
  return b_lo >= 0 && b_hi >= b_lo && b_hi <= A.max_boxes;
}

#ifndef MP_NMS_TINY_WARPS
#define MP_NMS_TINY_WARPS 8
#endif
constexpr int kTinyCap = 64, kTinyWarps = MP_NMS_TINY_WARPS;

struct TinyWarpSmem {
  float4 bx[kTinyCap];
  unsigned long long key[kTinyCap];
  unsigned long long mask[kTinyCap];
  int cls[kTinyCap];
  float score[kTinyCap];
  int src[kTinyCap];
  int order[kTinyCap];
  int keep[kTinyCap];
};

// One warp per frame (frames with <= 64 raw boxes; the typical case).  Same
// semantics and arithmetic as nms_frame (R18-R20); candidate index = position
// in input order, rank sort by unique (score desc, index) keys.
__global__ void __launch_bounds__(32 * kTinyWarps) nms_tiny_kernel(NmsArgs A, const mp_box* __restrict__ boxes,
                                                                   const int* __restrict__ win_box_off,
                                                                   const mp_window* __restrict__ windows,
                                                                   const int* __restrict__ frame_off,
                                                                   mp_box* __restrict__ ws_box, int* __restrict__ ws_src,
                                                                   int* __restrict__ ws_kept, int* __restrict__ mid_cnt,
                                                                   int* __restrict__ mid_list, int* __restrict__ d_status) {
  __shared__ TinyWarpSmem sm_all[kTinyWarps];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int f = blockIdx.x * kTinyWarps + wid;
  if (f >= A.F) return;
  TinyWarpSmem& S = sm_all[wid];
  int w_lo, w_hi, b_lo, b_hi;
  if (!frame_range(A, f, frame_off, win_box_off, w_lo, w_hi, b_lo, b_hi)) {
    if (lane == 0) {
      ws_kept[f] = 0;
      set_status(d_status, MP_ERR_INVALID);
    }
    return;
  }
  if (b_hi - b_lo > kTinyCap) {
    if (lane == 0) mid_list[atomicAdd(mid_cnt, 1)] = f;
    return;
  }
  // ---- a6: remap + ordered ballot compaction
  int n = 0;
#pragma unroll
  for (int h = 0; h < 2; h++) {
    const int b = b_lo + h * 32 + lane;
    bool ok = false;
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
    mp_box bb;
    if (b < b_hi) {
      const int wi = window_of(win_box_off, w_lo, w_hi, b);
      const mp_window w = windows[wi];
      bb = boxes[b];
      const int q = w.size_idx;
      ok = (q >= 0 && q < A.k) && remap(bb, w, A.ow[q], A.oh[q], A.score_thr, o);
    }
    const uint32_t m = __ballot_sync(0xffffffffu, ok);
    if (ok) {
      const int p = n + __popc(m & lanemask_lt());
      S.bx[p] = o;
      S.cls[p] = bb.cls;
      S.score[p] = bb.score;
      S.src[p] = b;
      S.key[p] = ((unsigned long long)score_desc_bits(bb.score) << 32) | (unsigned)p;
    }
    n += __popc(m);
  }
  __syncwarp();
  // ---- rank sort (keys are unique)
#pragma unroll
  for (int h = 0; h < 2; h++) {
    const int p = h * 32 + lane;
    if (p < n) {
      const unsigned long long kp = S.key[p];
      int rank = 0;
      for (int q2 = 0; q2 < n; q2++) rank += (S.key[q2] < kp) ? 1 : 0;
      S.order[rank] = p;
    }
  }
  __syncwarp();
  // ---- a7: IoU row masks over later candidates of the same class
#pragma unroll
  for (int h = 0; h < 2; h++) {
    const int i = h * 32 + lane;
    if (i < n) {
      const int qi = S.order[i];
      const float4 bi = S.bx[qi];
      const int ci = S.cls[qi];
      unsigned long long bits = 0;
      for (int j = i + 1; j < n; j++) {
        const int qj = S.order[j];
        if (S.cls[qj] == ci && suppresses(bi, S.bx[qj], A.iou_thr)) bits |= 1ull << j;
      }
      S.mask[i] = bits;
    }
  }
  __syncwarp();
  int nk = 0;
  if (lane == 0) {
    unsigned long long removed = 0;
    for (int i = 0; i < n; i++) {
      if (!((removed >> i) & 1ull)) {
        S.keep[nk++] = i;
        removed |= S.mask[i];
      }
    }
  }
  nk = __shfl_sync(0xffffffffu, nk, 0);
  __syncwarp();
  for (int r = lane; r < nk; r += 32) {
    const int q = S.order[S.keep[r]];
    const float4 o = S.bx[q];
    mp_box ob;
    ob.x1 = o.x;
    ob.y1 = o.y;
    ob.x2 = o.z;
    ob.y2 = o.w;
    ob.score = S.score[q];
    ob.cls = S.cls[q];
    ws_box[b_lo + r] = ob;
    ws_src[b_lo + r] = S.src[q];
  }
  if (lane == 0) ws_kept[f] = nk;
}

// Queued frames with 65..512 raw boxes, one CTA per frame (persistent).
__global__ void __launch_bounds__(kSmallThreads, MP_NMS_SMALL_MINB) nms_small_kernel(NmsArgs A, const mp_box* __restrict__ boxes,
                                                                  const int* __restrict__ win_box_off,
                                                                  const mp_window* __restrict__ windows,
                                                                  const int* __restrict__ frame_off,
                                                                  mp_box* __restrict__ ws_box, int* __restrict__ ws_src,
                                                                  int* __restrict__ ws_kept, const int* __restrict__ mid_cnt,
                                                                  const int* __restrict__ mid_list, int* __restrict__ large_cnt,
                                                                  int* __restrict__ large_list, int* __restrict__ d_status) {
  extern __shared__ __align__(16) unsigned char smem[];
  NmsSmem S;
  nms_smem_bytes(kSmallCap, kSmallMaskCap, &S, smem);
  const int nm = *mid_cnt;
  for (int li = blockIdx.x; li < nm; li += gridDim.x) {
    const int f = mid_list[li];
    int w_lo, w_hi, b_lo, b_hi;
    frame_range(A, f, frame_off, win_box_off, w_lo, w_hi, b_lo, b_hi);
    if (b_hi - b_lo > kSmallCap) {
      if (threadIdx.x == 0) large_list[atomicAdd(large_cnt, 1)] = f;
      continue;
    }
    nms_frame(A, f, b_lo, b_hi, w_lo, w_hi, S, kSmallCap, kSmallMaskCap, boxes, win_box_off, windows, ws_box, ws_src,
              ws_kept);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kLargeThreads) nms_large_kernel(NmsArgs A, const mp_box* __restrict__ boxes,
                                                                  const int* __restrict__ win_box_off,
                                                                  const mp_window* __restrict__ windows,
                                                                  const int* __restrict__ frame_off,
                                                                  mp_box* __restrict__ ws_box, int* __restrict__ ws_src,
                                                                  int* __restrict__ ws_kept, const int* __restrict__ large_cnt,
                                                                  const int* __restrict__ large_list, NmsGlobal g,
                                                                  int* __restrict__ d_status) {
  extern __shared__ __align__(16) unsigned char smem[];
  NmsSmem S;
  nms_smem_bytes(kLargeCap, kLargeMaskCap, &S, smem);
  const int nl = *large_cnt;
  for (int li = blockIdx.x; li < nl; li += gridDim.x) {
    const int f = large_list[li];
    int w_lo, w_hi, b_lo, b_hi;
    frame_range(A, f, frame_off, win_box_off, w_lo, w_hi, b_lo, b_hi);
    if (b_hi - b_lo > kLargeCap)
      nms_frame_global(A, f, b_lo, b_hi, w_lo, w_hi, S, g, boxes, win_box_off, windows, ws_box, ws_src, ws_kept);
    else
      nms_frame(A, f, b_lo, b_hi, w_lo, w_hi, S, kLargeCap, kLargeMaskCap, boxes, win_box_off, windows, ws_box,
                ws_src, ws_kept);
    __syncthreads();
  }
}

// 256 threads (not 1024): a 1024-thread CTA needs ~32 K registers, more than a
// persistent gather CTA leaves of an SM, and would wait for the gather to end.
__global__ void __launch_bounds__(kScanThreads, kScanMinBlocks) nms_scan_kernel(int F, const int* __restrict__ ws_kept,
                                                        int* __restrict__ out_frame_off, int max_out,
                                                        int* __restrict__ d_status) {
  __shared__ int tmp[40];
  for (int f = threadIdx.x; f < F; f += blockDim.x) out_frame_off[f] = ws_kept[f];
  __syncthreads();
  const int total = block_scan_global(out_frame_off, F, 1, tmp);
  if (threadIdx.x == 0) {
    out_frame_off[F] = total;
    if (total > max_out) set_status(d_status, MP_ERR_CAPACITY);
  }
}

__global__ void __launch_bounds__(256) nms_scatter_kernel(int F, const int* __restrict__ frame_off,
                                                          const int* __restrict__ win_box_off,
                                                          const mp_box* __restrict__ ws_box,
                                                          const int* __restrict__ ws_src, const int* __restrict__ ws_kept,
                                                          const int* __restrict__ out_frame_off, mp_box* __restrict__ out,
                                                          int* __restrict__ out_src, int max_out, int max_windows) {
  const int f = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (f >= F) return;
  const int n = ws_kept[f];
  if (n == 0) return;   // (frames with invalid ranges keep nothing)
  const int b_lo = win_box_off[min(max(frame_off[f], 0), max_windows)];
  const int base = out_frame_off[f];
  for (int r = lane; r < n; r += 32) {
    const int d = base + r;
    if (d >= max_out) break;
    out[d] = ws_box[b_lo + r];
    out_src[d] = ws_src[b_lo + r];
  }
}

struct NmsWs {
  size_t box_off, src_off, kept_off, lcnt_off, llist_off, mlist_off;
  size_t gbx_off, gcls_off, gscore_off, gsrc_off, gkey_off, gkey2_off, gkeep_off, gsupp_off, total;
};

static NmsWs nms_ws_layout(int F, int max_boxes) {
  NmsWs L;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  L.box_off = 0;
  L.src_off = al(sizeof(mp_box) * (size_t)max_boxes);
  L.kept_off = al(L.src_off + sizeof(int) * (size_t)max_boxes);
  L.lcnt_off = al(L.kept_off + sizeof(int) * (size_t)F);   // [0] large count, [1] mid count
  L.llist_off = al(L.lcnt_off + 2 * sizeof(int));
  L.mlist_off = al(L.llist_off + sizeof(int) * (size_t)F);
  // unbounded path (frames with > kLargeCap raw boxes): per raw box 49 bytes
  const size_t nb = (size_t)max_boxes;
  L.gbx_off = al(L.mlist_off + sizeof(int) * (size_t)F);
  L.gcls_off = al(L.gbx_off + sizeof(float4) * nb);
  L.gscore_off = al(L.gcls_off + sizeof(int) * nb);
  L.gsrc_off = al(L.gscore_off + sizeof(float) * nb);
  L.gkey_off = al(L.gsrc_off + sizeof(int) * nb);
  L.gkey2_off = al(L.gkey_off + 8 * nb);
  L.gkeep_off = al(L.gkey2_off + 8 * nb);
  L.gsupp_off = al(L.gkeep_off + sizeof(int) * nb);
  L.total = al(L.gsupp_off + nb) + 256;
  return L;
}

}  // namespace mpk

using namespace mpk;

extern "C" size_t mp_remap_nms_workspace_size(int32_t F, int32_t max_boxes) {
  if (F < 0 || max_boxes < 0) return 0;
  return nms_ws_layout(F, max_boxes).total;
}

extern "C" mp_status mp_remap_nms(const mp_box* d_boxes, const int32_t* d_win_box_off, const mp_window* d_windows,
                                  const int32_t* d_frame_off, int32_t max_windows, int32_t F, int32_t k,
                                  const mp_size* out_dims,
                                  int32_t W, int32_t H, float score_thr, float iou_thr, mp_box* d_out,
                                  int32_t* d_out_src, int32_t max_out, int32_t* d_out_frame_off, int32_t* d_status,
                                  int32_t max_boxes, void* d_ws, size_t ws_bytes, void* stream) {
  if (F < 0 || k < 1 || k > kMaxClasses || !out_dims || W < 1 || H < 1 || max_out < 0 || max_boxes < 0 ||
      max_windows < 0)
    return MP_ERR_INVALID;
  if (!d_out_frame_off || !d_status || !d_frame_off || !d_win_box_off) return MP_ERR_INVALID;
  if (max_out > 0 && (!d_out || !d_out_src)) return MP_ERR_INVALID;
  if (F > 0 && ((max_windows > 0 && !d_windows) || (max_boxes > 0 && !d_boxes))) return MP_ERR_INVALID;
  if (!(iou_thr == iou_thr) || !(score_thr == score_thr)) return MP_ERR_INVALID;
  NmsArgs A;
  memset(&A, 0, sizeof(A));
  A.F = F;
  A.k = k;
  A.max_out = max_out;
  A.max_boxes = max_boxes;
  A.max_windows = max_windows;
  A.score_thr = score_thr;
  A.iou_thr = iou_thr;
  for (int q = 0; q < k; q++) {
    if (out_dims[q].w < 1 || out_dims[q].h < 1) return MP_ERR_INVALID;
    A.ow[q] = out_dims[q].w;
    A.oh[q] = out_dims[q].h;
  }
  const NmsWs L = nms_ws_layout(F, max_boxes);
  if (!d_ws || ws_bytes < L.total) return MP_ERR_INVALID;
  unsigned char* ws = (unsigned char*)d_ws;
  mp_box* ws_box = (mp_box*)(ws + L.box_off);
  int* ws_src = (int*)(ws + L.src_off);
  int* ws_kept = (int*)(ws + L.kept_off);
  int* lcnt = (int*)(ws + L.lcnt_off);
  int* llist = (int*)(ws + L.llist_off);
  int* mcnt = lcnt + 1;
  int* mlist = (int*)(ws + L.mlist_off);
  NmsGlobal g;
  g.bx = (float4*)(ws + L.gbx_off);
  g.cls = (int*)(ws + L.gcls_off);
  g.score = (float*)(ws + L.gscore_off);
  g.src = (int*)(ws + L.gsrc_off);
  g.key = (unsigned long long*)(ws + L.gkey_off);
  g.key2 = (unsigned long long*)(ws + L.gkey2_off);
  g.keep = (int*)(ws + L.gkeep_off);
  g.supp = (unsigned char*)(ws + L.gsupp_off);
  cudaStream_t s = (cudaStream_t)stream;
  if (F > 0) {
    MP_CUDA_TRY(cudaMemsetAsync(lcnt, 0, 2 * sizeof(int), s));
    for (const void* k : {(const void*)nms_tiny_kernel, (const void*)nms_small_kernel,
                          (const void*)nms_large_kernel, (const void*)nms_scan_kernel,
                          (const void*)nms_scatter_kernel})
      MP_CUDA_TRY(prefer_max_shared(k));
    const size_t sm_small = nms_smem_bytes(kSmallCap, kSmallMaskCap, nullptr, nullptr);
    const size_t sm_large = nms_smem_bytes(kLargeCap, kLargeMaskCap, nullptr, nullptr);
    MP_CUDA_TRY(cudaFuncSetAttribute(nms_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_small));
    MP_CUDA_TRY(cudaFuncSetAttribute(nms_large_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_large));
    nms_tiny_kernel<<<(F + kTinyWarps - 1) / kTinyWarps, 32 * kTinyWarps, 0, s>>>(
        A, d_boxes, d_win_box_off, d_windows, d_frame_off, ws_box, ws_src, ws_kept, mcnt, mlist, d_status);
    MP_CUDA_TRY(cudaGetLastError());
    int dev = 0, sms = 0;
    MP_CUDA_TRY(cudaGetDevice(&dev));
    MP_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    nms_small_kernel<<<sms * 6, kSmallThreads, sm_small, s>>>(A, d_boxes, d_win_box_off, d_windows, d_frame_off,
                                                             ws_box, ws_src, ws_kept, mcnt, mlist, lcnt, llist,
                                                             d_status);
    MP_CUDA_TRY(cudaGetLastError());
    nms_large_kernel<<<sms * 2, kLargeThreads, sm_large, s>>>(A, d_boxes, d_win_box_off, d_windows, d_frame_off,
                                                          ws_box, ws_src, ws_kept, lcnt, llist, g, d_status);
    MP_CUDA_TRY(cudaGetLastError());
  }
  nms_scan_kernel<<<1, kScanThreads, 0, s>>>(F, ws_kept, d_out_frame_off, max_out, d_status);
  MP_CUDA_TRY(cudaGetLastError());
  if (F > 0) {
    nms_scatter_kernel<<<(F + 7) / 8, 256, 0, s>>>(F, d_frame_off, d_win_box_off, ws_box, ws_src, ws_kept,
                                                   d_out_frame_off, d_out, d_out_src, max_out, max_windows);
    MP_CUDA_TRY(cudaGetLastError());
  }
  return MP_OK;
}
