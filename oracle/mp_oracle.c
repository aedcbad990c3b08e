/*
 * mp_oracle.c — CPU ORACLE for the MultiScope proxy-guided window path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2103_14695_b200/) never links, imports or calls it,
 * and shares no code, header, table or helper with it.
 *
 * It is a plain, slow, obviously-correct C99 implementation of what the path
 * computes, written from the paper (PAPER.md = arXiv 2103.14695 LaTeX source)
 * and from the readings recorded in DESIGN.md §3 where the paper is silent.
 * Floating point: fp64 wherever the paper does not fix a precision, except
 * where an integer or ordering decision must be taken in the same precision as
 * the CUDA path (the threshold compare in fp32, NMS IoU in fp32, remap's final
 * fp32 rounding) — each such place says so.  Build with -O2 -ffp-contract=off.
 *
 * Pins (what ties this oracle to something other than itself) are listed in
 * tests/test_oracle_*.py and DESIGN.md §4.  Every function here is pinned;
 * there is no "parity unpinned" function.
 *
 * Citations: "P:n" = PAPER.md line n; "Rn" = reading n in DESIGN.md §3.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Own types (the oracle includes no product header).  Layouts are plain
 * int32/float records: window = 7 x int32, box = 5 x float + int32. */
typedef struct { int32_t w, h; } mpo_size;
typedef struct { int32_t frame, x, y, w, h, size_idx, slot; } mpo_window;
typedef struct { float x1, y1, x2, y2, score; int32_t cls; } mpo_box;

enum { MPO_OK = 0, MPO_ERR_INVALID = 1, MPO_ERR_CAPACITY = 3 };
enum { MPO_F32_NCHW = 0, MPO_U8_NHWC = 1, MPO_F64_NCHW = 2 };

/* ------------------------------------------------------------------------ */
/* a1. Threshold — P:150 "where the score exceeds a threshold parameter
 * B_proxy", "a binary grid consisting of a (possibly empty) set of
 * positive cells where the output scores exceeded B_proxy".  Reading R2:
 * strict ">", compared in fp32 (the scores' own precision); NaN is never
 * positive.  pos[r*C+c] = 1/0.  Returns the number of positive cells. */
int64_t mpo_threshold(const float* scores, int32_t R, int32_t C, float b_proxy, uint8_t* pos) {
  int64_t n = 0;
  for (int32_t r = 0; r < R; r++)
    for (int32_t c = 0; c < C; c++) {
      float s = scores[(int64_t)r * C + c];
      pos[(int64_t)r * C + c] = (s > b_proxy) ? 1 : 0;
      n += pos[(int64_t)r * C + c];
    }
  return n;
}

/* Bit-pack a positive grid: bit (c%32) of word c/32 of row r.  (ABI layout of
 * d_mask, include/mp.h.) */
void mpo_pack_mask(const uint8_t* pos, int32_t R, int32_t C, uint32_t* mask) {
  int32_t words = (C + 31) / 32;
  for (int32_t r = 0; r < R; r++)
    for (int32_t wd = 0; wd < words; wd++) {
      uint32_t m = 0;
      for (int32_t bit = 0; bit < 32; bit++) {
        int32_t c = wd * 32 + bit;
        if (c < C && pos[(int64_t)r * C + c]) m |= (1u << bit);
      }
      mask[(int64_t)r * words + wd] = m;
    }
}

/* ------------------------------------------------------------------------ */
/* a2. Connected components — P:184 "We initialize a cluster C_i for each
 * connected component of positive cells".  Reading R3: 4-connectivity;
 * components numbered in order of their first cell in a row-major scan.
 * Plain definition: flood fill (BFS) started from each unlabelled positive
 * cell in raster order.  labels[r*C+c] = component id or -1.  bbox[4*i..] =
 * (c0, r0, c1, r1), inclusive cell coordinates.  Returns the component count. */
int32_t mpo_components(const uint8_t* pos, int32_t R, int32_t C, int32_t* labels, int32_t* bbox) {
  int64_t N = (int64_t)R * C;
  int32_t* queue = (int32_t*)malloc(sizeof(int32_t) * (N > 0 ? N : 1));
  int32_t ncomp = 0;
  for (int64_t i = 0; i < N; i++) labels[i] = -1;
  for (int32_t r = 0; r < R; r++) {
    for (int32_t c = 0; c < C; c++) {
      int64_t start = (int64_t)r * C + c;
      if (!pos[start] || labels[start] >= 0) continue;
      int32_t id = ncomp++;
      int32_t c0 = c, r0 = r, c1 = c, r1 = r;
      int64_t head = 0, tail = 0;
      labels[start] = id;
      queue[tail++] = (int32_t)start;
      while (head < tail) {
        int32_t cell = queue[head++];
        int32_t cr = cell / C, cc = cell % C;
        if (cc < c0) c0 = cc;
        if (cc > c1) c1 = cc;
        if (cr < r0) r0 = cr;
        if (cr > r1) r1 = cr;
        /* the four edge neighbours: up, down, left, right */
        int32_t nr[4] = {cr - 1, cr + 1, cr, cr};
        int32_t nc[4] = {cc, cc, cc - 1, cc + 1};
        for (int q = 0; q < 4; q++) {
          if (nr[q] < 0 || nr[q] >= R || nc[q] < 0 || nc[q] >= C) continue;
          int64_t nb = (int64_t)nr[q] * C + nc[q];
          if (pos[nb] && labels[nb] < 0) {
            labels[nb] = id;
            queue[tail++] = (int32_t)nb;
          }
        }
      }
      bbox[4 * id + 0] = c0;
      bbox[4 * id + 1] = r0;
      bbox[4 * id + 2] = c1;
      bbox[4 * id + 3] = r1;
    }
  }
  free(queue);
  return ncomp;
}

/* ------------------------------------------------------------------------ */
/* Planner geometry.  Reading R1: a cell is cell_w x cell_h frame px, the last
 * row/column clipped to the frame.  Pixel bbox of a cell bbox (c0,r0,c1,r1):
 * [c0*cw, min((c1+1)*cw, W)) x [r0*ch, min((r1+1)*ch, H)). */
typedef struct {
  int32_t W, H, cw, ch, k;
  const mpo_size* sizes;
  const int64_t* cost;
} mpo_plan_ctx;

static void pix_extent(const mpo_plan_ctx* P, int32_t c0, int32_t r0, int32_t c1, int32_t r1,
                       int32_t* px0, int32_t* py0, int32_t* bw, int32_t* bh) {
  int32_t x0 = c0 * P->cw, y0 = r0 * P->ch;
  int32_t x1 = (c1 + 1) * P->cw, y1 = (r1 + 1) * P->ch;
  if (x1 > P->W) x1 = P->W;
  if (y1 > P->H) y1 = P->H;
  *px0 = x0;
  *py0 = y0;
  *bw = x1 - x0;
  *bh = y1 - y0;
}

/* P:184 "identify the smallest-area window size (w,h) that contains the
 * bounding box".  Reading R6: among sizes with w_i >= bw and h_i >= bh,
 * minimise (w_i*h_i, w_i, h_i).  Returns the index, or -1 if none fits (never
 * happens for a validated S, which contains (W,H)). */
int32_t mpo_smallest_window(const mpo_size* sizes, int32_t k, int32_t bw, int32_t bh) {
  int32_t best = -1;
  for (int32_t i = 0; i < k; i++) {
    if (sizes[i].w < bw || sizes[i].h < bh) continue;
    if (best < 0) { best = i; continue; }
    int64_t ai = (int64_t)sizes[i].w * sizes[i].h, ab = (int64_t)sizes[best].w * sizes[best].h;
    if (ai < ab || (ai == ab && (sizes[i].w < sizes[best].w ||
                                 (sizes[i].w == sizes[best].w && sizes[i].h < sizes[best].h))))
      best = i;
  }
  return best;
}

typedef struct { int32_t c0, r0, c1, r1, size; } cluster;

static int32_t cluster_size(const mpo_plan_ctx* P, int32_t c0, int32_t r0, int32_t c1, int32_t r1) {
  int32_t px0, py0, bw, bh;
  pix_extent(P, c0, r0, c1, r1, &px0, &py0, &bw, &bh);
  return mpo_smallest_window(P->sizes, P->k, bw, bh);
}

static int fits(const mpo_plan_ctx* P, int32_t c0, int32_t r0, int32_t c1, int32_t r1, int32_t s) {
  int32_t px0, py0, bw, bh;
  pix_extent(P, c0, r0, c1, r1, &px0, &py0, &bw, &bh);
  return bw <= P->sizes[s].w && bh <= P->sizes[s].h;
}

static int32_t imin(int32_t a, int32_t b) { return a < b ? a : b; }
static int32_t imax(int32_t a, int32_t b) { return a > b ? a : b; }

/*
 * a3 + a4 for one frame, from its component bounding boxes (in label order).
 * The greedy of P:184, step by step ("Grouping Cells during Execution"):
 *   "We then iterate over the clusters.  For each cluster C_i, we identify its
 *    closest neighbor C_j [R5: squared distance of bbox centres, ties -> the
 *    smallest list position].  We create a proposed merged cluster C_merged,
 *    and identify the smallest-area window size (w,h) that contains the
 *    bounding box of C_merged [R6].  For every other cluster C_k, we check if
 *    we can add C_k to C_merged without needing a larger window size [R7:
 *    k ascending, absorbed at once].  Finally ... we compare ... T_{w,h} with
 *    the sum of the time to process the individual clusters ... If the
 *    execution time for C_merged is smaller [R8: strict <], then we remove the
 *    individual clusters and add C_merged [R4: appended at the end].  We
 *    repeatedly loop over the clusters until we perform a pass without any new
 *    merges [R9]."
 *   P:186 "we construct a set of rectangular windows R by creating one
 *    rectangle for each cluster" — placement R10 (centred, clamped).
 *   R11: if est(R) > T[full] the plan becomes one full-frame window.
 *   R12: no components -> no windows.
 * Writes up to n_comp windows (frame, x, y, w, h, size_idx; slot = -1) and
 * returns the count.  *passes_out (optional) = number of passes run.
 */
int32_t mpo_plan_frame(const mpo_plan_ctx* P, const int32_t* comp_bbox, int32_t n_comp,
                       int32_t frame, mpo_window* out, int32_t* passes_out) {
  int32_t passes = 0;
  if (n_comp == 0) {
    if (passes_out) *passes_out = 0;
    return 0;
  }
  cluster* L = (cluster*)malloc(sizeof(cluster) * n_comp);
  uint8_t* member = (uint8_t*)malloc(n_comp);
  int32_t n = n_comp;
  for (int32_t i = 0; i < n; i++) {
    L[i].c0 = comp_bbox[4 * i + 0];
    L[i].r0 = comp_bbox[4 * i + 1];
    L[i].c1 = comp_bbox[4 * i + 2];
    L[i].r1 = comp_bbox[4 * i + 3];
    L[i].size = cluster_size(P, L[i].c0, L[i].r0, L[i].c1, L[i].r1);
  }
  int merged_in_pass = 1;
  while (merged_in_pass) {
    merged_in_pass = 0;
    passes++;
    int32_t i = 0;
    while (i < n && n >= 2) {
      /* (a) closest neighbour j != i; distance between bbox centres, in
       * doubled-cell units: centre_x*2 = c0 + c1 + 1 (the +1 cancels). */
      int32_t j = -1;
      int64_t best_d = 0;
      for (int32_t q = 0; q < n; q++) {
        if (q == i) continue;
        int64_t dx = (int64_t)(L[i].c0 + L[i].c1) - (L[q].c0 + L[q].c1);
        int64_t dy = (int64_t)(L[i].r0 + L[i].r1) - (L[q].r0 + L[q].r1);
        int64_t d = dx * dx + dy * dy;
        if (j < 0 || d < best_d) { j = q; best_d = d; }
      }
      /* (b) proposed merge and its smallest containing window size */
      int32_t mc0 = imin(L[i].c0, L[j].c0), mr0 = imin(L[i].r0, L[j].r0);
      int32_t mc1 = imax(L[i].c1, L[j].c1), mr1 = imax(L[i].r1, L[j].r1);
      int32_t s = cluster_size(P, mc0, mr0, mc1, mr1);
      memset(member, 0, n);
      member[i] = member[j] = 1;
      /* (c) absorb every other cluster that fits without a larger window */
      for (int32_t q = 0; q < n; q++) {
        if (member[q]) continue;
        int32_t nc0 = imin(mc0, L[q].c0), nr0 = imin(mr0, L[q].r0);
        int32_t nc1 = imax(mc1, L[q].c1), nr1 = imax(mr1, L[q].r1);
        if (fits(P, nc0, nr0, nc1, nr1, s)) {
          mc0 = nc0; mr0 = nr0; mc1 = nc1; mr1 = nr1;
          member[q] = 1;
        }
      }
      /* (d) accept iff T_merged < sum of the members' individual times */
      int64_t sum = 0;
      for (int32_t q = 0; q < n; q++)
        if (member[q]) sum += P->cost[L[q].size];
      if (P->cost[s] < sum) {
        int32_t before_i = 0, w = 0;
        for (int32_t q = 0; q < n; q++) {
          if (member[q]) {
            if (q < i) before_i++;
            continue;
          }
          L[w++] = L[q];
        }
        L[w].c0 = mc0; L[w].r0 = mr0; L[w].c1 = mc1; L[w].r1 = mr1; L[w].size = s;
        n = w + 1;
        i -= before_i;
        merged_in_pass = 1;
      } else {
        i++;
      }
    }
  }
  if (passes_out) *passes_out = passes;

  /* R11 full-frame fallback */
  int32_t full = -1;
  for (int32_t q = 0; q < P->k; q++)
    if (P->sizes[q].w == P->W && P->sizes[q].h == P->H) full = q;
  int64_t est = 0;
  for (int32_t q = 0; q < n; q++) est += P->cost[L[q].size];
  int32_t nw;
  if (est > P->cost[full]) {
    out[0].frame = frame; out[0].x = 0; out[0].y = 0;
    out[0].w = P->W; out[0].h = P->H; out[0].size_idx = full; out[0].slot = -1;
    nw = 1;
  } else {
    /* a4 placement, R10: centre the window on the bbox, clamp into frame */
    for (int32_t q = 0; q < n; q++) {
      int32_t px0, py0, bw, bh;
      pix_extent(P, L[q].c0, L[q].r0, L[q].c1, L[q].r1, &px0, &py0, &bw, &bh);
      int32_t ws = P->sizes[L[q].size].w, hs = P->sizes[L[q].size].h;
      int32_t x = px0 - (ws - bw) / 2;   /* ws >= bw, so / is floor */
      int32_t y = py0 - (hs - bh) / 2;
      if (x > P->W - ws) x = P->W - ws;
      if (x < 0) x = 0;
      if (y > P->H - hs) y = P->H - hs;
      if (y < 0) y = 0;
      out[q].frame = frame; out[q].x = x; out[q].y = y; out[q].w = ws; out[q].h = hs;
      out[q].size_idx = L[q].size; out[q].slot = -1;
    }
    nw = n;
  }
  free(L);
  free(member);
  return nw;
}

/* Host-side validation shared in meaning (not in code) with the ABI. */
static int plan_params_ok(int32_t W, int32_t H, int32_t cw, int32_t ch, int32_t k,
                          const mpo_size* sizes, const int64_t* cost) {
  if (W < 1 || H < 1 || cw < 1 || ch < 1 || k < 1 || k > 16 || !sizes || !cost) return 0;
  int full = 0;
  for (int32_t i = 0; i < k; i++) {
    if (sizes[i].w < 1 || sizes[i].h < 1 || sizes[i].w > W || sizes[i].h > H || cost[i] <= 0)
      return 0;
    if (sizes[i].w == W && sizes[i].h == H) full = 1;
    for (int32_t j = 0; j < k; j++) {
      if (i == j) continue;
      if (sizes[i].w == sizes[j].w && sizes[i].h == sizes[j].h) return 0;
      int64_t ai = (int64_t)sizes[i].w * sizes[i].h, aj = (int64_t)sizes[j].w * sizes[j].h;
      if (ai < aj && !(cost[i] < cost[j])) return 0;
    }
  }
  return full;
}

/*
 * Batched a1-a4 with the ABI's semantics (include/mp.h mp_plan_windows), on
 * host pointers.  windows: frame ascending, then list order; slot = rank among
 * the windows of the same size in that global order; frame_off CSR.
 * passes (optional, [F]) receives the merge pass count per frame.
 */
int32_t mpo_plan_windows(int32_t W, int32_t H, int32_t cw, int32_t ch, float b_proxy, int32_t k,
                         const mpo_size* sizes, const int64_t* cost, const float* scores,
                         int32_t F, uint32_t* mask, mpo_window* windows, int32_t max_windows,
                         int32_t* frame_off, int32_t* class_count, int32_t* passes) {
  if (!plan_params_ok(W, H, cw, ch, k, sizes, cost) || F < 0) return MPO_ERR_INVALID;
  int32_t R = (H + ch - 1) / ch, C = (W + cw - 1) / cw;
  int64_t N = (int64_t)R * C;
  mpo_plan_ctx P = {W, H, cw, ch, k, sizes, cost};
  uint8_t* pos = (uint8_t*)malloc(N);
  int32_t* labels = (int32_t*)malloc(sizeof(int32_t) * N);
  int32_t* bbox = (int32_t*)malloc(sizeof(int32_t) * 4 * N);
  mpo_window* fw = (mpo_window*)malloc(sizeof(mpo_window) * (N > 0 ? N : 1));
  int status = MPO_OK;
  int32_t total = 0;
  for (int32_t q = 0; q < k; q++) class_count[q] = 0;
  for (int32_t f = 0; f < F; f++) {
    const float* sc = scores + (int64_t)f * N;
    mpo_threshold(sc, R, C, b_proxy, pos);
    if (mask) mpo_pack_mask(pos, R, C, mask + (int64_t)f * R * ((C + 31) / 32));
    int32_t nc = mpo_components(pos, R, C, labels, bbox);
    int32_t pf = 0;
    int32_t nw = mpo_plan_frame(&P, bbox, nc, f, fw, &pf);
    if (passes) passes[f] = pf;
    frame_off[f] = total;
    for (int32_t q = 0; q < nw; q++) {
      fw[q].slot = class_count[fw[q].size_idx]++;
      if (total < max_windows) windows[total] = fw[q];
      else status = MPO_ERR_CAPACITY;
      total++;
    }
  }
  frame_off[F] = total;
  free(pos); free(labels); free(bbox); free(fw);
  return status;
}

/* ------------------------------------------------------------------------ */
/* a5. Gather + bilinear resize.  The paper never resizes (it decodes at the
 * detector resolution, and runs the detector "at each of those
 * sizes"); reading R15 fixes the convention: half-pixel centres
 * (align_corners=False), taps clamped to the crop, exact integer taps:
 *   n = (2d+1)*in - out;  n < 0 -> (i0=0, lambda=0);
 *   else i0 = floor(n / 2out), lambda = (n mod 2out) / 2out;
 *   i0 >= in-1 -> (i0=in-1, lambda=0);  i1 = min(i0+1, in-1).
 * Value (fp64): v = (1-ly)[(1-lx)p00 + lx p01] + ly[(1-lx)p10 + lx p11].
 * f32 out = v (0..255 scale, NCHW); u8 out = clamp(floor(v+0.5), 0, 255)
 * (R16, NHWC); f64 out (oracle only, for pins) = v, NCHW. */
void mpo_taps(int32_t in, int32_t out, int32_t d, int32_t* i0, int32_t* i1, double* lam) {
  int64_t n = (int64_t)(2 * (int64_t)d + 1) * in - out;
  int64_t a, rem;
  if (n < 0) {
    a = 0;
    rem = 0;
  } else {
    a = n / (2 * (int64_t)out);
    rem = n % (2 * (int64_t)out);
  }
  if (a >= in - 1) {
    a = in - 1;
    rem = 0;
  }
  *i0 = (int32_t)a;
  *i1 = (int32_t)(a + 1 < in - 1 ? a + 1 : in - 1);
  *lam = (double)rem / (double)(2 * (int64_t)out);
}

int32_t mpo_gather_resize(const uint8_t* const* frames, int32_t pitch, int32_t W, int32_t H,
                          int32_t F, const mpo_window* windows, int32_t n_win, int32_t k,
                          const mpo_size* sizes, const mpo_size* out_dims, void* const* out,
                          const int32_t* out_cap, int32_t fmt) {
  int status = MPO_OK;
  for (int32_t wi = 0; wi < n_win; wi++) {
    mpo_window win = windows[wi];
    if (win.frame < 0 || win.frame >= F || win.size_idx < 0 || win.size_idx >= k ||
        win.w != sizes[win.size_idx].w || win.h != sizes[win.size_idx].h || win.x < 0 ||
        win.y < 0 || win.x + win.w > W || win.y + win.h > H || win.slot < 0) {
      status = MPO_ERR_INVALID;
      continue;
    }
    int32_t kk = win.size_idx;
    if (win.slot >= out_cap[kk]) {
      status = MPO_ERR_CAPACITY;
      continue;
    }
    int32_t ow = out_dims[kk].w, oh = out_dims[kk].h;
    const uint8_t* fr = frames[win.frame];
    for (int32_t oy = 0; oy < oh; oy++) {
      int32_t y0, y1;
      double ly;
      mpo_taps(win.h, oh, oy, &y0, &y1, &ly);
      for (int32_t ox = 0; ox < ow; ox++) {
        int32_t x0, x1;
        double lx;
        mpo_taps(win.w, ow, ox, &x0, &x1, &lx);
        for (int32_t c = 0; c < 3; c++) {
          double p00 = fr[(int64_t)(win.y + y0) * pitch + (int64_t)(win.x + x0) * 3 + c];
          double p01 = fr[(int64_t)(win.y + y0) * pitch + (int64_t)(win.x + x1) * 3 + c];
          double p10 = fr[(int64_t)(win.y + y1) * pitch + (int64_t)(win.x + x0) * 3 + c];
          double p11 = fr[(int64_t)(win.y + y1) * pitch + (int64_t)(win.x + x1) * 3 + c];
          double v = (1.0 - ly) * ((1.0 - lx) * p00 + lx * p01) + ly * ((1.0 - lx) * p10 + lx * p11);
          int64_t plane = (int64_t)oh * ow;
          if (fmt == MPO_F32_NCHW) {
            float* o = (float*)out[kk];
            o[((int64_t)win.slot * 3 + c) * plane + (int64_t)oy * ow + ox] = (float)v;
          } else if (fmt == MPO_F64_NCHW) {
            double* o = (double*)out[kk];
            o[((int64_t)win.slot * 3 + c) * plane + (int64_t)oy * ow + ox] = v;
          } else {
            uint8_t* o = (uint8_t*)out[kk];
            double r = floor(v + 0.5);
            if (r < 0) r = 0;
            if (r > 255) r = 255;
            o[(((int64_t)win.slot * oh + oy) * ow + ox) * 3 + c] = (uint8_t)r;
          }
        }
      }
    }
  }
  return status;
}

/* ------------------------------------------------------------------------ */
/* NEXT-3: decode-native input.  The paper decodes
 * with ffmpeg "at the object detector resolution" and feeds the proxy a
 * low-resolution frame; it names no pixel format.  Reading R23
 * (DESIGN.md §3): the decoder's output is NV12 — a Y plane [H][pitch] followed
 * by an interleaved chroma plane [H/2][pitch] (U at even bytes, V at odd
 * bytes), W and H even; chroma sample (i, j) covers luma (2i..2i+1, 2j..2j+1),
 * i.e. the chroma value seen at luma position (r, c) is U[r>>1][2(c>>1)].
 * Each of Y, U, V is resampled with the R15 taps of the luma grid exactly as
 * one RGB channel is in mpo_gather_resize, then converted (ITU-R BT.601 /
 * BT.709 Y'CbCr -> R'G'B' definitions, 8-bit):
 *   Y' = (Y - yo) / ys,  Pb = (U - 128) / cs,  Pr = (V - 128) / cs
 *   limited range: yo = 16, ys = 219, cs = 224;  full range: yo = 0, ys = cs = 255
 *   R = 255 [Y' + 2(1-Kr) Pr]
 *   G = 255 [Y' - 2Kb(1-Kb)/Kg Pb - 2Kr(1-Kr)/Kg Pr],  Kg = 1 - Kr - Kb
 *   B = 255 [Y' + 2(1-Kb) Pb]
 * then clamped to [0, 255]; f32/f64 out = clamped value, u8 out =
 * floor(v + 0.5) (R16).  matrix 0 = BT.709 limited (Kr .2126, Kb .0722),
 * 1 = BT.601 limited (Kr .299, Kb .114), 2 = BT.709 full, 3 = BT.601 full. */
int32_t mpo_yuv_to_rgb(double Y, double U, double V, int32_t matrix, double* rgb) {
  double Kr, Kb, yo, ys, cs;
  if (matrix < 0 || matrix > 3) return MPO_ERR_INVALID;
  Kr = (matrix & 1) ? 0.299 : 0.2126;
  Kb = (matrix & 1) ? 0.114 : 0.0722;
  if (matrix < 2) {
    yo = 16.0;
    ys = 219.0;
    cs = 224.0;
  } else {
    yo = 0.0;
    ys = 255.0;
    cs = 255.0;
  }
  double Kg = 1.0 - Kr - Kb;
  double y = (Y - yo) / ys, pb = (U - 128.0) / cs, pr = (V - 128.0) / cs;
  double r = 255.0 * (y + 2.0 * (1.0 - Kr) * pr);
  double g = 255.0 * (y - 2.0 * Kb * (1.0 - Kb) / Kg * pb - 2.0 * Kr * (1.0 - Kr) / Kg * pr);
  double b = 255.0 * (y + 2.0 * (1.0 - Kb) * pb);
  double v[3] = {r, g, b};
  for (int c = 0; c < 3; c++) rgb[c] = v[c] < 0.0 ? 0.0 : (v[c] > 255.0 ? 255.0 : v[c]);
  return MPO_OK;
}

int32_t mpo_gather_resize_nv12(const uint8_t* const* frames, int32_t pitch, int32_t W, int32_t H,
                               int32_t F, const mpo_window* windows, int32_t n_win, int32_t k,
                               const mpo_size* sizes, const mpo_size* out_dims, void* const* out,
                               const int32_t* out_cap, int32_t fmt, int32_t matrix) {
  int status = MPO_OK;
  if ((W & 1) || (H & 1) || pitch < W || matrix < 0 || matrix > 3) return MPO_ERR_INVALID;
  for (int32_t wi = 0; wi < n_win; wi++) {
    mpo_window win = windows[wi];
    if (win.frame < 0 || win.frame >= F || win.size_idx < 0 || win.size_idx >= k ||
        win.w != sizes[win.size_idx].w || win.h != sizes[win.size_idx].h || win.x < 0 ||
        win.y < 0 || win.x + win.w > W || win.y + win.h > H || win.slot < 0) {
      status = MPO_ERR_INVALID;
      continue;
    }
    int32_t kk = win.size_idx;
    if (win.slot >= out_cap[kk]) {
      status = MPO_ERR_CAPACITY;
      continue;
    }
    int32_t ow = out_dims[kk].w, oh = out_dims[kk].h;
    const uint8_t* Yp = frames[win.frame];
    const uint8_t* UVp = Yp + (int64_t)H * pitch;
    for (int32_t oy = 0; oy < oh; oy++) {
      int32_t y0, y1;
      double ly;
      mpo_taps(win.h, oh, oy, &y0, &y1, &ly);
      int64_t r0 = win.y + y0, r1 = win.y + y1;
      for (int32_t ox = 0; ox < ow; ox++) {
        int32_t x0, x1;
        double lx;
        mpo_taps(win.w, ow, ox, &x0, &x1, &lx);
        int64_t c0 = win.x + x0, c1 = win.x + x1;
        double yuv[3], rgb[3];
        for (int32_t ch = 0; ch < 3; ch++) {
          double p00, p01, p10, p11;
          if (ch == 0) {
            p00 = Yp[r0 * pitch + c0];
            p01 = Yp[r0 * pitch + c1];
            p10 = Yp[r1 * pitch + c0];
            p11 = Yp[r1 * pitch + c1];
          } else {   /* U (ch 1) at byte 2(c>>1), V (ch 2) at 2(c>>1)+1 of chroma row r>>1 */
            int32_t o = ch - 1;
            p00 = UVp[(r0 >> 1) * pitch + 2 * (c0 >> 1) + o];
            p01 = UVp[(r0 >> 1) * pitch + 2 * (c1 >> 1) + o];
            p10 = UVp[(r1 >> 1) * pitch + 2 * (c0 >> 1) + o];
            p11 = UVp[(r1 >> 1) * pitch + 2 * (c1 >> 1) + o];
          }
          yuv[ch] = (1.0 - ly) * ((1.0 - lx) * p00 + lx * p01) + ly * ((1.0 - lx) * p10 + lx * p11);
        }
        mpo_yuv_to_rgb(yuv[0], yuv[1], yuv[2], matrix, rgb);
        int64_t plane = (int64_t)oh * ow;
        for (int32_t c = 0; c < 3; c++) {
          double v = rgb[c];
          if (fmt == MPO_F32_NCHW) {
            ((float*)out[kk])[((int64_t)win.slot * 3 + c) * plane + (int64_t)oy * ow + ox] = (float)v;
          } else if (fmt == MPO_F64_NCHW) {
            ((double*)out[kk])[((int64_t)win.slot * 3 + c) * plane + (int64_t)oy * ow + ox] = v;
          } else {
            ((uint8_t*)out[kk])[(((int64_t)win.slot * oh + oy) * ow + ox) * 3 + c] = (uint8_t)floor(v + 0.5);
          }
        }
      }
    }
  }
  return status;
}

/* ------------------------------------------------------------------------ */
/* a6. Remap one detector box (reading R18; not in the paper).  Returns 0 if
 * the box is dropped.  Steps: keep iff score > score_thr (NaN dropped);
 * clip each coordinate to [0,ow] / [0,oh] with fmin/fmax (a NaN coordinate
 * becomes the bound); drop if x2 <= x1 or y2 <= y1; map each coordinate
 * X = fp32( (x_l * w) / ow + x ) with the product, quotient and sum each
 * rounded in fp64 (the product is exact) and one final rounding to fp32. */
int32_t mpo_remap_box(mpo_box in, int32_t wx, int32_t wy, int32_t ww, int32_t wh, int32_t ow,
                      int32_t oh, float score_thr, mpo_box* out) {
  if (!(in.score > score_thr)) return 0;
  float x1 = fminf(fmaxf(in.x1, 0.0f), (float)ow);
  float x2 = fminf(fmaxf(in.x2, 0.0f), (float)ow);
  float y1 = fminf(fmaxf(in.y1, 0.0f), (float)oh);
  float y2 = fminf(fmaxf(in.y2, 0.0f), (float)oh);
  if (!(x2 > x1) || !(y2 > y1)) return 0;
  volatile double t;
  t = (double)x1 * (double)ww; t = t / (double)ow; t = t + (double)wx; out->x1 = (float)t;
  t = (double)y1 * (double)wh; t = t / (double)oh; t = t + (double)wy; out->y1 = (float)t;
  t = (double)x2 * (double)ww; t = t / (double)ow; t = t + (double)wx; out->x2 = (float)t;
  t = (double)y2 * (double)wh; t = t / (double)oh; t = t + (double)wy; out->y2 = (float)t;
  out->score = in.score;
  out->cls = in.cls;
  return 1;
}

/* a7 IoU in fp32, every operation rounded, none contracted (reading R19, the
 * formula order of torchvision's CPU nms kernel). */
float mpo_iou(mpo_box a, mpo_box b) {
  volatile float area_a = (a.x2 - a.x1) * (a.y2 - a.y1);
  volatile float area_b = (b.x2 - b.x1) * (b.y2 - b.y1);
  float xx1 = fmaxf(a.x1, b.x1), yy1 = fmaxf(a.y1, b.y1);
  float xx2 = fminf(a.x2, b.x2), yy2 = fminf(a.y2, b.y2);
  volatile float iw = xx2 - xx1;
  volatile float ih = yy2 - yy1;
  if (iw < 0.0f) iw = 0.0f;
  if (ih < 0.0f) ih = 0.0f;
  volatile float inter = iw * ih;
  volatile float uni = area_a + area_b;
  uni = uni - inter;
  volatile float r = inter / uni;
  return r;
}

typedef struct { float score; int32_t q; } cand_key;

static int cand_cmp(const void* pa, const void* pb) {
  const cand_key* a = (const cand_key*)pa;
  const cand_key* b = (const cand_key*)pb;
  /* score descending in fp32 value order (-0.0 == +0.0), then q ascending */
  if (a->score > b->score) return -1;
  if (a->score < b->score) return 1;
  return (a->q < b->q) ? -1 : (a->q > b->q);
}

/*
 * Batched a6+a7 with the ABI's semantics (include/mp.h mp_remap_nms) on host
 * pointers.  Per frame: the candidates are the boxes of the frame's windows
 * (window order, then box order) that survive remap; candidate index q =
 * global input box index.  Sort by (score desc, q asc); greedy: take each
 * not-yet-suppressed candidate in order, keep it, suppress every later
 * candidate of the same cls with IoU > iou_thr (strict).
 */
int32_t mpo_remap_nms(const mpo_box* boxes, const int32_t* win_box_off, const mpo_window* windows,
                      const int32_t* frame_off, int32_t F, int32_t k, const mpo_size* out_dims,
                      int32_t W, int32_t H, float score_thr, float iou_thr, mpo_box* out,
                      int32_t* out_src, int32_t max_out, int32_t* out_frame_off) {
  (void)W;
  (void)H;
  int status = MPO_OK;
  int32_t total = 0;
  for (int32_t f = 0; f < F; f++) {
    out_frame_off[f] = total;
    int32_t w_lo = frame_off[f], w_hi = frame_off[f + 1];
    int32_t b_lo = win_box_off[w_lo], b_hi = win_box_off[w_hi];
    int32_t nmax = b_hi - b_lo;
    if (nmax <= 0) continue;
    mpo_box* cb = (mpo_box*)malloc(sizeof(mpo_box) * nmax);
    int32_t* csrc = (int32_t*)malloc(sizeof(int32_t) * nmax);
    cand_key* key = (cand_key*)malloc(sizeof(cand_key) * nmax);
    uint8_t* supp = (uint8_t*)calloc(nmax, 1);
    int32_t n = 0;
    for (int32_t wi = w_lo; wi < w_hi; wi++) {
      mpo_window win = windows[wi];
      if (win.size_idx < 0 || win.size_idx >= k) { status = MPO_ERR_INVALID; continue; }
      int32_t ow = out_dims[win.size_idx].w, oh = out_dims[win.size_idx].h;
      for (int32_t b = win_box_off[wi]; b < win_box_off[wi + 1]; b++) {
        mpo_box r;
        if (mpo_remap_box(boxes[b], win.x, win.y, win.w, win.h, ow, oh, score_thr, &r)) {
          cb[n] = r;
          csrc[n] = b;
          key[n].score = (r.score == 0.0f) ? 0.0f : r.score; /* -0.0 -> +0.0 */
          key[n].q = n;
          n++;
        }
      }
    }
    qsort(key, n, sizeof(cand_key), cand_cmp);
    for (int32_t a = 0; a < n; a++) {
      int32_t ia = key[a].q;
      if (supp[ia]) continue;
      if (total < max_out) {
        out[total] = cb[ia];
        out_src[total] = csrc[ia];
      } else {
        status = MPO_ERR_CAPACITY;
      }
      total++;
      for (int32_t b = a + 1; b < n; b++) {
        int32_t ib = key[b].q;
        if (supp[ib] || cb[ib].cls != cb[ia].cls) continue;
        if (mpo_iou(cb[ia], cb[ib]) > iou_thr) supp[ib] = 1;
      }
    }
    free(cb); free(csrc); free(key); free(supp);
  }
  out_frame_off[F] = total;
  return status;
}

/* ------------------------------------------------------------------------ */
/* NEXT-1: proxy-module caching sweep, PAPER.md:281-283 (§3.5.2 "Proxy Model
 * Module"): "for each threshold B_j, we compute rectangular windows using the
 * cell grouping method ... on each frame ... our runtime estimate for this
 * resolution and threshold is T_proxy,i + sum_k T_{r_k.w,r_k.h} ... The recall
 * is the fraction of detections computed by theta_best that are covered by
 * rectangles in R_{i,j}."  Per threshold: plan all frames (mpo_plan_windows),
 * then per frame and detection test the frame's windows.  Reading R21:
 * covered = the detection lies inside a window; touched = positive-area
 * overlap.  out[5*j + {0..4}] = cost_sum, windows, full_frames,
 * dets_covered, dets_touched. */
int32_t mpo_proxy_sweep(int32_t W, int32_t H, int32_t cw, int32_t ch, int32_t k, const mpo_size* sizes,
                        const int64_t* cost, const float* scores, int32_t F, const float* thresholds,
                        int32_t J, const float* dets, const int32_t* det_off, int64_t* out) {
  int32_t R = (H + ch - 1) / ch, C = (W + cw - 1) / cw;
  int64_t maxw = (int64_t)F * ((int64_t)R * ((C + 1) / 2) + 1) + 1;
  mpo_window* win = (mpo_window*)malloc(sizeof(mpo_window) * maxw);
  int32_t* frame_off = (int32_t*)malloc(sizeof(int32_t) * (F + 1));
  int32_t* cc = (int32_t*)malloc(sizeof(int32_t) * (k > 0 ? k : 1));
  int32_t full = -1;
  for (int32_t q = 0; q < k; q++)
    if (sizes[q].w == W && sizes[q].h == H) full = q;
  int status = MPO_OK;
  for (int32_t j = 0; j < J && status == MPO_OK; j++) {
    int st = mpo_plan_windows(W, H, cw, ch, thresholds[j], k, sizes, cost, scores, F, NULL, win, (int32_t)maxw,
                              frame_off, cc, NULL);
    if (st != MPO_OK) { status = st; break; }
    int64_t* o = out + 5 * j;
    for (int32_t q = 0; q < 5; q++) o[q] = 0;
    for (int32_t f = 0; f < F; f++) {
      int32_t w0 = frame_off[f], w1 = frame_off[f + 1];
      for (int32_t wi = w0; wi < w1; wi++) o[0] += cost[win[wi].size_idx];
      o[1] += w1 - w0;
      if (w1 - w0 == 1 && win[w0].size_idx == full) o[2] += 1;
      for (int32_t d = det_off[f]; d < det_off[f + 1]; d++) {
        float x1 = dets[4 * d], y1 = dets[4 * d + 1], x2 = dets[4 * d + 2], y2 = dets[4 * d + 3];
        int in = 0, ov = 0;
        for (int32_t wi = w0; wi < w1; wi++) {
          float a0 = (float)win[wi].x, b0 = (float)win[wi].y;
          float a1 = (float)(win[wi].x + win[wi].w), b1 = (float)(win[wi].y + win[wi].h);
          if (x1 >= a0 && x2 <= a1 && y1 >= b0 && y2 <= b1) in = 1;
          if (x1 < a1 && x2 > a0 && y1 < b1 && y2 > b0) ov = 1;
        }
        o[3] += in;
        o[4] += ov;
      }
    }
  }
  free(win); free(frame_off); free(cc);
  return status;
}

/* ------------------------------------------------------------------------ */
/* NEXT-2: window-size selection objective, PAPER.md:190-195 ("Determining
 * Fixed Set of Window Sizes"): tot_time(S) = sum_t im_time(S, I_t),
 * im_time(S, I_t) = est(R(I_t; S)) with the cell grouping method of P:184 and
 * a perfect proxy (the caller passes 0/1 label grids).  For each candidate
 * (w,h): S' = S + {(w,h)}; tot[c] = sum over frames of est of the plan (after
 * the R11 fallback).  Plain loops over candidates and frames. */
int32_t mpo_window_set_cost(int32_t W, int32_t H, int32_t cw, int32_t ch, float b_proxy, int32_t k,
                            const mpo_size* sizes, const int64_t* cost, const float* scores, int32_t F,
                            const mpo_size* cand, const int64_t* cand_cost, int32_t n_cand, int64_t* tot) {
  int32_t R = (H + ch - 1) / ch, C = (W + cw - 1) / cw;
  int64_t maxw = (int64_t)F * ((int64_t)R * ((C + 1) / 2) + 1) + 1;
  mpo_window* win = (mpo_window*)malloc(sizeof(mpo_window) * maxw);
  int32_t* frame_off = (int32_t*)malloc(sizeof(int32_t) * (F + 1));
  mpo_size* sz = (mpo_size*)malloc(sizeof(mpo_size) * (k + 1));
  int64_t* cs = (int64_t*)malloc(sizeof(int64_t) * (k + 1));
  int32_t cc[17];
  int status = MPO_OK;
  for (int32_t q = 0; q < k; q++) { sz[q] = sizes[q]; cs[q] = cost[q]; }
  for (int32_t c = 0; c < n_cand; c++) {
    sz[k] = cand[c];
    cs[k] = cand_cost[c];
    int st = mpo_plan_windows(W, H, cw, ch, b_proxy, k + 1, sz, cs, scores, F, NULL, win, (int32_t)maxw,
                              frame_off, cc, NULL);
    if (st != MPO_OK) { status = st; break; }
    int64_t t = 0;
    for (int32_t i = 0; i < frame_off[F]; i++) t += cs[win[i].size_idx];
    tot[c] = t;
  }
  free(win); free(frame_off); free(sz); free(cs);
  return status;
}

/* ------------------------------------------------------------------------ */
/* NEXT-4a: Hungarian matching of detections to track prefixes — P:207 "We
 * apply the Hungarian algorithm to match detections with tracks based on
 * these scores ... If a detection d_j^(t) does not match with any track, we
 * initialize a new track prefix".  The paper gives no floor; reading
 * R24: maximise the total score over matchings
 * that use only pairs with score >= floor (floor > 0; NaN never allowed).
 * Written as the textbook square assignment: size S = max(m, n), cost
 * a[i][j] = -w[i][j] with w = score if allowed else 0 (and 0 on padding), so
 * a zero-weight pair in the optimum means "unmatched".  Solved with the
 * classic O(S^3) shortest-augmenting-path Hungarian method with row and
 * column potentials u, v (rows added one at a time; Dijkstra over columns
 * with slack minv[j], predecessor way[j]; arg-min ties -> a free column
 * first (it ends the search: every tie-break among minimum-slack columns
 * gives a shortest augmenting path), then the smallest column index).
 * All arithmetic fp64.  rows = track prefixes (m), columns = detections (n).
 * Outputs row_match[i] (column or -1), col_match[j] (row or -1), and *total
 * = sum of matched scores in row order (fp64). */
int32_t mpo_hungarian(const float* scores, int32_t m, int32_t n, float floor_, int32_t* row_match,
                      int32_t* col_match, double* total) {
  if (m < 0 || n < 0 || !(floor_ > 0.0f)) return MPO_ERR_INVALID;
  int32_t S = m > n ? m : n;
  for (int32_t i = 0; i < m; i++) row_match[i] = -1;
  for (int32_t j = 0; j < n; j++) col_match[j] = -1;
  *total = 0.0;
  if (S == 0) return MPO_OK;
  /* 1-indexed arrays as in the textbook formulation; index 0 is the virtual column */
  double* a = (double*)malloc(sizeof(double) * (size_t)(S + 1) * (S + 1));
  double* u = (double*)calloc(S + 1, sizeof(double));
  double* v = (double*)calloc(S + 1, sizeof(double));
  double* minv = (double*)malloc(sizeof(double) * (S + 1));
  int32_t* p = (int32_t*)calloc(S + 1, sizeof(int32_t));
  int32_t* way = (int32_t*)calloc(S + 1, sizeof(int32_t));
  char* used = (char*)malloc(S + 1);
  const double INF = 1e300;
  for (int32_t i = 1; i <= S; i++)
    for (int32_t j = 1; j <= S; j++) {
      double w = 0.0;
      if (i <= m && j <= n) {
        float s = scores[(int64_t)(i - 1) * n + (j - 1)];
        if (s >= floor_) w = (double)s; /* NaN compares false */
      }
      a[(int64_t)i * (S + 1) + j] = -w;
    }
  for (int32_t i = 1; i <= S; i++) {
    p[0] = i;
    int32_t j0 = 0;
    for (int32_t j = 0; j <= S; j++) {
      minv[j] = INF;
      used[j] = 0;
    }
    do {
      used[j0] = 1;
      int32_t i0 = p[j0], j1 = 0;
      double delta = INF;
      for (int32_t j = 1; j <= S; j++) {
        if (used[j]) continue;
        double cur = a[(int64_t)i0 * (S + 1) + j] - u[i0] - v[j];
        if (cur < minv[j]) {
          minv[j] = cur;
          way[j] = j0;
        }
        if (minv[j] < delta || (minv[j] == delta && p[j] == 0 && j1 != 0 && p[j1] != 0)) {
          delta = minv[j];
          j1 = j;
        }
      }
      for (int32_t j = 0; j <= S; j++) {
        if (used[j]) {
          u[p[j]] += delta;
          v[j] -= delta;
        } else {
          minv[j] -= delta;
        }
      }
      j0 = j1;
    } while (p[j0] != 0);
    do {
      int32_t j1 = way[j0];
      p[j0] = p[j1];
      j0 = j1;
    } while (j0);
  }
  /* p[j] = row assigned to column j; keep the pairs with positive weight */
  int32_t* rm = (int32_t*)malloc(sizeof(int32_t) * (S + 1));
  for (int32_t j = 1; j <= S; j++) rm[p[j]] = j;
  for (int32_t i = 1; i <= m; i++) {
    int32_t j = rm[i];
    if (j <= n && -a[(int64_t)i * (S + 1) + j] > 0.0) {
      row_match[i - 1] = j - 1;
      col_match[j - 1] = i - 1;
      *total += -a[(int64_t)i * (S + 1) + j];
    }
  }
  free(rm); free(a); free(u); free(v); free(minv); free(p); free(way); free(used);
  return MPO_OK;
}

/* ------------------------------------------------------------------------ */
/* NEXT-4b: track refinement (§3.4 "Refinement").
 * Reading R25: a track's path is the sequence of its
 * detections' box centres ((x1+x2)/2, (y1+y2)/2) in frame order (fp64);
 * "N points evenly spaced along each track" = points at arc lengths
 * L*i/(N-1), i = 0..N-1, along the polyline (L = total length), linearly
 * interpolated inside the segment reached; point 0 and point N-1 are the
 * first and last centres exactly; a track of one detection, or of length 0,
 * resamples to N copies of its first centre.  N = 20 in the paper. */
void mpo_track_resample(const double* pts, int32_t n, int32_t N, double* out) {
  if (n <= 0) return;
  double L = 0.0;
  for (int32_t k = 0; k + 1 < n; k++) {
    double dx = pts[2 * (k + 1)] - pts[2 * k], dy = pts[2 * (k + 1) + 1] - pts[2 * k + 1];
    L = L + sqrt(dx * dx + dy * dy);
  }
  for (int32_t i = 0; i < N; i++) {
    double x, y;
    if (n == 1 || L == 0.0 || i == 0) {
      x = pts[0];
      y = pts[1];
    } else if (i == N - 1) {
      x = pts[2 * (n - 1)];
      y = pts[2 * (n - 1) + 1];
    } else {
      double t = (L * (double)i) / (double)(N - 1);
      /* walk the segments: s = arc length at the start of segment k */
      double s = 0.0;
      int32_t k = 0;
      double seg = 0.0;
      for (k = 0; k + 1 < n; k++) {
        double dx = pts[2 * (k + 1)] - pts[2 * k], dy = pts[2 * (k + 1) + 1] - pts[2 * k + 1];
        seg = sqrt(dx * dx + dy * dy);
        if (s + seg >= t || k + 2 == n) break;
        s = s + seg;
      }
      double lam = seg > 0.0 ? (t - s) / seg : 0.0;
      if (lam > 1.0) lam = 1.0;
      if (lam < 0.0) lam = 0.0;
      x = pts[2 * k] + lam * (pts[2 * (k + 1)] - pts[2 * k]);
      y = pts[2 * k + 1] + lam * (pts[2 * (k + 1) + 1] - pts[2 * k + 1]);
    }
    out[2 * i] = x;
    out[2 * i + 1] = y;
  }
}

/* P:244 d(s1, s2) = (1/N) sum_i eucl(P(s1)[i], P(s2)[i]); summed in i order. */
double mpo_track_distance(const double* a, const double* b, int32_t N) {
  double s = 0.0;
  for (int32_t i = 0; i < N; i++) {
    double dx = a[2 * i] - b[2 * i], dy = a[2 * i + 1] - b[2 * i + 1];
    s = s + sqrt(dx * dx + dy * dy);
  }
  return s / (double)N;
}

/* P:243 "we begin by clustering the tracks in S* using DBSCAN".  Reading R26:
 * textbook DBSCAN over the T resampled paths [T][N][2] with distance d:
 * neighbourhood N(i) = {j : d(i,j) <= eps} (i included), core iff |N(i)| >=
 * min_pts; points visited in index order, each unvisited core point starts a
 * new cluster expanded breadth-first through core points (so clusters are
 * numbered by their smallest core index and a border point takes the first
 * cluster that reaches it); points never reached are noise and become
 * singleton clusters numbered after the DBSCAN clusters in index
 * order.  labels[i] = cluster id; is_core[i] = 0/1.  Returns the cluster
 * count (DBSCAN clusters + singletons); *n_dbscan = DBSCAN clusters only. */
int32_t mpo_dbscan(const double* paths, int32_t T, int32_t N, double eps, int32_t min_pts, int32_t* labels,
                   uint8_t* is_core, int32_t* n_dbscan) {
  uint8_t* adj = (uint8_t*)malloc((size_t)T * T + 1);
  int32_t* queue = (int32_t*)malloc(sizeof(int32_t) * (T + 1));
  for (int32_t i = 0; i < T; i++) {
    int32_t cnt = 0;
    for (int32_t j = 0; j < T; j++) {
      double d = mpo_track_distance(paths + (size_t)i * N * 2, paths + (size_t)j * N * 2, N);
      adj[(size_t)i * T + j] = d <= eps;
      cnt += d <= eps;
    }
    is_core[i] = cnt >= min_pts;
    labels[i] = -1;
  }
  int32_t C = 0;
  for (int32_t i = 0; i < T; i++) {
    if (labels[i] >= 0 || !is_core[i]) continue;
    int32_t c = C++;
    int32_t head = 0, tail = 0;
    labels[i] = c;
    queue[tail++] = i;
    while (head < tail) {
      int32_t q = queue[head++];
      if (!is_core[q]) continue; /* border points do not expand */
      for (int32_t j = 0; j < T; j++) {
        if (adj[(size_t)q * T + j] && labels[j] < 0) {
          labels[j] = c;
          queue[tail++] = j;
        }
      }
    }
  }
  *n_dbscan = C;
  for (int32_t i = 0; i < T; i++)
    if (labels[i] < 0) labels[i] = C++;
  free(adj);
  free(queue);
  return C;
}

/* P:245 "the center of a cluster ... p_i is the average of points in
 * {P(s)[i] | s in C}": members summed in index order (fp64), divided by the
 * member count.  centers [C][N][2], counts [C]. */
void mpo_cluster_centers(const double* paths, int32_t T, int32_t N, const int32_t* labels, int32_t C,
                         double* centers, int32_t* counts) {
  for (int32_t c = 0; c < C; c++) counts[c] = 0;
  for (size_t e = 0; e < (size_t)C * N * 2; e++) centers[e] = 0.0;
  for (int32_t i = 0; i < T; i++) {
    int32_t c = labels[i];
    counts[c]++;
    for (int32_t e = 0; e < 2 * N; e++) centers[(size_t)c * N * 2 + e] += paths[(size_t)i * N * 2 + e];
  }
  for (int32_t c = 0; c < C; c++)
    for (int32_t e = 0; e < 2 * N; e++) centers[(size_t)c * N * 2 + e] /= (double)counts[c];
}

/* Does the segment p->q intersect the closed box [x0,x1] x [y0,y1]?  (Slab
 * test on the segment's parameter range [0,1], fp64.) */
static int seg_box(double px, double py, double qx, double qy, double x0, double y0, double x1, double y1) {
  double t0 = 0.0, t1 = 1.0;
  double d[2] = {qx - px, qy - py}, p[2] = {px, py}, lo[2] = {x0, y0}, hi[2] = {x1, y1};
  for (int a = 0; a < 2; a++) {
    if (d[a] == 0.0) {
      if (p[a] < lo[a] || p[a] > hi[a]) return 0;
    } else {
      double ta = (lo[a] - p[a]) / d[a], tb = (hi[a] - p[a]) / d[a];
      if (ta > tb) { double t = ta; ta = tb; tb = t; }
      if (ta > t0) t0 = ta;
      if (tb < t1) t1 = tb;
      if (t0 > t1) return 0;
    }
  }
  return 1;
}

/* P:246-247 refinement of one track.  Reading R27: a cluster is a candidate
 * iff its centre path (polyline of N points) intersects the 3x3-cell square
 * around the cell (cell = `cell` px, cell index floor(p / cell)) of the
 * track's first or of its last centre ("cluster centers that pass close to
 * d_1 and d_n"); candidates are ranked by d(track, centre)
 * (ties: smaller cluster id) and taken in order until their member counts
 * sum to >= k ("keep the k = 10 closest cluster centers, where a cluster of n
 * tracks counts n times"); the new start (end) point is, per coordinate, the
 * member-count-weighted median of the taken centres' first (last) points:
 * the value at position ceil(W/2) of the ascending list in which each value
 * is repeated by its weight (the lower middle for even W).
 * path = the track's resampled N points; first/last = its first and last
 * centres.  Writes out[4] = (start x, start y, end x, end y) and returns the
 * number of clusters taken (0 = no candidate: out = first, last unchanged). */
static int cmp_dbl(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

static double wmedian(const double* vals, const int32_t* w, int32_t n) {
  /* expand, sort, pick position ceil(W/2) (1-indexed) */
  int64_t W = 0;
  for (int32_t i = 0; i < n; i++) W += w[i];
  double* e = (double*)malloc(sizeof(double) * (size_t)(W > 0 ? W : 1));
  int64_t t = 0;
  for (int32_t i = 0; i < n; i++)
    for (int32_t r = 0; r < w[i]; r++) e[t++] = vals[i];
  qsort(e, (size_t)W, sizeof(double), cmp_dbl);
  double v = e[(W + 1) / 2 - 1];
  free(e);
  return v;
}

int32_t mpo_refine_track(const double* path, int32_t N, const double* first, const double* last,
                         const double* centers, const int32_t* counts, int32_t C, double cell, int32_t k,
                         double* out) {
  out[0] = first[0];
  out[1] = first[1];
  out[2] = last[0];
  out[3] = last[1];
  double* dist = (double*)malloc(sizeof(double) * (C > 0 ? C : 1));
  int32_t* cand = (int32_t*)malloc(sizeof(int32_t) * (C > 0 ? C : 1));
  int32_t nc = 0;
  for (int32_t c = 0; c < C; c++) {
    const double* ctr = centers + (size_t)c * N * 2;
    int hit = 0;
    for (int e = 0; e < 2 && !hit; e++) {
      const double* pt = e ? last : first;
      double cx = floor(pt[0] / cell), cy = floor(pt[1] / cell);
      double x0 = (cx - 1.0) * cell, y0 = (cy - 1.0) * cell, x1 = (cx + 2.0) * cell, y1 = (cy + 2.0) * cell;
      for (int32_t i = 0; i + 1 < N && !hit; i++)
        hit = seg_box(ctr[2 * i], ctr[2 * i + 1], ctr[2 * i + 2], ctr[2 * i + 3], x0, y0, x1, y1);
    }
    if (hit) {
      cand[nc] = c;
      dist[nc] = mpo_track_distance(path, ctr, N);
      nc++;
    }
  }
  /* rank by (distance, id): insertion sort (candidate lists are short) */
  for (int32_t a = 1; a < nc; a++) {
    int32_t cc = cand[a];
    double dd = dist[a];
    int32_t b = a - 1;
    while (b >= 0 && (dist[b] > dd || (dist[b] == dd && cand[b] > cc))) {
      cand[b + 1] = cand[b];
      dist[b + 1] = dist[b];
      b--;
    }
    cand[b + 1] = cc;
    dist[b + 1] = dd;
  }
  int32_t taken = 0, wsum = 0;
  while (taken < nc && wsum < k) wsum += counts[cand[taken++]];
  if (taken > 0) {
    double* v = (double*)malloc(sizeof(double) * taken);
    int32_t* w = (int32_t*)malloc(sizeof(int32_t) * taken);
    for (int32_t q = 0; q < 4; q++) {
      int32_t pt = q < 2 ? 0 : N - 1, ax = q & 1;
      for (int32_t t = 0; t < taken; t++) {
        v[t] = centers[(size_t)cand[t] * N * 2 + 2 * pt + ax];
        w[t] = counts[cand[t]];
      }
      out[q] = wmedian(v, w, taken);
    }
    free(v);
    free(w);
  }
  free(dist);
  free(cand);
  return taken;
}
