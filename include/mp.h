/*
 * mp.h — C-ABI of the B200-native MultiScope proxy-guided window path.
 *
 * The library (paper_2103_14695_b200/libmp_b200.so, sm_100a) exposes the three
 * per-frame data-parallel calls of MultiScope's segmentation-proxy inference
 * (Bastani & Madden, arXiv 2103.14695, §3.3 "Inference" /
 * "Grouping Cells during Execution", lines 176-186), plus the two steps this
 * build adds around the detector (crop/resize in, remap/NMS out; SURVEY.md
 * §8(a) a5-a7, readings R15-R20 in DESIGN.md §3).
 *
 * Conventions common to every call
 *  - Ownership: the caller allocates and owns every buffer (the Python binding
 *    uses torch tensors).  The library never allocates, frees or retains device
 *    memory between calls.  Scratch memory comes in as (d_ws, ws_bytes) sized
 *    by the matching *_workspace_size() query.
 *  - "d_" pointers are DEVICE pointers; every other pointer is a HOST pointer
 *    read synchronously before the call returns.
 *  - Asynchrony: all device work is enqueued on stream `s` (a cudaStream_t,
 *    passed as void* so this header needs no CUDA include; NULL = legacy
 *    default stream).  The call returns without synchronising.  Device inputs
 *    must stay alive until the stream passes the call.  No call allocates or
 *    synchronises, so every call is CUDA-graph capturable.
 *  - Errors: invalid host parameters return MP_ERR_INVALID (or
 *    MP_ERR_UNSUPPORTED for valid-but-unsupported sizes) before anything is
 *    launched.  A failed launch returns MP_ERR_CUDA.  Data-dependent overflow
 *    (more windows / boxes than the caller's capacity) cannot be known on the
 *    host: the kernels store MP_ERR_CAPACITY into the device word *d_status
 *    (never clearing it; the caller zeroes it), still write all counts and
 *    offsets so the caller can grow buffers and retry, and skip writes that
 *    would fall outside the buffers.
 *  - Determinism: outputs are a pure function of the inputs, independent of
 *    launch configuration, stream, or how frames are sharded across GPUs.
 *    The library is re-entrant and keeps no global data state; the only
 *    process-wide state is a cache of immutable driver facts (the tensor-map
 *    encoder entry point, per-device SM counts, per-kernel attribute /
 *    occupancy results, the max-shared carveout already set), filled on first
 *    use under a mutex, so steady-state calls issue only their launches.
 */
#ifndef MP_H_
#define MP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MP_OK = 0,
  MP_ERR_INVALID = 1,     /* bad host parameters (checked before any launch) */
  MP_ERR_CUDA = 2,        /* a CUDA launch / attribute call failed            */
  MP_ERR_CAPACITY = 3,    /* device-side: an output buffer was too small      */
  MP_ERR_UNSUPPORTED = 4  /* valid but beyond this build's limits             */
} mp_status;

/* A window size (w_i, h_i) in S, in frame pixels.  PAPER.md:182 "a fixed set
 * of window sizes ... S = {(w_1,h_1),...,(w_k,h_k)}". */
typedef struct { int32_t w, h; } mp_size;

/* One rectangle r_i = (r.x, r.y, r.w, r.h) of R_t, plus the
 * frame it belongs to, the index of its size in S, and `slot` = its index in
 * the batched detector input of that size class (rank among the windows of
 * that size in (frame, list) order).  28 bytes, frame pixels. */
typedef struct { int32_t frame, x, y, w, h, size_idx, slot; } mp_window;

/* A detection box, corner form, 24 bytes.  Detector output (input of
 * mp_remap_nms) is in the window's detector-input pixels [0,ow]x[0,oh];
 * output of mp_remap_nms is in frame pixels.  Reading R17. */
typedef struct { float x1, y1, x2, y2, score; int32_t cls; } mp_box;

typedef enum {
  MP_OUT_F32_NCHW = 0,  /* class k tensor: float [cap_k][3][oh_k][ow_k], 0..255 scale, RGB */
  MP_OUT_U8_NHWC = 1    /* class k tensor: uint8 [cap_k][oh_k][ow_k][3], round-half-up      */
} mp_out_format;

/* Planner parameters.  PAPER.md:178 (B_proxy), :182 (S, T_{w,h}), :193 (the
 * full frame (W,H) is always in S). */
typedef struct {
  int32_t W, H;            /* frame size, px, 1..16384                                   */
  int32_t cell_w, cell_h;  /* cell size in frame px (paper: 32x32);
                              grid = ceil(H/cell_h) rows x ceil(W/cell_w) cols; the last
                              row/col is clipped to the frame (reading R1)                 */
  float b_proxy;           /* a cell is positive iff score > b_proxy (strict, R2)         */
  int32_t k;               /* |S|, 1..16                                                  */
  const mp_size* sizes;    /* host [k]: distinct, 1<=w<=W, 1<=h<=H, MUST contain (W,H)    */
  const int64_t* cost;     /* host [k]: T_{w,h} > 0 and area_i < area_j => T_i < T_j
                              (R13; pairs of equal area are unconstrained)                */
} mp_plan_params;

/* Bytes of scratch mp_plan_windows needs for F frames (0 on invalid params). */
size_t mp_plan_workspace_size(const mp_plan_params* p, int32_t F);

/*
 * mp_plan_windows — steps a1-a4: threshold the per-cell proxy scores
 * (PAPER.md:178), form one cluster per 4-connected component of positive cells
 * ("We initialize a cluster C_i for each connected component"),
 * run the greedy agglomerative merge of PAPER.md:184 under the costs T
 * (R4-R9, R11-R13), and emit one window per final cluster, centred on the
 * cluster's bounding box and clamped into the frame (R10).
 *
 *  d_scores      device float [F][R][C] row-major, R = ceil(H/cell_h), C = ceil(W/cell_w).
 *  d_mask        device uint32 [F][R][ceil(C/32)] or NULL: bit (c%32) of word c/32
 *                of row r is cell (r,c)'s positive flag; padding bits are 0.
 *  d_windows     device mp_window [max_windows]: all windows of all frames,
 *                frame ascending, then final cluster-list order.
 *  d_frame_off   device int32 [F+1]: CSR, windows of frame f are
 *                [d_frame_off[f], d_frame_off[f+1]); d_frame_off[F] = total
 *                (the true total even on overflow).
 *  d_class_count device int32 [k]: number of windows of each size (true counts).
 *  d_status      device int32: set to MP_ERR_CAPACITY if total > max_windows.
 *  Execution: one CTA per frame; frames with <= 256 horizontal runs of
 *  positive cells are planned in shared memory by a 128-thread tier, others by
 *  a persistent 128-thread tier whose CTAs hold up to 960 runs in shared
 *  memory (~26 KB with int16 run / box coordinates: three fit beside a
 *  persistent f32 gather CTA on the same SM, two beside a u8 one);
 *  frames with more runs (up to R*ceil(C/2)) are planned by a third tier
 *  whose run/component arrays live in a per-CTA global scratch slot in d_ws
 *  (same arithmetic).
 *  Limits: R*C <= 65536 cells (4K at 32 px = 8160, 8K = 32400); larger
 *  grids (and grids whose bit rows alone exceed shared memory) return
 *  MP_ERR_UNSUPPORTED.  (W, H <= 16384 keep every cell row / column index
 *  within the planner's int16 run and box coordinates.)
 */
mp_status mp_plan_windows(const mp_plan_params* p, const float* d_scores, int32_t F,
                          uint32_t* d_mask, mp_window* d_windows, int32_t max_windows,
                          int32_t* d_frame_off, int32_t* d_class_count, int32_t* d_status,
                          void* d_ws, size_t ws_bytes, void* stream);

/* Bytes of scratch mp_gather_resize needs for k size classes with output
 * dims out_dims[k] and batch capacities out_cap[k] (0 on invalid params). */
size_t mp_gather_workspace_size(int32_t k, const mp_size* out_dims, const int32_t* out_cap);

/*
 * mp_gather_resize — step a5: gather every window's crop from its full
 * resolution frame and bilinearly resample it to its size class's detector
 * input dims, writing one batched tensor per size class (PAPER.md:152
 * "initializes the detector on the GPU to execute at each of those sizes";
 * resampling convention R15/R16: half-pixel centres, taps clamped to the crop,
 * exact integer tap positions, fp32 arithmetic).
 *
 *  d_frame_ptrs  device array [F] of device-accessible pointers; frame f is
 *                uint8 [H][pitch] with RGB24 pixels, 16-byte aligned.  A frame
 *                may live in HBM or in page-locked host memory (cudaHostAlloc /
 *                cudaHostRegister, mapped under UVA): the kernel then reads
 *                only the window footprints over PCIe (zero-copy; bit-identical
 *                results, no staging copy of the whole frame).
 *  pitch         bytes per frame row, multiple of 16, >= 3*W.
 *  d_windows     device mp_window[max_windows]; the windows gathered are the
 *                first n_win = min(d_frame_off[F], max_windows) (read on
 *                device).  d_frame_off[F] > max_windows (a plan that overflowed
 *                this buffer reports its true total) sets *d_status =
 *                MP_ERR_CAPACITY; the records in the buffer are still gathered
 *                and nothing past the buffer is read.
 *                Each window must lie inside the frame, have
 *                (w,h) == sizes[size_idx], and slots of a class must be
 *                0..count-1 (as mp_plan_windows produces; violations set
 *                *d_status = MP_ERR_INVALID and skip the window).
 *  sizes         host [k] window sizes; out_dims host [k] (ow_k, oh_k) >= 1.
 *  d_out         host [k] of device pointers to class tensors (see
 *                mp_out_format), 16-byte aligned, batch capacity out_cap[k].
 *  A class with more than out_cap[k] windows sets MP_ERR_CAPACITY and the
 *  extra slots are skipped.
 */
mp_status mp_gather_resize(const uint8_t* const* d_frame_ptrs, int32_t pitch, int32_t W,
                           int32_t H, int32_t F, const mp_window* d_windows,
                           const int32_t* d_frame_off, int32_t max_windows, int32_t k, const mp_size* sizes,
                           const mp_size* out_dims, void* const* d_out, const int32_t* out_cap,
                           mp_out_format fmt, int32_t* d_status, void* d_ws, size_t ws_bytes,
                           void* stream);

/*
 * mp_gather_resize_strided — mp_gather_resize for the common case where the F
 * frames live in one allocation at a constant stride (a decoded batch):
 * frame f = d_frames + f * frame_stride.  Same results bit for bit; the source
 * box of each tile is staged with ONE 3-D TMA tensor copy (per-class tensor
 * map encoded on the host each call) instead of one bulk copy per row.
 *
 *  d_frames      device-accessible (HBM, or mapped page-locked host memory:
 *                zero-copy, as in mp_gather_resize), 16-byte aligned.
 *  frame_stride  bytes, multiple of 16, >= H * pitch, < 2^40.
 *  Other arguments as mp_gather_resize.  The workspace is the same.
 */
mp_status mp_gather_resize_strided(const uint8_t* d_frames, int64_t frame_stride, int32_t pitch, int32_t W,
                                   int32_t H, int32_t F, const mp_window* d_windows,
                                   const int32_t* d_frame_off, int32_t max_windows, int32_t k, const mp_size* sizes,
                                   const mp_size* out_dims, void* const* d_out, const int32_t* out_cap,
                                   mp_out_format fmt, int32_t* d_status, void* d_ws, size_t ws_bytes,
                                   void* stream);

/* ---------------------------------------------------------------------------
 * NEXT-3: decode-native input.  The paper decodes with
 * ffmpeg "at the object detector resolution" and feeds the proxy
 * a low-resolution frame; a GPU decoder (NVDEC) emits NV12.
 * Reading R23 fixes the format and conversion.
 */
typedef enum {
  MP_BT709_LIMITED = 0,   /* Kr .2126, Kb .0722; Y 16..235, C 16..240 (default for HD) */
  MP_BT601_LIMITED = 1,   /* Kr .299,  Kb .114 */
  MP_BT709_FULL = 2,      /* Y, C 0..255 */
  MP_BT601_FULL = 3       /* JFIF */
} mp_color_matrix;

/*
 * mp_gather_resize_nv12 — step a5 fed directly from NV12 decoder output: for
 * every window, the R15 bilinear resample of its Y, U and V samples (chroma
 * sample (i,j) covers luma (2i..2i+1, 2j..2j+1)) to its class's detector-input
 * dims, converted to R'G'B' with `matrix` and clamped to [0,255] (R23), written
 * in the same per-class layouts as mp_gather_resize (F32 NCHW 0..255 or U8
 * NHWC).  One read of each window's luma and chroma footprint (two TMA tensor
 * copies per tile); the conversion is fused into the resample's epilogue.
 * Used both for the detector crops and for the full-frame proxy input (a
 * full-frame window whose class has the proxy resolution as out_dims).
 *
 *  d_frames      device-accessible (HBM, or mapped page-locked host memory:
 *                zero-copy), 16-byte aligned; frame f at d_frames + f*frame_stride:
 *                Y plane [H][pitch] then interleaved UV plane [H/2][pitch]
 *                (U at even, V at odd bytes).
 *  frame_stride  bytes, multiple of 16, >= (H + H/2) * pitch, < 2^40.
 *  pitch         bytes per row of both planes, multiple of 16, >= W.
 *  W, H          frame size in pixels, both even.
 *  matrix        mp_color_matrix; anything else -> MP_ERR_INVALID.
 *  Other arguments, workspace, status and launch count as mp_gather_resize.
 */
mp_status mp_gather_resize_nv12(const uint8_t* d_frames, int64_t frame_stride, int32_t pitch, int32_t W,
                                int32_t H, int32_t F, const mp_window* d_windows, const int32_t* d_frame_off,
                                int32_t max_windows, int32_t k, const mp_size* sizes, const mp_size* out_dims, void* const* d_out,
                                const int32_t* out_cap, mp_out_format fmt, mp_color_matrix matrix,
                                int32_t* d_status, void* d_ws, size_t ws_bytes, void* stream);

/* Bytes of scratch mp_remap_nms needs for F frames and max_boxes raw boxes. */
size_t mp_remap_nms_workspace_size(int32_t F, int32_t max_boxes);

/*
 * mp_remap_nms — steps a6-a7 (not in the paper; readings R17-R20): for every
 * raw detector box of every window, drop it unless score > score_thr, clip it
 * to the detector-input extent [0,ow]x[0,oh], drop it if degenerate, map it to
 * frame pixels with one fp64 rounding sequence X = fp32(x_l*w/ow + x); then
 * per frame run class-aware greedy NMS in (score desc, candidate index asc)
 * order, suppressing a later same-class box iff its fp32 IoU > iou_thr.
 *
 *  d_boxes        device mp_box[n_box]; n_box = d_win_box_off[n_win] <= max_boxes.
 *  d_win_box_off  device int32 [n_win+1]: boxes of window i are
 *                 [d_win_box_off[i], d_win_box_off[i+1]) (window order).
 *  d_windows, d_frame_off  as produced by mp_plan_windows; d_windows holds
 *                 max_windows records and frame f's windows are
 *                 [min(d_frame_off[f], max_windows), min(d_frame_off[f+1], max_windows))
 *                 (windows a plan could not store do not exist; nothing past the
 *                 buffer is read).  n_win = min(d_frame_off[F], max_windows).
 *  out_dims       host [k] detector-input dims per size class.
 *  d_out, d_out_src  device [max_out]: kept boxes (frame px) and the index of
 *                 the input box each came from; frame-major, keep order.
 *  d_out_frame_off device int32 [F+1]: CSR of kept boxes (true totals).
 *  max_boxes      capacity of d_boxes; frames whose boxes extend past it are
 *                 skipped with *d_status = MP_ERR_INVALID.
 *  No per-frame limit: frames with up to 1024 raw boxes are merged in shared
 *  memory (tiers of <= 64 / <= 512 / <= 1024 raw boxes, each CTA small enough
 *  to run beside a persistent gather on the same SM); frames with more take a
 *  global-memory path inside the same launch (same arithmetic and results,
 *  O(n^2) IoUs over L2 — slow for very large n).  The workspace grows with
 *  max_boxes (~80 bytes per raw box).
 */
mp_status mp_remap_nms(const mp_box* d_boxes, const int32_t* d_win_box_off,
                       const mp_window* d_windows, const int32_t* d_frame_off, int32_t max_windows, int32_t F,
                       int32_t k, const mp_size* out_dims, int32_t W, int32_t H,
                       float score_thr, float iou_thr, mp_box* d_out, int32_t* d_out_src,
                       int32_t max_out, int32_t* d_out_frame_off, int32_t* d_status,
                       int32_t max_boxes, void* d_ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * NEXT-1: proxy-module caching sweep (§3.5.2 "Proxy Model
 * Module").  "for each threshold B_j, we compute rectangular windows using the
 * cell grouping method ... on each frame.  ... our runtime estimate for this
 * resolution and threshold is T_proxy,i + sum_k T_{r_k.w, r_k.h} ... The recall
 * is the fraction of detections computed by theta_best that are covered by
 * rectangles in R_{i,j}."
 *
 * One call = one proxy resolution i (one score-grid geometry) and J thresholds.
 * Single pass: one CTA per frame reads the frame's score grid once and ranks
 * every cell against the thresholds sorted ascending (rank = number of
 * thresholds the score exceeds; score > B_j <=> rank > position of B_j), so
 * each threshold's mask comes from shared memory; a threshold whose mask
 * equals the next-lower one's reuses that plan.  For every threshold the
 * frames are planned exactly as mp_plan_windows does (a1-a4, same readings)
 * and the per-threshold totals are accumulated:
 *   cost_sum      sum over frames and windows of T (the detector part of the
 *                 runtime estimate; the caller adds T_proxy,i)
 *   windows       number of windows
 *   full_frames   frames whose plan is the single full-frame window
 *   dets_covered  detections lying entirely inside some window of their frame
 *                 (reading R21: "covered" = contained, the detector must see
 *                 the whole object in one window)
 *   dets_touched  detections overlapping some window with positive area
 *                 (SPEC.md:251's looser reading, reported alongside)
 * recall_j = dets_covered / n_det.
 *
 *  p             planner parameters; p->b_proxy is ignored.
 *  d_scores      device float [F][R][C].
 *  thresholds    host float [J], 1 <= J <= 64, any order, duplicates allowed, no NaN;
 *                d_out row j belongs to thresholds[j].
 *  d_dets        device float [n_det][4] (x1, y1, x2, y2) frame px, the theta_best
 *                detections, frame-major; d_det_off device int32 [F+1] CSR.
 *  d_out         device mp_sweep_result [J] (overwritten).
 */
typedef struct {
  int64_t cost_sum, windows, full_frames, dets_covered, dets_touched;
} mp_sweep_result;

size_t mp_proxy_sweep_workspace_size(const mp_plan_params* p, int32_t F);

mp_status mp_proxy_sweep(const mp_plan_params* p, const float* d_scores, int32_t F, const float* thresholds,
                         int32_t J, const float* d_dets, const int32_t* d_det_off, mp_sweep_result* d_out,
                         void* d_ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * NEXT-2: window-size set selection (§3.3 "Determining Fixed
 * Set of Window Sizes").  "on each iteration, we select the size (w,h) that
 * minimizes tot_time(S + {(w,h)})", tot_time(S) = sum_t im_time(S, I_t) and
 * im_time = est(R(I_t; S)) with "the proxy model perform[ing] perfectly"
 * (positive cells = cells of the theta_best detections).
 *
 * mp_window_set_cost evaluates, for every candidate c, tot[c] = sum over the F
 * frames of est(R(I_f; S + {cand[c]})) — one greedy step's objective for all
 * candidates in one launch (grid frames x candidate blocks); the caller takes
 * the arg-min (ties: smaller area, then smaller w — reading R22) and repeats
 * k-1 times (paper_2103_14695_b200.window_sets.select_window_sizes).
 *
 *  p           the current set S (must contain (W,H)), |S| <= 15; p->b_proxy
 *              thresholds d_scores (pass a perfect-proxy 0/1 grid and e.g. 0.5).
 *  d_cand      device mp_size [n_cand] candidate sizes; d_cand_cost device
 *              int64 [n_cand] their T.  Each S + {cand[c]} must be a valid set
 *              (R13/R14: inside the frame, distinct from S, T > 0, strictly
 *              monotone in area against S) — checked ON THE DEVICE: an invalid
 *              candidate gets tot[c] = INT64_MAX (never the arg-min) and
 *              *d_status = MP_ERR_INVALID.
 *  d_tot       device int64 [n_cand] (overwritten).
 *  Launches: window_set_init + window_set_cost; no host copy or
 *  synchronisation (graph-capturable).  Split the candidates across GPUs
 *  and take the arg-min of the per-GPU arg-mins (window_sets.py).
 */
mp_status mp_window_set_cost(const mp_plan_params* p, const float* d_scores, int32_t F, const mp_size* d_cand,
                             const int64_t* d_cand_cost, int32_t n_cand, int64_t* d_tot, int32_t* d_status,
                             void* stream);

/* ---------------------------------------------------------------------------
 * NEXT-4a: Hungarian matching of detections to track prefixes (PAPER.md:207
 * "We apply the Hungarian algorithm to match detections with tracks based on
 * these scores, and add each detection to the track that it matches with. If
 * a detection d_j^(t) does not match with any track, we initialize a new
 * track prefix").  The scores p_ij come from the tracker model
 * (outside this library).  Batched over independent problems (clips).
 *
 * Reading R24: per problem, maximise the total score over
 * matchings that use only pairs with score >= floor_ (NaN never matched), via
 * the square assignment of size S = max(m, n) on cost -w (w = score if
 * allowed else 0, zero padding) with the textbook shortest-augmenting-path
 * Hungarian method in fp64 (rows added in order; Dijkstra arg-min ties -> a
 * free (unassigned) column first, since it ends the search, then the smallest
 * column index — any tie rule yields a shortest augmenting path, so the total
 * is optimal either way; the oracle uses the same rule, so matchings are
 * identical, not just equally good).
 *
 *  d_scores    device float; problem b's [m][n] row-major matrix starts at
 *              d_scores + problems[b].score_off (rows = track prefixes,
 *              columns = detections).
 *  d_problems  device mp_assign_problem [B].
 *  floor_      > 0, else MP_ERR_INVALID.
 *  max_dim     host bound on max(m, n) over the batch, <= 1024 (sizes shared
 *              memory); a problem with max(m, n) > max_dim gets *d_status =
 *              MP_ERR_CAPACITY and all -1 outputs.
 *  d_row_match device int32: row i of problem b -> matched column or -1, at
 *              d_row_match[row_off + i]; d_col_match likewise per column.
 *  d_total     device double [B]: sum of matched scores (fp64, row order).
 *  Problems with m, n < 0 or negative offsets: *d_status = MP_ERR_INVALID.
 *  Launches: memset + warp-per-problem kernel (S <= 64), then for the larger
 *  ones (queued on the device) a warp-per-problem kernel with the scores in
 *  shared memory (S <= 160, if max_dim > 64) and a CTA-per-problem kernel
 *  (S <= 1024, if max_dim > 160).  Graph-capturable.
 */
typedef struct {
  int64_t score_off;
  int32_t m, n, row_off, col_off;
} mp_assign_problem;

size_t mp_hungarian_workspace_size(int32_t B);

mp_status mp_hungarian(const float* d_scores, const mp_assign_problem* d_problems, int32_t B, float floor_,
                       int32_t max_dim, int32_t* d_row_match, int32_t* d_col_match, double* d_total,
                       int32_t* d_status, void* d_ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * NEXT-4b: track refinement (§3.4 "Refinement").  Offline:
 * the training tracks S* are resampled, clustered with DBSCAN and their
 * cluster centres indexed; online: each (reduced-rate) track is extended to
 * the member-weighted median start and end of its k nearest cluster centres.
 * Readings R25-R27.  All arithmetic fp64 in the oracle's order
 * (results bit-identical to oracle/).  A track set is given as detection
 * boxes float [n_det][4] (x1, y1, x2, y2), frame order within a track, with a
 * CSR d_track_off int32 [T+1].
 */

/* mp_track_resample — R25: each track's box-centre path resampled to N points
 * evenly spaced in arc length ("we compute N points evenly spaced along each
 * track").  d_paths double [T][N][2]; d_ends double [T][4] (first and
 * last centre: x0, y0, x1, y1), may be NULL.  Tracks with no detection get
 * zeros.  2 <= N <= 64, else MP_ERR_INVALID.  One kernel. */
mp_status mp_track_resample(const float* d_boxes, const int32_t* d_track_off, int32_t T, int32_t N,
                            double* d_paths, double* d_ends, void* stream);

/* mp_dbscan — R26: DBSCAN of T resampled paths under d(s1,s2) = mean
 * point distance, neighbourhood d <= eps, core iff >= min_pts
 * neighbours (self included); clusters numbered by smallest core index,
 * border tracks join the lowest-numbered cluster with a core neighbour, noise
 * tracks become singleton clusters numbered after them (index order).
 *  d_labels  device int32 [T] cluster id per track.
 *  d_is_core device uint8 [T] (may be NULL).
 *  d_nclust  device int32 [2]: [0] = DBSCAN clusters, [1] = all clusters.
 *  eps > 0, min_pts >= 1, T <= 65536, else MP_ERR_INVALID.
 *  Launches: memset + adjacency (warp per track pair block, early exit once
 *  the partial distance sum clearly exceeds eps*N) + core/union/label kernels
 *  + two single-CTA scans (cluster and singleton numbering). */
size_t mp_dbscan_workspace_size(int32_t T);
mp_status mp_dbscan(const double* d_paths, int32_t T, int32_t N, double eps, int32_t min_pts, int32_t* d_labels,
                    uint8_t* d_is_core, int32_t* d_nclust, void* d_ws, size_t ws_bytes, void* stream);

/* mp_cluster_centers — P:245: the centre of cluster c is the pointwise mean of
 * its members' paths (members summed in index order, fp64).  C = d_nclust[1]
 * (device); clusters c >= C_max are not written (*d_status = MP_ERR_CAPACITY).
 * d_centers double [C_max][N][2]; d_counts int32 [C_max]. */
mp_status mp_cluster_centers(const double* d_paths, int32_t T, int32_t N, const int32_t* d_labels,
                             const int32_t* d_nclust, int32_t C_max, double* d_centers, int32_t* d_counts,
                             int32_t* d_status, void* stream);

/* mp_refine_tracks — P:246-247 / R27: for each query track q (its resampled
 * path d_paths[q] and end centres d_ends[q] from mp_track_resample): the
 * candidate clusters are those whose centre polyline intersects the 3x3-cell
 * square (cells of `cell` px) around the cell of the track's first or last
 * centre — found through a grid index over the centres (cell -> clusters,
 * built in the workspace on every call) and confirmed by an exact
 * segment/square test; candidates are ranked by (d(track, centre), id) and
 * taken until their member counts reach k; d_out[q] = (start x, start y,
 * end x, end y) = per-coordinate member-weighted medians of the taken
 * centres' first / last points (unchanged end centres if no candidate);
 * d_taken[q] = clusters taken.
 *  W, H: frame size (grid extent; centres outside are clamped into the grid).
 *  cell > 0, 1 <= k, max_cand: per-query candidate capacity (<= 1024;
 *  exceeding it sets *d_status = MP_ERR_CAPACITY and the query is left
 *  unchanged).  C = d_nclust[1] <= C_max <= 65536.
 *  Launches: memset + index count + scan + index fill + query (warp per query). */
size_t mp_refine_workspace_size(int32_t W, int32_t H, double cell, int32_t C_max, int32_t N);
mp_status mp_refine_tracks(const double* d_paths, const double* d_ends, int32_t Q, int32_t N,
                           const double* d_centers, const int32_t* d_counts, const int32_t* d_nclust,
                           int32_t C_max, int32_t W, int32_t H, double cell, int32_t k, int32_t max_cand,
                           double* d_out, int32_t* d_taken, int32_t* d_status, void* d_ws, size_t ws_bytes,
                           void* stream);

/* Launch setting of the persistent gather kernels (mp_gather_resize*): leave
 * `sms` SMs' worth of CTAs out of the grid (process-wide, read at every
 * subsequent gather launch from any host thread; default 0 = one wave of
 * resident CTAs on every SM).  A u8 gather CTA leaves room beside it for only
 * one or two latency-bound planner CTAs (mp_plan_windows of the next batch, run
 * on another stream), which then issue at a fraction of their solo rate, and
 * none for the plan's single-CTA scan or the smallest remap/NMS tier, which
 * then wait for the gather to end; SMs left free run them at full rate.  Worth
 * it when those side kernels, not the gather, bound a pipelined step (u8
 * output: 1 SM, 16 on 4K dense frames — DESIGN.md 6f); it costs the gather
 * the SMs it leaves (f32: no gain).
 *  0 <= sms <= 1024, else MP_ERR_INVALID (the setting is unchanged).  Launches
 *  nothing; the grid is clamped to at least one SM. */
mp_status mp_gather_set_sm_reserve(int32_t sms);

/* Human-readable name of a status code (static string, never NULL). */
const char* mp_status_string(mp_status st);

/* Number of device kernels the library launches per call (diagnostic, used
 * by bench.py to count launches): which = 0 plan, 1 gather, 2 remap_nms,
 * 3 proxy_sweep, 4 window_set_cost, 5 hungarian, 6 track_resample,
 * 7 dbscan, 8 cluster_centers, 9 refine_tracks.  The plan adds one launch
 * (plan_huge_kernel) for grids with R*ceil(C/2) > 960 possible runs. */
int32_t mp_launches_per_call(int32_t which);

#ifdef __cplusplus
}
#endif
#endif /* MP_H_ */
