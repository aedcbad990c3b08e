/* c_abi_demo.c — the C-ABI of libmp_b200.so (include/mp.h) used from plain C
 * with the CUDA runtime: plan windows for one tiny frame, gather + resize its
 * crop, remap + NMS three detector boxes, and check the results against
 * values derived by hand from the readings in DESIGN.md §3.
 *
 * Build (tests/test_c_abi_gpu.py does this):
 *   gcc -std=c99 -I include -I /usr/local/cuda/include examples/c_abi_demo.c \
 *       -L paper_2103_14695_b200 -lmp_b200 -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,<abs path to paper_2103_14695_b200> -o c_abi_demo
 */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "mp.h"

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return 1;                                                                \
    }                                                                          \
  } while (0)
#define MP(x)                                                                  \
  do {                                                                         \
    mp_status s_ = (x);                                                        \
    if (s_ != MP_OK) {                                                         \
      fprintf(stderr, "%s at %s:%d\n", mp_status_string(s_), __FILE__, __LINE__); \
      return 1;                                                                \
    }                                                                          \
  } while (0)
#define EXPECT(c)                                                              \
  do {                                                                         \
    if (!(c)) {                                                                \
      fprintf(stderr, "check failed: %s (line %d)\n", #c, __LINE__);           \
      return 2;                                                                \
    }                                                                          \
  } while (0)

int main(void) {
  /* ---- a1-a4: one 256x128 frame, 32-px cells (4 rows x 8 columns), one
   * positive cell (row 1, column 2) -> bbox x [64,96) y [32,64) -> the 64x64
   * size (R6), centred and clamped (R10): window (48, 16, 64, 64). */
  const int W = 256, H = 128, R = 4, C = 8, F = 1;
  mp_size sizes[2] = {{64, 64}, {256, 128}};
  int64_t cost[2] = {20, 64};
  mp_plan_params p = {W, H, 32, 32, 0.5f, 2, sizes, cost};
  float h_scores[R * C];
  for (int i = 0; i < R * C; i++) h_scores[i] = 0.1f;
  h_scores[1 * C + 2] = 0.9f;
  float* d_scores;
  mp_window* d_win;
  int32_t *d_fo, *d_cc, *d_st;
  void* d_ws;
  size_t ws = mp_plan_workspace_size(&p, F);
  EXPECT(ws > 0);
  CK(cudaMalloc((void**)&d_scores, sizeof(h_scores)));
  enum { MAXW = 16 };   /* window buffer capacity */
  CK(cudaMalloc((void**)&d_win, MAXW * sizeof(mp_window)));
  CK(cudaMalloc((void**)&d_fo, (F + 1) * sizeof(int32_t)));
  CK(cudaMalloc((void**)&d_cc, 2 * sizeof(int32_t)));
  CK(cudaMalloc((void**)&d_st, sizeof(int32_t)));
  CK(cudaMalloc(&d_ws, ws));
  CK(cudaMemcpy(d_scores, h_scores, sizeof(h_scores), cudaMemcpyHostToDevice));
  CK(cudaMemset(d_st, 0, sizeof(int32_t)));
  MP(mp_plan_windows(&p, d_scores, F, NULL, d_win, MAXW, d_fo, d_cc, d_st, d_ws, ws, NULL));
  mp_window h_win[16];
  int32_t h_fo[2], h_cc[2], h_st;
  CK(cudaMemcpy(h_fo, d_fo, sizeof(h_fo), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h_cc, d_cc, sizeof(h_cc), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&h_st, d_st, sizeof(h_st), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h_win, d_win, sizeof(mp_window), cudaMemcpyDeviceToHost));
  EXPECT(h_st == MP_OK && h_fo[0] == 0 && h_fo[1] == 1 && h_cc[0] == 1 && h_cc[1] == 0);
  EXPECT(h_win[0].frame == 0 && h_win[0].x == 48 && h_win[0].y == 16 && h_win[0].w == 64 &&
         h_win[0].h == 64 && h_win[0].size_idx == 0 && h_win[0].slot == 0);
  printf("window: frame %d x %d y %d w %d h %d size %d slot %d\n", h_win[0].frame, h_win[0].x, h_win[0].y,
         h_win[0].w, h_win[0].h, h_win[0].size_idx, h_win[0].slot);

  /* ---- a5: a constant RGB frame (every byte 100) -> every resampled value 100 */
  const int pitch = 3 * W;   /* 768, a multiple of 16 */
  mp_size out_dims[2] = {{32, 32}, {128, 64}};
  int32_t caps[2] = {1, 1};
  uint8_t* d_frame;
  float *d_out0, *d_out1;
  CK(cudaMalloc((void**)&d_frame, (size_t)H * pitch));
  CK(cudaMemset(d_frame, 100, (size_t)H * pitch));
  CK(cudaMalloc((void**)&d_out0, 3 * 32 * 32 * sizeof(float)));
  CK(cudaMalloc((void**)&d_out1, 3 * 128 * 64 * sizeof(float)));
  void* outs[2] = {d_out0, d_out1};
  size_t gws = mp_gather_workspace_size(2, out_dims, caps);
  void* d_gws;
  CK(cudaMalloc(&d_gws, gws));
  MP(mp_gather_resize_strided(d_frame, (int64_t)H * pitch, pitch, W, H, F, d_win, d_fo, MAXW, 2, sizes, out_dims,
                              outs, caps, MP_OUT_F32_NCHW, d_st, d_gws, gws, NULL));
  float h_out[3 * 32 * 32];
  CK(cudaMemcpy(h_out, d_out0, sizeof(h_out), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&h_st, d_st, sizeof(h_st), cudaMemcpyDeviceToHost));
  EXPECT(h_st == MP_OK);
  for (int i = 0; i < 3 * 32 * 32; i++) EXPECT(h_out[i] == 100.0f);
  printf("crop: 3x32x32 f32, all 100.0\n");

  /* ---- a6-a7: boxes in the window's 32x32 detector input; x -> x*64/32 + 48,
   * y -> y*64/32 + 16 (R18).  A (0.9, class 0) suppresses B (0.8, class 0,
   * IoU 0.89 > 0.5); C (0.7, class 1) is kept (class-aware, R19). */
  mp_box h_boxes[3] = {{4, 4, 20, 20, 0.9f, 0}, {5, 5, 21, 21, 0.8f, 0}, {4, 4, 20, 20, 0.7f, 1}};
  int32_t h_wbo[2] = {0, 3};
  mp_box *d_boxes, *d_keep;
  int32_t *d_wbo, *d_src, *d_kfo;
  CK(cudaMalloc((void**)&d_boxes, sizeof(h_boxes)));
  CK(cudaMalloc((void**)&d_keep, sizeof(h_boxes)));
  CK(cudaMalloc((void**)&d_wbo, sizeof(h_wbo)));
  CK(cudaMalloc((void**)&d_src, 3 * sizeof(int32_t)));
  CK(cudaMalloc((void**)&d_kfo, (F + 1) * sizeof(int32_t)));
  CK(cudaMemcpy(d_boxes, h_boxes, sizeof(h_boxes), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_wbo, h_wbo, sizeof(h_wbo), cudaMemcpyHostToDevice));
  size_t nws = mp_remap_nms_workspace_size(F, 3);
  void* d_nws;
  CK(cudaMalloc(&d_nws, nws));
  MP(mp_remap_nms(d_boxes, d_wbo, d_win, d_fo, MAXW, F, 2, out_dims, W, H, 0.25f, 0.5f, d_keep, d_src, 3, d_kfo, d_st, 3,
                  d_nws, nws, NULL));
  mp_box h_keep[3];
  int32_t h_src[3], h_kfo[2];
  CK(cudaMemcpy(h_keep, d_keep, sizeof(h_keep), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h_src, d_src, sizeof(h_src), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h_kfo, d_kfo, sizeof(h_kfo), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&h_st, d_st, sizeof(h_st), cudaMemcpyDeviceToHost));
  EXPECT(h_st == MP_OK && h_kfo[0] == 0 && h_kfo[1] == 2);
  EXPECT(h_src[0] == 0 && h_src[1] == 2);
  EXPECT(h_keep[0].x1 == 56.0f && h_keep[0].y1 == 24.0f && h_keep[0].x2 == 88.0f && h_keep[0].y2 == 56.0f);
  EXPECT(h_keep[1].cls == 1 && h_keep[1].score == 0.7f);
  printf("kept: %d boxes, first (%.1f %.1f %.1f %.1f)\n", h_kfo[1], h_keep[0].x1, h_keep[0].y1, h_keep[0].x2,
         h_keep[0].y2);
  printf("C-ABI demo OK\n");
  return 0;
}
