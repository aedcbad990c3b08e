"""paper_2103_14695_b200 — B200-native hot path of MultiScope (arXiv 2103.14695):
proxy-guided window detection around the detector.

The compute lives in libmp_b200.so (hand-written CUDA for sm_100a behind the
C-ABI of include/mp.h); this package is its thin Python binding plus a buffer
-owning pipeline wrapper.  Importing it without the built library raises —
there is no CPU fallback.
"""
from ._binding import (MP_BT601_FULL, MP_BT601_LIMITED, MP_BT709_FULL, MP_BT709_LIMITED,  # noqa: F401
                       MP_ERR_CAPACITY, MP_ERR_CUDA, MP_ERR_INVALID, MP_ERR_UNSUPPORTED, MP_OK,
                       MP_OUT_F32_NCHW, MP_OUT_U8_NHWC, LIB_PATH, MPError, PlanParams, launches_per_call,
                       mp_gather_resize, mp_gather_resize_nv12, mp_gather_set_sm_reserve, mp_gather_resize_strided, mp_gather_workspace_size,
                       mp_plan_windows, mp_plan_workspace_size,
                       mp_proxy_sweep, mp_proxy_sweep_workspace_size, mp_remap_nms, mp_remap_nms_workspace_size,
                       mp_window_set_cost, status_string,
                       ASSIGN_PROBLEM_DTYPE, assign_problems, mp_hungarian, mp_hungarian_workspace_size,
                       mp_track_resample, mp_dbscan, mp_dbscan_workspace_size, mp_cluster_centers,
                       mp_refine_workspace_size, mp_refine_tracks)
from .pipeline import PipelinedRunner, WindowPipeline  # noqa: F401
