// mp_abi.cu — the small non-compute entry points of the C-ABI (include/mp.h).
#include "mp_internal.cuh"

extern "C" const char* mp_status_string(mp_status st) {
  switch (st) {
    case MP_OK: return "MP_OK";
    case MP_ERR_INVALID: return "MP_ERR_INVALID: invalid parameters";
    case MP_ERR_CUDA: return "MP_ERR_CUDA: a CUDA launch or attribute call failed";
    case MP_ERR_CAPACITY: return "MP_ERR_CAPACITY: an output buffer was too small";
    case MP_ERR_UNSUPPORTED: return "MP_ERR_UNSUPPORTED: beyond this build's limits";
  }
  return "unknown mp_status";
}

// Kernel launches per call (for bench.py's gpu_launches count):
//   plan: memset (not a kernel) + plan_fast + plan_full + plan_scan + plan_scatter
//         (+ plan_huge when R*ceil(C/2) > 960, not counted here)
//   gather: gather_prep + gather_kernel
//   remap_nms: memset (not a kernel) + tiny + small + large + scan + scatter
//   proxy_sweep: memset (not a kernel) + proxy_sweep_kernel
//   window_set_cost: window_set_init + window_set_cost
//   hungarian: memset (not a kernel) + hung_warp_kernel + hung_mid_kernel (max_dim > 64)
//              + hung_block_kernel (max_dim > 160)
//   track_resample: 1;  dbscan: memset + adj + core + union + root + scan + label + scan + noise (8);
//   cluster_centers: 1;  refine_tracks: 3 memsets + index count + scan + fill + query (4)
extern "C" int32_t mp_launches_per_call(int32_t which) {
  switch (which) {
    case 0: return 4;
    case 1: return 2;
    case 2: return 5;
    case 3: return 1;
    case 4: return 2;
    case 5: return 3;
    case 6: return 1;
    case 7: return 8;
    case 8: return 1;
    case 9: return 4;
  }
  return 0;
}
