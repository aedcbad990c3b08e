// mp_internal.cuh — device helpers shared by the sm_100a kernels of
// libmp_b200.so (never by the oracle).  PTX wrappers for mbarriers and 1-D
// bulk (TMA-engine) copies, warp/block scans, and the host-side status enum.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <mutex>

#include "../../include/mp.h"

namespace mpk {

constexpr int kMaxClasses = 16;
// 128 threads capped at 64 registers (8 K): the plan's scan then fits beside a
// persistent f32 gather CTA and its co-running side CTAs and finishes before
// the gather does (256 threads waited for the gather to end: c2 f32 step
// 1.430 -> 1.414 ms, DESIGN 6f); dev A/B builds may override.
#ifndef MP_SCAN_THREADS
#define MP_SCAN_THREADS 128
#endif
#ifndef MP_SCAN_MINB
#define MP_SCAN_MINB 8
#endif
constexpr int kScanThreads = MP_SCAN_THREADS;   // single-CTA CSR scans of the plan / NMS
constexpr int kScanMinBlocks = MP_SCAN_MINB;    // (register cap via __launch_bounds__)

// ----------------------------------------------------------------- status
__device__ __forceinline__ void set_status(int32_t* d_status, int32_t code) {
  if (d_status) atomicCAS(d_status, 0, code);   // first error wins; never cleared
}

// ----------------------------------------------------------------- warp helpers
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}

__device__ __forceinline__ long long warp_sum_i64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int warp_incl_scan(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int w = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += w;
  }
  return v;
}

// Block-wide exclusive scan of a[0..n) in shared memory, in place; returns the
// total.  `tmp` = shared scratch of >= 33 ints.  All threads must call.
__device__ __forceinline__ int block_excl_scan_smem(int* a, int n, int* tmp) {
  const int nt = blockDim.x, tid = threadIdx.x;
  const int per = (n + nt - 1) / nt;
  const int lo = min(n, tid * per), hi = min(n, lo + per);
  int s = 0;
  for (int i = lo; i < hi; i++) s += a[i];
  const int lane = tid & 31, wid = tid >> 5, nw = (nt + 31) >> 5;
  int inc = warp_incl_scan(s);
  if (lane == 31) tmp[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int v = lane < nw ? tmp[lane] : 0;
    int vi = warp_incl_scan(v);
    if (lane < nw) tmp[lane] = vi - v;
    if (lane == nw - 1) tmp[32] = vi;
  }
  __syncthreads();
  int run = tmp[wid] + inc - s;
  for (int i = lo; i < hi; i++) {
    int v = a[i];
    a[i] = run;
    run += v;
  }
  int total = tmp[32];
  __syncthreads();
  return total;
}

// Block-wide exclusive scan over a strided global int sequence
// a[0], a[stride], ... (n items) in place; returns the total.  One CTA.
// Each thread owns a contiguous run of items and reads it in batches of
// kScanBatch independent loads (one memory latency per batch, not per item:
// the single-CTA scans sit on the pipeline's critical path between two
// gathers).
constexpr int kScanBatch = 8;
__device__ __forceinline__ int block_scan_global(int* a, int n, int stride, int* tmp) {
  const int nt = blockDim.x, tid = threadIdx.x;
  const int per = (n + nt - 1) / nt;
  const int lo = min(n, tid * per), hi = min(n, lo + per);
  int s = 0;
  for (int i0 = lo; i0 < hi; i0 += kScanBatch) {
    int v[kScanBatch];
#pragma unroll
    for (int j = 0; j < kScanBatch; j++) v[j] = i0 + j < hi ? a[(size_t)(i0 + j) * stride] : 0;
#pragma unroll
    for (int j = 0; j < kScanBatch; j++) s += v[j];
  }
  const int lane = tid & 31, wid = tid >> 5, nw = (nt + 31) >> 5;
  int inc = warp_incl_scan(s);
  if (lane == 31) tmp[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int v = lane < nw ? tmp[lane] : 0;
    int vi = warp_incl_scan(v);
    if (lane < nw) tmp[lane] = vi - v;
    if (lane == nw - 1) tmp[32] = vi;
  }
  __syncthreads();
  int run = tmp[wid] + inc - s;
  for (int i0 = lo; i0 < hi; i0 += kScanBatch) {
    int v[kScanBatch];
#pragma unroll
    for (int j = 0; j < kScanBatch; j++) v[j] = i0 + j < hi ? a[(size_t)(i0 + j) * stride] : 0;
#pragma unroll
    for (int j = 0; j < kScanBatch; j++)
      if (i0 + j < hi) {
        a[(size_t)(i0 + j) * stride] = run;
        run += v[j];
      }
  }
  int total = tmp[32];
  __syncthreads();
  return total;
}

// ----------------------------------------------------------------- mbarrier / bulk copy (sm_90+ PTX, sm_100a here)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// Same, but the waiting thread is suspended in hardware (up to ~1 ms per try)
// instead of spinning, so waiting consumer warps take no issue slots.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAITS_%=;\n}" ::"r"(addr),
      "r"(parity), "r"(0x100000u)
      : "memory");
}

// 1-D bulk copy global -> shared through the TMA engine (SASS UBLKCP);
// completion is signalled as tx bytes on `bar`.  src/dst 16-B aligned,
// bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// 3-D TMA tensor copy global -> shared (SASS UTMALDG), completion as tx bytes
// on `bar`.  c0 is the innermost coordinate (in tensor elements).
__device__ __forceinline__ void tma_load_3d(void* dst_smem, const void* tmap, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst_smem)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// sm_100 TMA row gather: four rows r0..r3 (arbitrary indices) of a 2-D tensor
// map whose box is {width, 1}, starting at column c0, land back to back in
// shared memory (4 x width elements); completion as tx bytes on `bar`.
__device__ __forceinline__ void tma_gather4(void* dst_smem, const void* tmap, int c0, int r0, int r1, int r2,
                                            int r3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst_smem)),
      "l"(tmap), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}

// ----------------------------------------------------------------- misc
__host__ __device__ __forceinline__ int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace mpk

#define MP_CUDA_TRY(expr)                                  \
  do {                                                     \
    cudaError_t e_ = (expr);                               \
    if (e_ != cudaSuccess) {                               \
      (void)cudaGetLastError();                            \
      return MP_ERR_CUDA;                                  \
    }                                                      \
  } while (0)

namespace mpk {
// Every kernel of the hot path asks for the maximum shared-memory carveout
// (228 KB shared, the rest L1).  The carveout of an SM is fixed while CTAs are
// resident on it and defaults to the smallest one that fits the first kernel
// there: a persistent gather CTA of ~122 KB would leave the SM at the 132-KB
// carveout, with no room for the plan / remap-NMS CTAs of the neighbouring
// batches, which then queue until the gather ends.  Set once per (kernel,
// device).
inline cudaError_t prefer_max_shared(const void* fn) {
  static std::mutex mu;
  static const void* seen_fn[128];
  static int seen_dev[128];
  static int n = 0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  for (int i = 0; i < n; i++)
    if (seen_fn[i] == fn && seen_dev[i] == dev) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
  if (e == cudaSuccess && n < 128) {
    seen_fn[n] = fn;
    seen_dev[n] = dev;
    n++;
  }
  return e;
}
}  // namespace mpk
