// mp_assign.cu — NEXT-4a: batched Hungarian matching of detections to track
// prefixes (reading R24 in DESIGN.md §3).
//
// Each problem b is a scores matrix [m][n] (rows = track prefixes, columns =
// detections).  R24: maximise the total score over matchings that use only
// pairs with score >= floor, solved as the square assignment of size
// S = max(m, n) on cost a = -w (w = score if allowed, else 0; zero padding)
// with the shortest-augmenting-path Hungarian method: rows are added one at a
// time; for each, a Dijkstra-like scan over the columns keeps the slack
// minv[j] = min over visited rows of a[i][j] - u[i] - v[j] and its predecessor
// way[j], moves to the arg-min column (ties -> a free column first, then the
// smallest j: a free minimum ends the search at once), shifts the
// potentials u, v by that minimum, and stops at a free column; the path is
// then flipped.  All arithmetic is fp64 in the same order as the oracle, so
// the matchings are identical (not merely equally good).
//
// Parallel form: a GROUP of G threads solves one problem; thread t owns the
// columns j = 1 + t + G*k (k < KMAX), holding minv[j], v[j] and used[j] in
// registers; u[], p[] (column -> row) and way[] live in shared memory.  Each
// Dijkstra step = one coalesced read of row i0 of the scores (the columns of
// a row are consecutive), a group arg-min of (delta, j), and the potential
// update.  Tier 1: G = 32 (one warp per problem) for S <= 64; tier 2: one warp
// per problem with 5 columns per lane and the scores staged in shared memory
// for S <= 160 (warp-synchronous steps at shared-memory latency); tier 3:
// G = 256 (one CTA per problem) for S <= 1024.  Tiers 2 and 3 are queued on
// the device by tier 1.
#include "mp_internal.cuh"

namespace mpk {

constexpr int kHungWarpMax = 64;     // tier 1: S <= 64 (2 columns per lane)
constexpr int kHungMidMax = 160;     // tier 2: S <= 160 (5 columns per lane, scores in smem: <= 100 KB)
constexpr int kHungBlockMax = 1024;  // tier 2: S <= 1024 (4 columns per thread)
constexpr int kHungBlock = 256;

struct HungArgs {
  const float* scores;
  const mp_assign_problem* probs;
  int B;
  float floor_;
  int max_dim;
  int* row_match;
  int* col_match;
  double* total;
  int* status;
  int* q_cnt;    // [0]: tier-2 queue length, [1]: tier-3 queue length
  int* q_list;   // tier 2 at [0, B), tier 3 at [B, 2B)
};

// weight of pair (i, j), 1-indexed, of a problem; 0 outside [1,m] x [1,n] or below the floor.
// SMEM: the matrix was staged in shared memory (plain loads) instead of global (__ldg).
template <bool SMEM = false>
__device__ __forceinline__ double hung_w(const float* sc, int m, int n, float floor_, int i, int j) {
  if (i > m || j > n) return 0.0;
  const float s = SMEM ? sc[(size_t)(i - 1) * n + (j - 1)] : __ldg(sc + (size_t)(i - 1) * n + (j - 1));
  return (s >= floor_) ? (double)s : 0.0;   // NaN compares false
}

template <int G>
struct Group;

template <>
struct Group<32> {   // one warp
  __device__ static void sync() { __syncwarp(); }
  // lexicographic arg-min of (d, j) over the group; every lane gets the result
  // (callers pass j = busy * 2^30 + column, so free columns win ties)
  __device__ static void argmin(double& d, int& j, double*, int*) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, d, o);
      const int oj = __shfl_xor_sync(0xffffffffu, j, o);
      if (od < d || (od == d && oj < j)) {
        d = od;
        j = oj;
      }
    }
  }
};

template <>
struct Group<kHungBlock> {   // one CTA
  __device__ static void sync() { __syncthreads(); }
  __device__ static void argmin(double& d, int& j, double* sd, int* sj) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    Group<32>::argmin(d, j, nullptr, nullptr);
    if (lane == 0) {
      sd[wid] = d;
      sj[wid] = j;
    }
    __syncthreads();
    d = sd[0];
    j = sj[0];
    for (int w = 1; w < kHungBlock / 32; w++) {   // same order in every thread -> same result
      const double od = sd[w];
      const int oj = sj[w];
      if (od < d || (od == d && oj < j)) {
        d = od;
        j = oj;
      }
    }
    __syncthreads();   // sd/sj reusable
  }
};

// Solve one problem with a group of G threads (tid = rank in the group).
// Shared: u[S+1] (double), p[S+1], way[S+1] (int), red_d/red_j scratch.
template <int G, int KMAX, bool SMEM = false>
__device__ void hung_solve(const HungArgs& A, const mp_assign_problem& pb, int tid, double* u, int* p, int* way,
                           double* red_d, int* red_j, const float* sc_smem = nullptr) {
  using Grp = Group<G>;
  const int m = pb.m, n = pb.n, S = max(m, n);
  const float* sc = SMEM ? sc_smem : A.scores + pb.score_off;
  const double INF = 1e300;
  for (int j = tid; j <= S; j += G) {
    u[j] = 0.0;
    p[j] = 0;
    way[j] = 0;
  }
  double v[KMAX], minv[KMAX];
  bool used[KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; k++) v[k] = 0.0;
  Grp::sync();
  for (int i = 1; i <= S; i++) {
    if (tid == 0) p[0] = i;
#pragma unroll
    for (int k = 0; k < KMAX; k++) {
      minv[k] = INF;
      used[k] = false;
    }
    int j0 = 0;
    Grp::sync();
    while (true) {
      // used[j0] = true (column 0 is virtual and always used)
#pragma unroll
      for (int k = 0; k < KMAX; k++)
        if (j0 == 1 + tid + G * k) used[k] = true;
      const int i0 = p[j0];
      const double ui0 = u[i0];
      double delta = INF;
      int key = 0x7fffffff;   // busy(j) << 30 | j of the best column: free columns first, then smallest j
#pragma unroll
      for (int k = 0; k < KMAX; k++) {
        const int j = 1 + tid + G * k;
        if (j <= S && !used[k]) {
          const double a = -hung_w<SMEM>(sc, m, n, A.floor_, i0, j);
          const double cur = __dsub_rn(__dsub_rn(a, ui0), v[k]);
          if (cur < minv[k]) {
            minv[k] = cur;
            way[j] = j0;
          }
          const int kj = (p[j] != 0 ? (1 << 30) : 0) | j;
          if (minv[k] < delta || (minv[k] == delta && kj < key)) {
            delta = minv[k];
            key = kj;
          }
        }
      }
      Grp::argmin(delta, key, red_d, red_j);
      const int j1 = key & ((1 << 30) - 1);
      Grp::sync();   // every read of u[i0] precedes the updates below
      // potentials: used columns (their rows) shift by +delta / -delta, the others' slack by -delta
#pragma unroll
      for (int k = 0; k < KMAX; k++) {
        const int j = 1 + tid + G * k;
        if (j <= S) {
          if (used[k]) {
            u[p[j]] = __dadd_rn(u[p[j]], delta);
            v[k] = __dsub_rn(v[k], delta);
          } else {
            minv[k] = __dsub_rn(minv[k], delta);
          }
        }
      }
      if (tid == 0) u[p[0]] = __dadd_rn(u[p[0]], delta);   // column 0
      Grp::sync();
      j0 = j1;
      if (p[j0] == 0) break;
    }
    Grp::sync();   // every thread has read p[j0] for the exit test before it changes
    // flip the augmenting path (sequential, short)
    if (tid == 0) {
      do {
        const int jj = way[j0];
        p[j0] = p[jj];
        j0 = jj;
      } while (j0);
    }
    Grp::sync();
  }
}

// Write one solved problem's outputs (p[] in shared memory; u[] reused as the
// per-row matched weight so the total is summed in row order like the oracle).
template <int G>
__device__ void hung_emit(const HungArgs& A, const mp_assign_problem& pb, int b, int tid, double* u, const int* p) {
  const int m = pb.m, n = pb.n, S = max(m, n);
  const float* sc = A.scores + pb.score_off;
  for (int i = tid; i < m; i += G) A.row_match[pb.row_off + i] = -1;
  for (int j = tid; j < n; j += G) A.col_match[pb.col_off + j] = -1;
  for (int i = tid; i <= S; i += G) u[i] = 0.0;
  Group<G>::sync();
  for (int j = 1 + tid; j <= S; j += G) {
    const int i = p[j];
    if (j <= n && i >= 1 && i <= m) {
      const double w = hung_w(sc, m, n, A.floor_, i, j);
      if (w > 0.0) {
        A.row_match[pb.row_off + i - 1] = j - 1;
        A.col_match[pb.col_off + j - 1] = i - 1;
        u[i] = w;
      }
    }
  }
  Group<G>::sync();
  if (tid == 0) {
    double t = 0.0;
    for (int i = 1; i <= m; i++) t = __dadd_rn(t, u[i]);
    A.total[b] = t;
  }
  Group<G>::sync();
}

__device__ void hung_fail(const HungArgs& A, const mp_assign_problem& pb, int b, int tid, int G, int code) {
  if (pb.m > 0 && pb.row_off >= 0)
    for (int i = tid; i < pb.m; i += G) A.row_match[pb.row_off + i] = -1;
  if (pb.n > 0 && pb.col_off >= 0)
    for (int j = tid; j < pb.n; j += G) A.col_match[pb.col_off + j] = -1;
  if (tid == 0) {
    A.total[b] = 0.0;
    set_status(A.status, code);
  }
}

constexpr int kHungWarpsPerCta = 8;

__global__ void __launch_bounds__(32 * kHungWarpsPerCta) hung_warp_kernel(const HungArgs A) {
  __shared__ double s_u[kHungWarpsPerCta][kHungWarpMax + 1];
  __shared__ int s_p[kHungWarpsPerCta][kHungWarpMax + 1];
  __shared__ int s_way[kHungWarpsPerCta][kHungWarpMax + 1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int gw = blockIdx.x * kHungWarpsPerCta + wid, nw = gridDim.x * kHungWarpsPerCta;
  for (int b = gw; b < A.B; b += nw) {
    const mp_assign_problem pb = A.probs[b];
    if (pb.m < 0 || pb.n < 0 || pb.score_off < 0 || pb.row_off < 0 || pb.col_off < 0) {
      hung_fail(A, pb, b, lane, 32, MP_ERR_INVALID);
      continue;
    }
    const int S = max(pb.m, pb.n);
    if (S > A.max_dim) {
      hung_fail(A, pb, b, lane, 32, MP_ERR_CAPACITY);
      continue;
    }
    if (pb.m == 0 || pb.n == 0) {   // nothing to match
      hung_fail(A, pb, b, lane, 32, MP_OK);
      continue;
    }
    if (S > kHungWarpMax) {   // tiers 2 / 3
      if (lane == 0) {
        if (S <= kHungMidMax) A.q_list[atomicAdd(&A.q_cnt[0], 1)] = b;
        else A.q_list[A.B + atomicAdd(&A.q_cnt[1], 1)] = b;
      }
      continue;
    }
    hung_solve<32, 2>(A, pb, lane, s_u[wid], s_p[wid], s_way[wid], nullptr, nullptr);
    hung_emit<32>(A, pb, b, lane, s_u[wid], s_p[wid]);
  }
}

// Tier 2: one warp per problem (one warp per CTA), the problem's [m][n]
// scores staged once in shared memory so every Dijkstra step reads its row at
// shared-memory latency instead of L2's; warp-synchronous steps (no CTA
// barriers).  S <= kHungMidMax (the m*n floats must fit the dynamic smem).
__global__ void __launch_bounds__(32) hung_mid_kernel(const HungArgs A) {
  extern __shared__ __align__(16) unsigned char hsm2[];
  double* u = reinterpret_cast<double*>(hsm2);
  int* p = reinterpret_cast<int*>(u + (kHungMidMax + 1));
  int* way = p + (kHungMidMax + 1);
  float* sc = reinterpret_cast<float*>(way + (kHungMidMax + 1));
  const int lane = threadIdx.x;
  const int nq = A.q_cnt[0];
  for (int qi = blockIdx.x; qi < nq; qi += gridDim.x) {
    const int b = A.q_list[qi];
    const mp_assign_problem pb = A.probs[b];
    const float* g = A.scores + pb.score_off;
    const int mn = pb.m * pb.n;
    for (int e = lane; e < mn; e += 32) sc[e] = __ldg(g + e);
    __syncwarp();
    hung_solve<32, kHungMidMax / 32, true>(A, pb, lane, u, p, way, nullptr, nullptr, sc);
    hung_emit<32>(A, pb, b, lane, u, p);
  }
}

__global__ void __launch_bounds__(kHungBlock) hung_block_kernel(const HungArgs A) {
  extern __shared__ __align__(16) unsigned char hsm[];
  double* u = reinterpret_cast<double*>(hsm);
  int* p = reinterpret_cast<int*>(u + (A.max_dim + 1));
  int* way = p + (A.max_dim + 1);
  __shared__ double red_d[kHungBlock / 32];
  __shared__ int red_j[kHungBlock / 32];
  const int nq = A.q_cnt[1];
  for (int qi = blockIdx.x; qi < nq; qi += gridDim.x) {
    const int b = A.q_list[A.B + qi];
    const mp_assign_problem pb = A.probs[b];
    hung_solve<kHungBlock, kHungBlockMax / kHungBlock>(A, pb, threadIdx.x, u, p, way, red_d, red_j);
    hung_emit<kHungBlock>(A, pb, b, threadIdx.x, u, p);
  }
}

}  // namespace mpk

using namespace mpk;

extern "C" size_t mp_hungarian_workspace_size(int32_t B) {
  if (B < 0) return 0;
  return 256 + (((size_t)2 * B * sizeof(int) + 255) & ~size_t(255));
}

extern "C" mp_status mp_hungarian(const float* d_scores, const mp_assign_problem* d_problems, int32_t B,
                                  float floor_, int32_t max_dim, int32_t* d_row_match, int32_t* d_col_match,
                                  double* d_total, int32_t* d_status, void* d_ws, size_t ws_bytes, void* stream) {
  if (B < 0 || !(floor_ > 0.0f) || max_dim < 0 || max_dim > kHungBlockMax || !d_status) return MP_ERR_INVALID;
  if (B == 0) return MP_OK;
  if (!d_problems || !d_total || !d_row_match || !d_col_match || !d_scores) return MP_ERR_INVALID;
  if (!d_ws || ws_bytes < mp_hungarian_workspace_size(B)) return MP_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  HungArgs A;
  A.scores = d_scores;
  A.probs = d_problems;
  A.B = B;
  A.floor_ = floor_;
  A.max_dim = max_dim;
  A.row_match = d_row_match;
  A.col_match = d_col_match;
  A.total = d_total;
  A.status = d_status;
  A.q_cnt = (int*)d_ws;
  A.q_list = (int*)((unsigned char*)d_ws + 256);
  MP_CUDA_TRY(cudaMemsetAsync(A.q_cnt, 0, 2 * sizeof(int), s));
  int dev = 0, sms = 0;
  MP_CUDA_TRY(cudaGetDevice(&dev));
  MP_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int grid1 = max(1, min((B + kHungWarpsPerCta - 1) / kHungWarpsPerCta, sms * 16));
  hung_warp_kernel<<<grid1, 32 * kHungWarpsPerCta, 0, s>>>(A);
  MP_CUDA_TRY(cudaGetLastError());
  if (max_dim > kHungWarpMax) {
    const int md = min(max_dim, kHungMidMax);
    const size_t smem2 = (size_t)(kHungMidMax + 1) * (sizeof(double) + 2 * sizeof(int)) + (size_t)md * md * sizeof(float);
    MP_CUDA_TRY(cudaFuncSetAttribute(hung_mid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
    hung_mid_kernel<<<sms * 2, 32, smem2, s>>>(A);
    MP_CUDA_TRY(cudaGetLastError());
  }
  if (max_dim > kHungMidMax) {
    const size_t smem = (size_t)(max_dim + 1) * (sizeof(double) + 2 * sizeof(int));
    MP_CUDA_TRY(cudaFuncSetAttribute(hung_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    hung_block_kernel<<<sms * 4, kHungBlock, smem, s>>>(A);
    MP_CUDA_TRY(cudaGetLastError());
  }
  return MP_OK;
}
