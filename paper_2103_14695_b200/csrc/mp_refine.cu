// mp_refine.cu — NEXT-4b: track refinement (§3.4
// "Refinement"; readings R25-R27 in DESIGN.md §3).
//
//   mp_track_resample   thread per track: box centres, arc length, N points
//   mp_dbscan           adjacency bitmask (CTA tile 8 x 32 track pairs, paths
//                       staged in shared memory, early exit once the partial
//                       distance sum clearly exceeds eps*N), core flags,
//                       union-find over core-core edges (linking the larger
//                       root under the smaller, so a root is its component's
//                       smallest core index), cluster numbering by a scan in
//                       index order, border / noise labels
//   mp_cluster_centers  thread per cluster, members summed in index order
//   mp_refine_tracks    grid index over the centres (count / scan / fill),
//                       then one warp per query track: candidate gather from
//                       the index, exact segment/square test, distances,
//                       (distance, id) ranking, k-weighted medians
//
// Every floating-point step is fp64 with explicit rounding (__dadd_rn, ...)
// in the oracle's order, so results are bit-identical to oracle/.
#include <math.h>

#include "mp_internal.cuh"

namespace mpk {

// ------------------------------------------------------------------ resample
__global__ void track_resample_kernel(const float* __restrict__ boxes, const int* __restrict__ off, int T, int N,
                                      double* __restrict__ paths, double* __restrict__ ends) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int a = off[t], n = off[t + 1] - a;
  double* out = paths + (size_t)t * N * 2;
  auto cx = [&](int k) { return __dmul_rn(__dadd_rn((double)boxes[4 * (a + k)], (double)boxes[4 * (a + k) + 2]), 0.5); };
  auto cy = [&](int k) { return __dmul_rn(__dadd_rn((double)boxes[4 * (a + k) + 1], (double)boxes[4 * (a + k) + 3]), 0.5); };
  if (n <= 0) {
    for (int i = 0; i < 2 * N; i++) out[i] = 0.0;
    if (ends)
      for (int i = 0; i < 4; i++) ends[4 * t + i] = 0.0;
    return;
  }
  auto seglen = [&](int k) {
    const double dx = __dsub_rn(cx(k + 1), cx(k)), dy = __dsub_rn(cy(k + 1), cy(k));
    return __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
  };
  double L = 0.0;
  for (int k = 0; k + 1 < n; k++) L = __dadd_rn(L, seglen(k));
  const double x0 = cx(0), y0 = cy(0), xl = cx(n - 1), yl = cy(n - 1);
  if (ends) {
    ends[4 * t] = x0;
    ends[4 * t + 1] = y0;
    ends[4 * t + 2] = xl;
    ends[4 * t + 3] = yl;
  }
  // monotone walk: point i's segment is the first k with s_k + seg_k >= t_i
  // (or the last); t_i is non-decreasing, so the search resumes where the
  // previous point stopped (the same prefix sums as the oracle's restart)
  int k = 0;
  double s = 0.0, seg = (n > 1) ? seglen(0) : 0.0;
  for (int i = 0; i < N; i++) {
    double x, y;
    if (n == 1 || L == 0.0 || i == 0) {
      x = x0;
      y = y0;
    } else if (i == N - 1) {
      x = xl;
      y = yl;
    } else {
      const double tt = __ddiv_rn(__dmul_rn(L, (double)i), (double)(N - 1));
      while (!(__dadd_rn(s, seg) >= tt || k + 2 == n)) {
        s = __dadd_rn(s, seg);
        k++;
        seg = seglen(k);
      }
      double lam = seg > 0.0 ? __ddiv_rn(__dsub_rn(tt, s), seg) : 0.0;
      if (lam > 1.0) lam = 1.0;
      if (lam < 0.0) lam = 0.0;
      x = __dadd_rn(cx(k), __dmul_rn(lam, __dsub_rn(cx(k + 1), cx(k))));
      y = __dadd_rn(cy(k), __dmul_rn(lam, __dsub_rn(cy(k + 1), cy(k))));
    }
    out[2 * i] = x;
    out[2 * i + 1] = y;
  }
}

// P:244 mean point distance, summed in point order (a, b: [N][2])
__device__ __forceinline__ double path_dist(const double* a, const double* b, int N) {
  double s = 0.0;
  for (int i = 0; i < N; i++) {
    const double dx = __dsub_rn(a[2 * i], b[2 * i]), dy = __dsub_rn(a[2 * i + 1], b[2 * i + 1]);
    s = __dadd_rn(s, __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy))));
  }
  return __ddiv_rn(s, (double)N);
}

// ------------------------------------------------------------------ DBSCAN
constexpr int kAdjRows = 8;   // CTA tile: 8 rows (warps) x 32 columns (lanes)
constexpr int kMaxN = 64;

__global__ void __launch_bounds__(32 * kAdjRows) dbscan_adj_kernel(const double* __restrict__ paths, int T, int N,
                                                                 double eps, double prune, int words,
                                                                 uint32_t* __restrict__ adj) {
  extern __shared__ double sp[];   // [kAdjRows + 32][N][2]
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int i0 = blockIdx.y * kAdjRows, j0 = blockIdx.x * 32;
  const int per = 2 * N;
  for (int e = threadIdx.x; e < (kAdjRows + 32) * per; e += blockDim.x) {
    const int r = e / per, c = e - r * per;
    const int tr = r < kAdjRows ? i0 + r : j0 + (r - kAdjRows);
    sp[e] = tr < T ? paths[(size_t)tr * per + c] : 0.0;
  }
  __syncthreads();
  const int i = i0 + wid, j = j0 + lane;
  bool nb = false;
  if (i < T && j < T) {
    const double* a = sp + wid * per;
    const double* b = sp + (kAdjRows + lane) * per;
    double s = 0.0;
    int p = 0;
    for (; p < N; p++) {
      const double dx = __dsub_rn(a[2 * p], b[2 * p]), dy = __dsub_rn(a[2 * p + 1], b[2 * p + 1]);
      s = __dadd_rn(s, __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy))));
      if (s > prune) break;   // the full sum / N is certainly > eps (prune = eps*N*(1 + 2^-40))
    }
    nb = p == N && __ddiv_rn(s, (double)N) <= eps;
  }
  const uint32_t bits = __ballot_sync(0xffffffffu, nb);
  if (lane == 0 && i < T && j0 < T) adj[(size_t)i * words + (j0 >> 5)] = bits;
}

__global__ void dbscan_core_kernel(const uint32_t* __restrict__ adj, int T, int words, int min_pts,
                                   uint8_t* __restrict__ core, uint32_t* __restrict__ coremask,
                                   int* __restrict__ parent) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= T) return;
  int c = 0;
  for (int w = 0; w < words; w++) c += __popc(adj[(size_t)i * words + w]);
  const bool k = c >= min_pts;
  core[i] = k;
  parent[i] = i;
  if (k) atomicOr(&coremask[i >> 5], 1u << (i & 31));
}

__device__ int guf_find(int* parent, int x) {
  while (true) {
    const int p = parent[x];
    if (p == x) return x;
    const int g = parent[p];
    if (g != p) atomicCAS(&parent[x], p, g);   // path halving
    x = p;
  }
}

// link the larger root under the smaller: a root is the smallest index of its set
__device__ void guf_unite(int* parent, int a, int b) {
  while (true) {
    a = guf_find(parent, a);
    b = guf_find(parent, b);
    if (a == b) return;
    if (a > b) {
      const int t = a;
      a = b;
      b = t;
    }
    if (atomicCAS(&parent[b], b, a) == b) return;
  }
}

__global__ void dbscan_union_kernel(const uint32_t* __restrict__ adj, int T, int words,
                                    const uint32_t* __restrict__ coremask, int* __restrict__ parent) {
  const int lane = threadIdx.x & 31;
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= T || !((coremask[i >> 5] >> (i & 31)) & 1u)) return;
  for (int w = lane; w < words; w += 32) {
    uint32_t bits = adj[(size_t)i * words + w] & coremask[w];
    while (bits) {
      const int j = (w << 5) + __ffs(bits) - 1;
      bits &= bits - 1;
      if (j > i) guf_unite(parent, i, j);
    }
  }
}

// roots are final once the unions are done: point every core track straight
// at its root (keeps the forest valid for concurrent finds) and flag roots
__global__ void dbscan_root_kernel(int T, const uint8_t* __restrict__ core, int* __restrict__ parent,
                                   int* __restrict__ flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= T) return;
  int r = i;
  if (core[i]) {
    r = guf_find(parent, i);
    parent[i] = r;
  }
  flag[i] = (core[i] && r == i) ? 1 : 0;
}

__global__ void scan_kernel(int* a, int n, int* total) {
  __shared__ int tmp[33];
  const int t = block_scan_global(a, n, 1, tmp);
  if (threadIdx.x == 0) *total = t;
}

// labels: core -> id of its root; border -> smallest id over core neighbours; noise -> -1 (flag2 = 1)
// parent[] of core tracks = their root (dbscan_root_kernel); cid[root] = cluster id
__global__ void dbscan_label_kernel(const uint32_t* __restrict__ adj, int T, int words,
                                    const uint8_t* __restrict__ core, const uint32_t* __restrict__ coremask,
                                    const int* __restrict__ parent, const int* __restrict__ cid,
                                    int* __restrict__ labels, int* __restrict__ flag2, uint8_t* __restrict__ is_core) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= T) return;
  int lab;
  if (core[i]) {
    lab = cid[parent[i]];
  } else {
    lab = 0x7fffffff;
    for (int w = 0; w < words; w++) {
      uint32_t bits = adj[(size_t)i * words + w] & coremask[w];
      while (bits) {
        const int j = (w << 5) + __ffs(bits) - 1;
        bits &= bits - 1;
        lab = min(lab, cid[parent[j]]);
      }
    }
    if (lab == 0x7fffffff) lab = -1;
  }
  labels[i] = lab;
  flag2[i] = lab < 0 ? 1 : 0;
  if (is_core) is_core[i] = core[i];
}

__global__ void dbscan_noise_kernel(int T, const int* __restrict__ rank, const int* __restrict__ nclust,
                                    int* __restrict__ labels, int* __restrict__ out_nclust) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < T && labels[i] < 0) labels[i] = nclust[0] + rank[i];
  if (i == 0) {
    out_nclust[0] = nclust[0];
    out_nclust[1] = nclust[0] + nclust[1];
  }
}

// ------------------------------------------------------------------ centres
// One CTA per cluster: the members are found in index order chunk by chunk
// (block scan of label == c over 1024 tracks), then threads t < 2N add their
// coordinate of each member in that order (the oracle's summation order).
constexpr int kCtrThreads = 256, kCtrChunk = 1024;

__global__ void __launch_bounds__(kCtrThreads) cluster_centers_kernel(const double* __restrict__ paths, int T, int N,
                                                                     const int* __restrict__ labels,
                                                                     const int* __restrict__ nclust, int C_max,
                                                                     double* __restrict__ centers,
                                                                     int* __restrict__ counts, int* __restrict__ status) {
  __shared__ int mem[kCtrChunk];
  __shared__ int tmp[33];
  __shared__ int nmem;
  const int c = blockIdx.x;
  const int C = nclust[1];
  if (c == 0 && threadIdx.x == 0 && C > C_max) set_status(status, MP_ERR_CAPACITY);
  if (c >= C) return;
  const int tid = threadIdx.x;
  double acc = 0.0;   // thread tid < 2N owns coordinate tid
  int cnt = 0;
  for (int base = 0; base < T; base += kCtrChunk) {
    // flags of this chunk -> member positions (index order)
    constexpr int per = kCtrChunk / kCtrThreads;
    int f[per], s = 0;
#pragma unroll
    for (int r = 0; r < per; r++) {
      const int i = base + tid * per + r;
      f[r] = (i < T && labels[i] == c) ? 1 : 0;
      s += f[r];
    }
    const int lane = tid & 31, wid = tid >> 5;
    const int inc = warp_incl_scan(s);
    if (lane == 31) tmp[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      const int v = lane < kCtrThreads / 32 ? tmp[lane] : 0;
      const int vi = warp_incl_scan(v);
      if (lane < kCtrThreads / 32) tmp[lane] = vi - v;
      if (lane == kCtrThreads / 32 - 1) nmem = vi;
    }
    __syncthreads();
    int pos = tmp[wid] + inc - s;
#pragma unroll
    for (int r = 0; r < per; r++)
      if (f[r]) mem[pos++] = base + tid * per + r;
    __syncthreads();
    const int nm = nmem;
    if (tid < 2 * N)
      for (int m = 0; m < nm; m++) acc = __dadd_rn(acc, paths[(size_t)mem[m] * N * 2 + tid]);
    cnt += nm;
    __syncthreads();
  }
  if (c < C_max) {
    if (tid < 2 * N) centers[(size_t)c * N * 2 + tid] = __ddiv_rn(acc, (double)cnt);
    if (tid == 0) counts[c] = cnt;
  }
}

// ------------------------------------------------------------------ refine
struct RefineArgs {
  const double* paths;
  const double* ends;
  int Q, N;
  const double* centers;
  const int* counts;
  const int* nclust;
  int C_max, gw, gh;
  double cell;
  int k, max_cand;
  double* out;
  int* taken;
  int* status;
  int* cell_off;   // [gw*gh + 1]
  int* cell_cur;   // [gw*gh]
  int* cell_ids;   // [total registrations]
  int ids_cap;
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// cell index of coordinate v (floor(v / cell)), saturated to [-2, n + 1] before the int conversion
__device__ __forceinline__ int cell_of(double v, double cell, int n) {
  return (int)fmin(fmax(floor(__ddiv_rn(v, cell)), -2.0), (double)n + 1.0);
}

// cells of the (1-cell expanded) bounding box of segment s of centre c
__device__ __forceinline__ void seg_cells(const RefineArgs& A, const double* ctr, int s, int& cx0, int& cy0, int& cx1,
                                          int& cy1) {
  const double px = ctr[2 * s], py = ctr[2 * s + 1], qx = ctr[2 * s + 2], qy = ctr[2 * s + 3];
  cx0 = clampi(cell_of(fmin(px, qx), A.cell, A.gw) - 1, 0, A.gw - 1);
  cx1 = clampi(cell_of(fmax(px, qx), A.cell, A.gw) + 1, 0, A.gw - 1);
  cy0 = clampi(cell_of(fmin(py, qy), A.cell, A.gh) - 1, 0, A.gh - 1);
  cy1 = clampi(cell_of(fmax(py, qy), A.cell, A.gh) + 1, 0, A.gh - 1);
}

__global__ void refine_index_count_kernel(const RefineArgs A) {
  const int C = min(A.nclust[1], A.C_max);
  const int S = A.N - 1;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < C * S; e += gridDim.x * blockDim.x) {
    const int c = e / S, s = e - c * S;
    int x0, y0, x1, y1;
    seg_cells(A, A.centers + (size_t)c * A.N * 2, s, x0, y0, x1, y1);
    for (int y = y0; y <= y1; y++)
      for (int x = x0; x <= x1; x++) atomicAdd(&A.cell_off[y * A.gw + x], 1);
  }
}

__global__ void refine_index_fill_kernel(const RefineArgs A) {
  const int C = min(A.nclust[1], A.C_max);
  const int S = A.N - 1;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < C * S; e += gridDim.x * blockDim.x) {
    const int c = e / S, s = e - c * S;
    int x0, y0, x1, y1;
    seg_cells(A, A.centers + (size_t)c * A.N * 2, s, x0, y0, x1, y1);
    for (int y = y0; y <= y1; y++)
      for (int x = x0; x <= x1; x++) {
        const int slot = A.cell_off[y * A.gw + x] + atomicAdd(&A.cell_cur[y * A.gw + x], 1);
        if (slot < A.ids_cap) A.cell_ids[slot] = c;
        else set_status(A.status, MP_ERR_CAPACITY);
      }
  }
}

// exact slab test of segment p->q against the closed box [x0,x1] x [y0,y1] (oracle seg_box)
__device__ bool seg_box(double px, double py, double qx, double qy, double x0, double y0, double x1, double y1) {
  double t0 = 0.0, t1 = 1.0;
  const double d[2] = {__dsub_rn(qx, px), __dsub_rn(qy, py)}, p[2] = {px, py}, lo[2] = {x0, y0}, hi[2] = {x1, y1};
#pragma unroll
  for (int a = 0; a < 2; a++) {
    if (d[a] == 0.0) {
      if (p[a] < lo[a] || p[a] > hi[a]) return false;
    } else {
      double ta = __ddiv_rn(__dsub_rn(lo[a], p[a]), d[a]), tb = __ddiv_rn(__dsub_rn(hi[a], p[a]), d[a]);
      if (ta > tb) {
        const double t = ta;
        ta = tb;
        tb = t;
      }
      if (ta > t0) t0 = ta;
      if (tb < t1) t1 = tb;
      if (t0 > t1) return false;
    }
  }
  return true;
}

constexpr int kRefWarps = 4;

// shared bytes per query warp (16-B multiple so every warp's doubles stay aligned)
__host__ __device__ __forceinline__ size_t refine_warp_bytes(int cap, int C_max) {
  return ((size_t)cap * (2 * 4 + 4 + 8 + 4) + 16 + (size_t)((C_max + 31) / 32) * 4 + 15) & ~size_t(15);
}
constexpr int kRefMaxCand = 1024;

__global__ void __launch_bounds__(32 * kRefWarps) refine_query_kernel(const RefineArgs A) {
  extern __shared__ __align__(16) unsigned char rsm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int cap = A.max_cand;
  // per warp: raw ids [2*cap] int, unique ids [cap] int, dist [cap] double, order [cap] int,
  // seen-bitmap [ceil(C_max/32)] words (cleared again after each query)
  const int bm_words = (A.C_max + 31) / 32;
  unsigned char* base = rsm + (size_t)wid * refine_warp_bytes(cap, A.C_max);
  int* raw = reinterpret_cast<int*>(base);
  int* uniq = raw + 2 * cap;
  double* dist = reinterpret_cast<double*>(uniq + cap + (cap & 1));
  int* ord = reinterpret_cast<int*>(dist + cap);
  unsigned int* seen = reinterpret_cast<unsigned int*>(ord + cap);
  for (int w = lane; w < bm_words; w += 32) seen[w] = 0u;
  __syncwarp();
  const int N = A.N;
  const int C = min(A.nclust[1], A.C_max);
  for (int q = blockIdx.x * kRefWarps + wid; q < A.Q; q += gridDim.x * kRefWarps) {
    const double* path = A.paths + (size_t)q * N * 2;
    const double fx = A.ends[4 * q], fy = A.ends[4 * q + 1], lx = A.ends[4 * q + 2], ly = A.ends[4 * q + 3];
    // 1. raw candidate ids from the 4x4 cells around each end (the closed
    //    3x3-cell squares reach into the 4th row/column): lane = one cell
    int nraw = 0;
    bool over = false;
    {
      const int e = lane >> 4, cxo = (lane & 3) - 1, cyo = ((lane >> 2) & 3) - 1;
      const double px = e ? lx : fx, py = e ? ly : fy;
      const int x = cell_of(px, A.cell, A.gw) + cxo, y = cell_of(py, A.cell, A.gh) + cyo;
      int a = 0, b = 0;
      if (x >= 0 && x < A.gw && y >= 0 && y < A.gh) {
        a = min(A.cell_off[y * A.gw + x], A.ids_cap);
        b = min(A.cell_off[y * A.gw + x + 1], A.ids_cap);
      }
      const int len = b - a;
      const int incl = warp_incl_scan(len);
      nraw = __shfl_sync(0xffffffffu, incl, 31);
      if (nraw <= 2 * cap)
        for (int t = 0; t < len; t++) raw[incl - len + t] = A.cell_ids[a + t];
    }
    if (nraw > 2 * cap) over = true;
    __syncwarp();
    // 2. unique ids (first claim of each id in the seen-bitmap), then ascending
    int nu = 0;
    if (!over) {
      for (int base0 = 0; base0 < nraw; base0 += 32) {
        const int t = base0 + lane;
        bool first = false;
        int v = 0;
        if (t < nraw) {
          v = raw[t];
          const unsigned int bit = 1u << (v & 31);
          first = !(atomicOr(&seen[v >> 5], bit) & bit);
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, first);
        if (first) {
          const int slot = nu + __popc(bal & lanemask_lt());
          if (slot < cap) ord[slot] = v;
        }
        nu += __popc(bal);
      }
      __syncwarp();
      for (int t = lane; t < nraw; t += 32) seen[raw[t] >> 5] = 0u;   // clear for the next query
      if (nu > cap) over = true;
    }
    __syncwarp();
    if (over) {
      if (lane == 0) {
        set_status(A.status, MP_ERR_CAPACITY);
        A.out[4 * q] = fx;
        A.out[4 * q + 1] = fy;
        A.out[4 * q + 2] = lx;
        A.out[4 * q + 3] = ly;
        A.taken[q] = 0;
      }
      __syncwarp();
      continue;
    }
    for (int t = lane; t < nu; t += 32) {   // sort unique ids by rank
      const int v = ord[t];
      int r = 0;
      for (int u = 0; u < nu; u++) r += ord[u] < v;
      uniq[r] = v;
    }
    __syncwarp();
    // 3. exact test + distance for each candidate (in id order), compacted
    int nc = 0;
    for (int base0 = 0; base0 < nu; base0 += 32) {
      const int t = base0 + lane;
      bool hit = false;
      double d = 0.0;
      int c = 0;
      if (t < nu) {
        c = uniq[t];
        const double* ctr = A.centers + (size_t)c * N * 2;
        for (int e = 0; e < 2 && !hit; e++) {
          const double px = e ? lx : fx, py = e ? ly : fy;
          const double gx = floor(__ddiv_rn(px, A.cell)), gy = floor(__ddiv_rn(py, A.cell));
          const double x0 = __dmul_rn(__dsub_rn(gx, 1.0), A.cell), y0 = __dmul_rn(__dsub_rn(gy, 1.0), A.cell);
          const double x1 = __dmul_rn(__dadd_rn(gx, 2.0), A.cell), y1 = __dmul_rn(__dadd_rn(gy, 2.0), A.cell);
          for (int i = 0; i + 1 < N && !hit; i++)
            hit = seg_box(ctr[2 * i], ctr[2 * i + 1], ctr[2 * i + 2], ctr[2 * i + 3], x0, y0, x1, y1);
        }
        if (hit) d = path_dist(path, ctr, N);
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, hit);
      if (hit) {
        const int slot = nc + __popc(bal & lanemask_lt());
        raw[slot] = c;      // reuse raw[] for the hit ids
        dist[slot] = d;
      }
      nc += __popc(bal);
    }
    __syncwarp();
    // 4. rank by (distance, id)
    for (int t = lane; t < nc; t += 32) {
      const double dv = dist[t];
      const int cv = raw[t];
      int r = 0;
      for (int u = 0; u < nc; u++) r += (dist[u] < dv || (dist[u] == dv && raw[u] < cv));
      ord[r] = t;
    }
    __syncwarp();
    // 5. take until the member counts reach k; weighted medians (lane 0; <= k entries)
    if (lane == 0) {
      int ntk = 0, wsum = 0;
      while (ntk < nc && wsum < A.k) wsum += A.counts[raw[ord[ntk++]]];
      double res[4] = {fx, fy, lx, ly};
      if (ntk > 0) {
        for (int qq = 0; qq < 4; qq++) {
          const int pt = qq < 2 ? 0 : N - 1, ax = qq & 1;
          // the value at position ceil(W/2) of the weight-expanded ascending list:
          // walk the distinct values upwards, accumulating their weights
          const int target = (wsum + 1) / 2;
          double lo_bound = -INFINITY;
          int acc = 0;
          double val = 0.0;
          while (true) {
            // next distinct value above lo_bound and its total weight
            double nv = INFINITY;
            for (int t = 0; t < ntk; t++) {
              const double v = A.centers[(size_t)raw[ord[t]] * N * 2 + 2 * pt + ax];
              if (v > lo_bound && v < nv) nv = v;
            }
            int w = 0;
            for (int t = 0; t < ntk; t++) {
              const int cc = raw[ord[t]];
              if (A.centers[(size_t)cc * N * 2 + 2 * pt + ax] == nv) w += A.counts[cc];
            }
            if (nv == INFINITY) break;   // (unreachable for finite centres)
            acc += w;
            val = nv;
            lo_bound = nv;
            if (acc >= target) break;
          }
          res[qq] = val;
        }
      }
      for (int qq = 0; qq < 4; qq++) A.out[4 * q + qq] = res[qq];
      A.taken[q] = ntk;
    }
    __syncwarp();
  }
}

}  // namespace mpk

using namespace mpk;

extern "C" mp_status mp_track_resample(const float* d_boxes, const int32_t* d_track_off, int32_t T, int32_t N,
                                       double* d_paths, double* d_ends, void* stream) {
  if (T < 0 || N < 2 || N > kMaxN) return MP_ERR_INVALID;
  if (T == 0) return MP_OK;
  if (!d_track_off || !d_paths) return MP_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  track_resample_kernel<<<(T + 127) / 128, 128, 0, s>>>(d_boxes, d_track_off, T, N, d_paths, d_ends);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

struct DbWs {
  size_t adj, coremask, parent, flag, flag2, core, cnt, total;
};

static bool dbscan_layout(int T, DbWs* L) {
  if (T < 0 || T > 65536) return false;
  const size_t words = (size_t)(T + 31) / 32;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  L->adj = 0;
  L->coremask = al(L->adj + (size_t)T * words * 4);
  L->parent = al(L->coremask + words * 4);
  L->flag = al(L->parent + (size_t)T * 4);
  L->flag2 = al(L->flag + (size_t)T * 4);
  L->core = al(L->flag2 + (size_t)T * 4);
  L->cnt = al(L->core + (size_t)T);
  L->total = al(L->cnt + 4 * sizeof(int));
  return true;
}

extern "C" size_t mp_dbscan_workspace_size(int32_t T) {
  DbWs L;
  return dbscan_layout(T, &L) ? L.total : 0;
}

extern "C" mp_status mp_dbscan(const double* d_paths, int32_t T, int32_t N, double eps, int32_t min_pts,
                               int32_t* d_labels, uint8_t* d_is_core, int32_t* d_nclust, void* d_ws, size_t ws_bytes,
                               void* stream) {
  DbWs L;
  if (!dbscan_layout(T, &L) || N < 2 || N > kMaxN || !(eps > 0.0) || min_pts < 1 || !d_nclust) return MP_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  if (T == 0) {
    MP_CUDA_TRY(cudaMemsetAsync(d_nclust, 0, 2 * sizeof(int), s));
    return MP_OK;
  }
  if (!d_paths || !d_labels || !d_ws || ws_bytes < L.total) return MP_ERR_INVALID;
  unsigned char* ws = (unsigned char*)d_ws;
  uint32_t* adj = (uint32_t*)(ws + L.adj);
  uint32_t* coremask = (uint32_t*)(ws + L.coremask);
  int* parent = (int*)(ws + L.parent);
  int* flag = (int*)(ws + L.flag);
  int* flag2 = (int*)(ws + L.flag2);
  int* cnt = (int*)(ws + L.cnt);
  uint8_t* core = ws + L.core;
  const int words = (T + 31) / 32;
  MP_CUDA_TRY(cudaMemsetAsync(coremask, 0, (size_t)words * 4, s));
  const size_t smem = (size_t)(kAdjRows + 32) * N * 2 * sizeof(double);
  const double prune = eps * (double)N * (1.0 + 9.094947017729282e-13);   // eps*N*(1 + 2^-40)
  dim3 grid(words, (T + kAdjRows - 1) / kAdjRows);
  dbscan_adj_kernel<<<grid, 32 * kAdjRows, smem, s>>>(d_paths, T, N, eps, prune, words, adj);
  MP_CUDA_TRY(cudaGetLastError());
  dbscan_core_kernel<<<(T + 255) / 256, 256, 0, s>>>(adj, T, words, min_pts, core, coremask, parent);
  MP_CUDA_TRY(cudaGetLastError());
  dbscan_union_kernel<<<(T * 32 + 255) / 256, 256, 0, s>>>(adj, T, words, coremask, parent);
  MP_CUDA_TRY(cudaGetLastError());
  dbscan_root_kernel<<<(T + 255) / 256, 256, 0, s>>>(T, core, parent, flag);
  MP_CUDA_TRY(cudaGetLastError());
  scan_kernel<<<1, 1024, 0, s>>>(flag, T, &cnt[0]);   // flag -> cluster id of each root
  MP_CUDA_TRY(cudaGetLastError());
  dbscan_label_kernel<<<(T + 255) / 256, 256, 0, s>>>(adj, T, words, core, coremask, parent, flag, d_labels, flag2,
                                                      d_is_core);
  MP_CUDA_TRY(cudaGetLastError());
  scan_kernel<<<1, 1024, 0, s>>>(flag2, T, &cnt[1]);
  MP_CUDA_TRY(cudaGetLastError());
  dbscan_noise_kernel<<<(T + 255) / 256, 256, 0, s>>>(T, flag2, cnt, d_labels, d_nclust);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" mp_status mp_cluster_centers(const double* d_paths, int32_t T, int32_t N, const int32_t* d_labels,
                                        const int32_t* d_nclust, int32_t C_max, double* d_centers, int32_t* d_counts,
                                        int32_t* d_status, void* stream) {
  if (T < 0 || N < 2 || N > kMaxN || C_max < 0 || !d_nclust || !d_status) return MP_ERR_INVALID;
  if (C_max == 0) return MP_OK;
  if (!d_centers || !d_counts || (T > 0 && (!d_paths || !d_labels))) return MP_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  cluster_centers_kernel<<<C_max, kCtrThreads, 0, s>>>(d_paths, T, N, d_labels, d_nclust, C_max, d_centers, d_counts,
                                                      d_status);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

static bool refine_grid(int W, int H, double cell, int* gw, int* gh) {
  if (W < 1 || H < 1 || !(cell > 0.0)) return false;
  const double a = ceil((double)W / cell), b = ceil((double)H / cell);
  if (a > 16384 || b > 16384) return false;
  *gw = (int)a;
  *gh = (int)b;
  return true;
}

struct RefWs {
  size_t off, cur, ids, total;
  int ids_cap;
};

static bool refine_layout(int W, int H, double cell, int C_max, int N, RefWs* L) {
  int gw, gh;
  if (!refine_grid(W, H, cell, &gw, &gh) || C_max < 0 || C_max > 65536 || N < 2 || N > kMaxN) return false;
  const size_t G = (size_t)gw * gh;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  // registrations: each segment's 1-cell expanded bbox; bounded by C_max * (N-1) * 16 cells on average (checked)
  const size_t cap = (size_t)C_max * (N - 1) * 64 + 1024;
  L->off = 0;
  L->cur = al((G + 1) * 4);
  L->ids = al(L->cur + G * 4);
  L->total = al(L->ids + cap * 4);
  L->ids_cap = (int)(cap < ((size_t)1 << 30) ? cap : ((size_t)1 << 30));
  return true;
}

extern "C" size_t mp_refine_workspace_size(int32_t W, int32_t H, double cell, int32_t C_max, int32_t N) {
  RefWs L;
  return refine_layout(W, H, cell, C_max, N, &L) ? L.total : 0;
}

extern "C" mp_status mp_refine_tracks(const double* d_paths, const double* d_ends, int32_t Q, int32_t N,
                                      const double* d_centers, const int32_t* d_counts, const int32_t* d_nclust,
                                      int32_t C_max, int32_t W, int32_t H, double cell, int32_t k, int32_t max_cand,
                                      double* d_out, int32_t* d_taken, int32_t* d_status, void* d_ws,
                                      size_t ws_bytes, void* stream) {
  RefWs L;
  if (!refine_layout(W, H, cell, C_max, N, &L) || Q < 0 || k < 1 || max_cand < 1 || max_cand > kRefMaxCand ||
      !d_status || !d_nclust)
    return MP_ERR_INVALID;
  if (Q == 0) return MP_OK;
  if (!d_paths || !d_ends || !d_out || !d_taken || !d_ws || ws_bytes < L.total) return MP_ERR_INVALID;
  if (C_max > 0 && (!d_centers || !d_counts)) return MP_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  RefineArgs A;
  A.paths = d_paths;
  A.ends = d_ends;
  A.Q = Q;
  A.N = N;
  A.centers = d_centers;
  A.counts = d_counts;
  A.nclust = d_nclust;
  A.C_max = C_max;
  refine_grid(W, H, cell, &A.gw, &A.gh);
  A.cell = cell;
  A.k = k;
  A.max_cand = max_cand;
  A.out = d_out;
  A.taken = d_taken;
  A.status = d_status;
  unsigned char* ws = (unsigned char*)d_ws;
  A.cell_off = (int*)(ws + L.off);
  A.cell_cur = (int*)(ws + L.cur);
  A.cell_ids = (int*)(ws + L.ids);
  A.ids_cap = L.ids_cap;
  const int G = A.gw * A.gh;
  MP_CUDA_TRY(cudaMemsetAsync(A.cell_off, 0, (size_t)(G + 1) * 4, s));
  MP_CUDA_TRY(cudaMemsetAsync(A.cell_cur, 0, (size_t)G * 4, s));
  int dev = 0, sms = 0;
  MP_CUDA_TRY(cudaGetDevice(&dev));
  MP_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (C_max > 0) {
    refine_index_count_kernel<<<sms * 4, 256, 0, s>>>(A);
    MP_CUDA_TRY(cudaGetLastError());
  }
  scan_kernel<<<1, 1024, 0, s>>>(A.cell_off, G + 1, A.cell_cur);   // cell_cur[0] <- total (then re-zeroed)
  MP_CUDA_TRY(cudaGetLastError());
  MP_CUDA_TRY(cudaMemsetAsync(A.cell_cur, 0, (size_t)G * 4, s));
  if (C_max > 0) {
    refine_index_fill_kernel<<<sms * 4, 256, 0, s>>>(A);
    MP_CUDA_TRY(cudaGetLastError());
  }
  const size_t per_warp = refine_warp_bytes(max_cand, C_max);
  const size_t smem = per_warp * kRefWarps;
  if (smem > 200 * 1024) return MP_ERR_UNSUPPORTED;
  MP_CUDA_TRY(cudaFuncSetAttribute(refine_query_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = (Q + kRefWarps - 1) / kRefWarps < sms * 16 ? (Q + kRefWarps - 1) / kRefWarps : sms * 16;
  refine_query_kernel<<<grid, 32 * kRefWarps, smem, s>>>(A);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}
