// mp_plan.cu — steps a1-a4 of the proxy-guided window path on sm_100a:
// threshold the proxy score grid, label 4-connected components of positive
// cells, run the greedy agglomerative merge of PAPER.md:184 and place one
// window per cluster.  Readings R1-R14 are in DESIGN.md §3.
//
// Launches (all on the caller's stream, no host sync):
//   memset                     tier queue counter
//   K1-K3 plan_fast_kernel     one 128-thread CTA per frame (shared memory for
//                              <= 256 runs): ballot threshold -> run extraction
//                              -> shared-memory union-find over runs ->
//                              component bboxes -> warp-0 greedy merge ->
//                              placement into per-frame scratch; frames with
//                              more runs are queued
//         plan_full_kernel     persistent over the queue, shared memory for
//                              R*ceil(C/2) runs (checkerboard worst case)
//   K4a   plan_scan_kernel     one CTA: frame CSR + per-class slot bases
//   K4b   plan_scatter_kernel  warp per frame: final window records + slots
#include <climits>

#include "mp_internal.cuh"

namespace mpk {

struct PlanArgs {
  int W, H, cw, ch, R, C, words, k, full, maxc;
  float b;
  int order[kMaxClasses];          // size indices sorted by (w*h, w, h)  (R6)
  int sw[kMaxClasses], sh[kMaxClasses];
  long long cost[kMaxClasses];
};

// R6: smallest-area size containing (bw, bh); ties by smaller w then h.
__device__ __forceinline__ int smallest_size(const PlanArgs& P, int bw, int bh) {
  for (int q = 0; q < P.k; q++) {
    int i = P.order[q];
    if (P.sw[i] >= bw && P.sh[i] >= bh) return i;
  }
  return P.full;   // unreachable: (W,H) is in S
}

// R1: pixel extent of a cell bbox, last row/col clipped to the frame.
__device__ __forceinline__ void extent(const PlanArgs& P, int c0, int r0, int c1, int r1, int& px0,
                                       int& py0, int& bw, int& bh) {
  px0 = c0 * P.cw;
  py0 = r0 * P.ch;
  bw = min((c1 + 1) * P.cw, P.W) - px0;
  bh = min((r1 + 1) * P.ch, P.H) - py0;
}

__device__ __forceinline__ int uf_find(volatile int* parent, int x) {
  while (true) {
    int p = parent[x];
    if (p == x) return x;
    int gp = parent[p];
    // path halving; the store is an atomic CAS so concurrent finds/links never
    // race on a plain write (gp is an ancestor either way)
    if (gp != p) atomicCAS(const_cast<int*>(parent + x), p, gp);
    x = p;
  }
}

// Link the larger root under the smaller one, so every final root is the
// smallest run index of its component (= its first run in row-major order).
__device__ __forceinline__ void uf_unite(int* parent, int a, int b) {
  volatile int* vp = parent;
  while (true) {
    a = uf_find(vp, a);
    b = uf_find(vp, b);
    if (a == b) return;
    if (a > b) {
      int t = a;
      a = b;
      b = t;
    }
    int old = atomicCAS(&parent[b], b, a);
    if (old == b) return;
    b = old;
  }
}

// 16-bit min (kMax = false) / max of a non-negative value into a shared or
// global int16 entry: a CAS loop on the aligned 32-bit word holding it (there
// are no 16-bit atomicMin / atomicMax); the neighbouring entry of the word is
// carried through unchanged.
template <bool kMax>
__device__ __forceinline__ void atomic_minmax_s16(short* p, int v) {
  unsigned* w = (unsigned*)((size_t)p & ~(size_t)3);
  const int sh = ((size_t)p & 2) ? 16 : 0;
  unsigned old = *(volatile unsigned*)w;
  while (true) {
    const int cur = (short)(old >> sh);
    if (kMax ? cur >= v : cur <= v) return;
    const unsigned nv = (old & ~(0xFFFFu << sh)) | ((unsigned)(v & 0xFFFF) << sh);
    const unsigned prev = atomicCAS(w, old, nv);
    if (prev == old) return;
    old = prev;
  }
}

struct PlanSmem {
  uint32_t* bits;
  int *row_off, *tmp, *parent, *cid, *run;
  short *bc0, *br0, *bc1, *br1;   // component boxes in cells (int16 like the runs: half the bytes)
  short *rrow, *rcs, *rce;
  unsigned char *csz, *memb;
};

__host__ __device__ inline size_t plan_smem_bytes(int R, int words, int maxc, PlanSmem* out,
                                                  unsigned char* base) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 15) & ~size_t(15);
    return base ? base + o : nullptr;
  };
  PlanSmem s;
  s.bits = (uint32_t*)take(sizeof(uint32_t) * R * words);
  s.row_off = (int*)take(sizeof(int) * (R + 1));
  s.tmp = (int*)take(sizeof(int) * 40);
  s.run = (int*)take(sizeof(int) * kMaxClasses);
  // per-component arrays hold one spare entry: the CTA-cooperative merge
  // appends a merged cluster before it compacts (coop_merge, cap = maxc + 1)
  s.parent = (int*)take(sizeof(int) * (maxc + 1));
  s.cid = (int*)take(sizeof(int) * (maxc + 1));
  s.bc0 = (short*)take(sizeof(short) * (maxc + 1));
  s.br0 = (short*)take(sizeof(short) * (maxc + 1));
  s.bc1 = (short*)take(sizeof(short) * (maxc + 1));
  s.br1 = (short*)take(sizeof(short) * (maxc + 1));
  s.rrow = (short*)take(sizeof(short) * maxc);
  s.rcs = (short*)take(sizeof(short) * maxc);
  s.rce = (short*)take(sizeof(short) * maxc);
  s.csz = (unsigned char*)take(maxc + 1);
  s.memb = (unsigned char*)take(maxc + 1);
  if (out) *out = s;
  return off;
}

constexpr int kPlanThreads = 128;      // full-capacity tier (128 threads: two CTAs fit beside a gather CTA)
constexpr int kFastThreads = 128;      // fast tier: frames with <= kFastCap runs
constexpr int kFastCap = 256;
// full tier: runs held in shared memory (~24 KB at 960 runs with int16
// component boxes + ~1.5 KB static: three CTAs fit in the ~108 KB a c4 f32
// gather CTA leaves of an SM and two in the ~55 KB beside the u8 ring, so all
// 300 frames of a c4 batch plan in one wave beside the gather); beyond -> the
// huge tier (global scratch).  c4 (4K, 68 x 120 cells) frames have
// 756-888 runs.
constexpr int kMidCap = 960;
// largest cell grid: the fast / full tiers keep only the bit rows and run
// offsets of the grid in shared memory, the huge tier's per-run arrays are in
// global scratch (R*ceil(C/2) runs), and run rows / columns are int16
constexpr int kMaxCells = 65536;
constexpr int kFullGrid = 4;        // plan_full CTAs per SM (one frame each at c4: 300 frames)
constexpr int kHugeGrid = 1;        // plan_huge CTAs per SM (each owns a global scratch slot)

constexpr int kCoopMergeMin = 96;   // components above which the whole CTA runs the merge

// Block-wide minimum of a 64-bit key; `red` = 2 x kRedWarps shared slots
// used alternately (par) so consecutive calls need one barrier each.
constexpr int kRedWarps = 8;   // every planner CTA has <= 256 threads
__device__ __forceinline__ unsigned long long block_min_u64(unsigned long long v, unsigned long long* red,
                                                            int& par) {
  v = warp_min_u64(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned long long* r = red + kRedWarps * par;
  if (lane == 0) r[wid] = v;
  __syncthreads();
  unsigned long long m = ~0ull;
  for (int w = 0; w < nw; w++) m = r[w] < m ? r[w] : m;
  par ^= 1;
  return m;
}

extern __shared__ __align__(16) unsigned char smem_raw[];

// a3 with the whole CTA (exactly the P:184 greedy of the warp-0 path below:
// same nearest-neighbour metric and ties, same ascending absorption, strict
// acceptance, remove + append); used when a frame has many components.
//
// The cluster list is kept as an append-only array with dead flags instead
// of being compacted after every accepted merge: members are flagged dead
// and the merged cluster is appended at the end.  The alive entries keep
// exactly the order of the compacted list (compaction is stable and appends
// at the end), so positions compare the same way for the R5 tie rule and the
// R7 ascending absorption, and "i -= before_i" becomes "the next alive entry
// after i".  The array is compacted only at the start of a pass and when it
// is full (capacity `cap`).  Dense frames accept most proposals (c4 4K
// drone frames: ~175 steps, ~90 % accepted), so this removes the per-merge
// block scan and chunked moves (~10 of the ~14 barriers of an accepted step).
//
// Per step (3 barriers): block arg-min for the nearest alive neighbour; every
// warp ballots its 32-entry chunks against the initial merged box (a cluster
// that does not fit it can never fit the grown box, R7); warp 0 walks only
// those candidates in ascending order, decides, flags the members dead,
// appends the merged cluster and finds the next i, then publishes.
constexpr int kAbsList = 64;   // absorbed members recorded by warp 0 (beyond: block-wide mark)

#ifdef MP_PLAN_PROF
// development builds only (-DMP_PLAN_PROF): thread 0's clock64 cycles per
// cooperative-merge phase, summed over all CTAs: [0] arg-min + its barrier,
// [1] fit ballots + barrier, [2] warp-0 walk + publish barrier, [3] steps
__device__ unsigned long long g_plan_prof[4];
#define MP_PROF_T(v) long long v = clock64();
#define MP_PROF_ADD(k, d) if (threadIdx.x == 0) atomicAdd(&g_plan_prof[k], (unsigned long long)(d));
#else
#define MP_PROF_T(v)
#define MP_PROF_ADD(k, d)
#endif

// FW: words of initial-fit ballots, one per 32 list entries (len <= 32 FW):
// the shared-memory tiers (<= kMidCap + 1 entries) keep their static shared
// memory small so three full-tier CTAs fit beside a gather CTA.
template <int FW>
__device__ int coop_merge(const PlanArgs& P, const PlanSmem& S, int n, int cap) {
  __shared__ unsigned long long red[2 * kRedWarps];
  __shared__ int pub[8];
  __shared__ uint32_t fitm[FW];
  __shared__ int absl[kAbsList];
  int par = 0;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, BS = blockDim.x, NW = BS >> 5;
  const long long* T = P.cost;
  unsigned char* dead = S.memb;   // dead flag per entry
  int* gen_of = S.cid;            // entry absorbed in proposal number gen_of[q] (overflow path)
  int* scan = S.parent;           // compaction scratch (free once components are labelled)
  int len = n, alive = n, gen = 0;
  for (int q = tid; q < len; q += BS) {
    dead[q] = 0;
    gen_of[q] = -1;
  }
  __syncthreads();
  // stable removal of the dead entries; returns the new position of entry
  // `keep_pos` (alive, or == len -> the new len)
  auto compact = [&](int keep_pos) -> int {
    for (int q = tid; q < len; q += BS) scan[q] = dead[q] ? 0 : 1;
    __syncthreads();
    const int kept = block_excl_scan_smem(scan, len, S.tmp);
    const int np = keep_pos < len ? scan[keep_pos] : kept;
    for (int base = 0; base < len; base += BS) {
      const int q = base + tid;
      bool keep = false;
      int v0 = 0, v1 = 0, v2 = 0, v3 = 0, d = 0;
      unsigned char vs = 0;
      if (q < len) {
        keep = !dead[q];
        d = scan[q];
        v0 = S.bc0[q]; v1 = S.br0[q]; v2 = S.bc1[q]; v3 = S.br1[q]; vs = S.csz[q];
      }
      __syncthreads();   // elements only move to lower indices: read the chunk before writing it
      if (keep) {
        S.bc0[d] = v0; S.br0[d] = v1; S.bc1[d] = v2; S.br1[d] = v3; S.csz[d] = vs;
      }
      __syncthreads();
    }
    for (int q = tid; q < kept; q += BS) {
      dead[q] = 0;
      gen_of[q] = -1;
    }
    __syncthreads();
    len = kept;
    return np;
  };
  bool again = true;
  while (again) {
    again = false;
    if (len != alive) compact(len);   // each pass starts on the compacted list
    int i = 0;
    while (i < len && alive >= 2) {
      if (len >= cap) i = compact(i);   // full: no room to append a merged cluster
      gen++;
      MP_PROF_T(t0)
      const int ic0 = S.bc0[i], ir0 = S.br0[i], ic1 = S.bc1[i], ir1 = S.br1[i];
      const int sx = ic0 + ic1, sy = ir0 + ir1;
      unsigned long long best = ~0ull;
      for (int j = tid; j < len; j += BS) {
        if (j == i || dead[j]) continue;
        const int dx = sx - (S.bc0[j] + S.bc1[j]);
        const int dy = sy - (S.br0[j] + S.br1[j]);
        const unsigned long long key = ((unsigned long long)(unsigned)(dx * dx + dy * dy) << 32) | (unsigned)j;
        best = key < best ? key : best;
      }
      best = block_min_u64(best, red, par);
      MP_PROF_T(t1)
      const int j = (int)(best & 0xffffffffu);
      int m0 = min(ic0, S.bc0[j]), n0 = min(ir0, S.br0[j]);
      int m1 = max(ic1, S.bc1[j]), n1 = max(ir1, S.br1[j]);
      int px0, py0, bw, bh;
      extent(P, m0, n0, m1, n1, px0, py0, bw, bh);
      const int s = smallest_size(P, bw, bh);
      const int ws = P.sw[s], hs = P.sh[s];
      // initial-fit ballots (all warps)
      const int nch = (len + 31) >> 5;
      for (int c = wid; c < nch; c += NW) {
        const int q = (c << 5) + lane;
        bool fit = false;
        if (q < len && q != i && q != j && !dead[q]) {
          int qx, qy, qw, qh;
          extent(P, min(m0, S.bc0[q]), min(n0, S.br0[q]), max(m1, S.bc1[q]), max(n1, S.br1[q]), qx, qy, qw, qh);
          fit = (qw <= ws) && (qh <= hs);
        }
        const uint32_t msk = __ballot_sync(0xffffffffu, fit);
        if (lane == 0) fitm[c] = msk;
      }
      __syncthreads();
      MP_PROF_T(t2)
      if (wid == 0) {
        // absorption (k ascending, each fitting cluster at once, R7) over the
        // initial candidates only
        long long sum = T[S.csz[i]] + T[S.csz[j]];
        int n_abs = 0;
        for (int c0 = 0; c0 < nch; c0 += 32) {
          const uint32_t word = (c0 + lane < nch) ? fitm[c0 + lane] : 0u;
          uint32_t nz = __ballot_sync(0xffffffffu, word != 0u);
          while (nz) {
            const int c = c0 + __ffs(nz) - 1;
            nz &= nz - 1;
            // lanes re-test this word's remaining candidates against the current
            // box at once; the first fitting one is absorbed and the ones before
            // it dropped (they cannot fit the grown box either)
            uint32_t rem = fitm[c];
            while (rem) {
              const int q = (c << 5) + lane;
              bool fit = false;
              if ((rem >> lane) & 1u) {
                int qx, qy, qw, qh;
                extent(P, min(m0, S.bc0[q]), min(n0, S.br0[q]), max(m1, S.bc1[q]), max(n1, S.br1[q]), qx, qy, qw,
                       qh);
                fit = (qw <= ws) && (qh <= hs);
              }
              const uint32_t fm = __ballot_sync(0xffffffffu, fit);
              if (!fm) break;
              const int bq = __ffs(fm) - 1;
              const int qq = (c << 5) + bq;
              m0 = min(m0, S.bc0[qq]);
              n0 = min(n0, S.br0[qq]);
              m1 = max(m1, S.bc1[qq]);
              n1 = max(n1, S.br1[qq]);
              sum += T[S.csz[qq]];
              if (lane == 0) {
                if (n_abs < kAbsList) absl[n_abs] = qq;
                else gen_of[qq] = gen;
              }
              n_abs++;
              rem &= (bq == 31) ? 0u : ~((2u << bq) - 1u);
            }
          }
        }
        // (d) accept iff strictly faster (R8): members dead, merged appended
        const bool acc = T[s] < sum;
        int ni = i + 1;
        if (acc) {
          __syncwarp();   // absl / gen_of writes of lane 0
          if (lane == 0) {
            dead[i] = 1;
            dead[j] = 1;
            S.bc0[len] = m0; S.br0[len] = n0; S.bc1[len] = m1; S.br1[len] = n1;
            S.csz[len] = (unsigned char)s;
            dead[len] = 0;
            gen_of[len] = -1;
          }
          for (int a = lane; a < min(n_abs, kAbsList); a += 32) dead[absl[a]] = 1;
          if (n_abs > kAbsList)
            for (int q = lane; q < len; q += 32)
              if (gen_of[q] == gen) dead[q] = 1;
          __syncwarp();
          // next alive entry after i (the appended cluster at len is alive)
          ni = len + 1;
          for (int base = i + 1; base <= len; base += 32) {
            const int q = base + lane;
            const uint32_t al = __ballot_sync(0xffffffffu, q <= len && !dead[q]);
            if (al) {
              ni = base + __ffs(al) - 1;
              break;
            }
          }
        } else {
          for (int base = i + 1; base < len + 32; base += 32) {
            const int q = base + lane;
            const uint32_t al = __ballot_sync(0xffffffffu, q < len && !dead[q]);
            if (al || base >= len) {
              ni = al ? base + __ffs(al) - 1 : len;
              break;
            }
          }
        }
        if (lane == 0) {
          pub[0] = acc ? 1 : 0;
          pub[1] = ni;
          pub[2] = n_abs;
        }
      }
      __syncthreads();
      MP_PROF_T(t3)
      MP_PROF_ADD(0, t1 - t0)
      MP_PROF_ADD(1, t2 - t1)
      MP_PROF_ADD(2, t3 - t2)
      MP_PROF_ADD(3, 1)
      const int acc = pub[0];
      i = pub[1];
      if (acc) {
        alive -= pub[2] + 1;   // members (2 + n_abs) removed, merged added
        len++;
        again = true;
      }
    }
  }
  if (len != alive) compact(len);
  return len;
}

// The whole per-frame plan (a1-a4) with the CTA; `cap` = run/component
// capacity of the shared-memory layout.  Returns false (having queued the
// frame) if the frame has more runs than `cap`.  GB (the huge tier): the
// per-run and per-component arrays live in the CTA's global scratch slot
// `gbig` (capacity maxc, L2-resident) and only the bit rows and scan scratch
// in shared memory; a separate instantiation, so the shared-memory tiers keep
// plain LDS/STS accesses.
// FW: fit-ballot words of the cooperative merge (list length <= 32 FW)
constexpr int kFwSmall = (kMidCap + 1 + 31) / 32 + 1;   // shared-memory tiers
constexpr int kFwFull = 256;                             // sweep / window-set kernels (whole frame in smem)
constexpr int kFwHuge = kMaxCells / 32 + 2;              // global tier: up to R*ceil(C/2) + 1 <= kMaxCells + 1 entries
template <bool GB = false, int FW = kFwFull>
__device__ __forceinline__ bool plan_frame(const PlanArgs& P, int f, int cap, const float* __restrict__ scores,
                                           uint32_t* __restrict__ mask_out, int4* __restrict__ ws_win,
                                           int* __restrict__ ws_count, int* __restrict__ ws_cls,
                                           int* __restrict__ q_cnt, int* __restrict__ q_list,
                                           long long* est_out = nullptr, unsigned char* gbig = nullptr,
                                           const unsigned char* rk = nullptr, int jpos = 0) {
  PlanSmem S;
  plan_smem_bytes(P.R, P.words, GB ? 0 : cap, &S, smem_raw);
  if (GB) {
    PlanSmem G;
    plan_smem_bytes(P.R, P.words, P.maxc, &G, gbig);
    S.parent = G.parent; S.cid = G.cid;
    S.bc0 = G.bc0; S.br0 = G.br0; S.bc1 = G.bc1; S.br1 = G.br1;
    S.rrow = G.rrow; S.rcs = G.rcs; S.rce = G.rce;
    S.csz = G.csz; S.memb = G.memb;
    cap = P.maxc;
  }
  const int R = P.R, C = P.C, words = P.words;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarps = blockDim.x >> 5;
  const float* sc = scores + (size_t)f * R * C;

  // ---- a1: threshold, one warp-ballot per 32 cells of a row (R2);
  // four (row, word) loads per warp in flight before the ballots.
  const int RW = R * words;
  if (rk) {
    // NEXT-1 single pass: the frame's cells were ranked once against the
    // ascending thresholds (rk[c] = #{j : score_c > B_j}), so score_c > B_jpos
    // <=> rk[c] > jpos; the score grid is not re-read per threshold
    for (int rw = wid; rw < RW; rw += nwarps) {
      const int r = rw / words, c = (rw - r * words) * 32 + lane;
      const uint32_t m = __ballot_sync(0xffffffffu, c < C && (int)rk[r * C + c] > jpos);
      if (lane == 0) S.bits[rw] = m;
    }
  } else
  for (int base = wid; base < RW; base += 4 * nwarps) {
    float v[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int rw = base + u * nwarps;
      v[u] = -INFINITY;
      if (rw < RW) {
        const int r = rw / words, c = (rw - r * words) * 32 + lane;
        if (c < C) v[u] = __ldg(sc + (size_t)r * C + c);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int rw = base + u * nwarps;
      if (rw < RW) {
        const uint32_t m = __ballot_sync(0xffffffffu, v[u] > P.b);   // NaN -> false
        if (lane == 0) {
          S.bits[rw] = m;
          if (mask_out) mask_out[(size_t)f * RW + rw] = m;
        }
      }
    }
  }
  __syncthreads();

  // ---- a2: horizontal runs of positive cells (run starts = m & ~(m<<1 | carry))
  for (int r = tid; r < R; r += blockDim.x) {
    int n = 0;
    uint32_t prev = 0;
    for (int w = 0; w < words; w++) {
      const uint32_t m = S.bits[r * words + w];
      n += __popc(m & ~((m << 1) | (prev >> 31)));
      prev = m;
    }
    S.row_off[r] = n;
  }
  __syncthreads();
  const int nruns = block_excl_scan_smem(S.row_off, R, S.tmp);
  const int ext_cap = cap + 1;   // entries of the per-component arrays
  if (nruns > cap) {   // too many runs for this tier's shared memory: queue for the next tier
    if (tid == 0) q_list[atomicAdd(q_cnt, 1)] = f;
    return false;
  }
  for (int r = tid; r < R; r += blockDim.x) {
    const int base = S.row_off[r];
    int ns = 0, ne = 0;
    uint32_t prev = 0;
    for (int w = 0; w < words; w++) {
      const uint32_t m = S.bits[r * words + w];
      const uint32_t next = (w + 1 < words) ? S.bits[r * words + w + 1] : 0u;
      uint32_t starts = m & ~((m << 1) | (prev >> 31));
      uint32_t ends = m & ~((m >> 1) | (next << 31));
      while (starts) {
        const int b = __ffs(starts) - 1;
        starts &= starts - 1;
        S.rcs[base + ns] = (short)(w * 32 + b);
        S.rrow[base + ns] = (short)r;
        ns++;
      }
      while (ends) {
        const int b = __ffs(ends) - 1;
        ends &= ends - 1;
        S.rce[base + ne] = (short)(w * 32 + b);
        ne++;
      }
      prev = m;
    }
  }
  for (int u = tid; u < nruns; u += blockDim.x) S.parent[u] = u;
  if (tid == 0) S.row_off[R] = nruns;
  __syncthreads();

  // 4-connectivity (R3): a run touches the runs of the previous row that share a column.
  for (int u = tid; u < nruns; u += blockDim.x) {
    const int r = S.rrow[u];
    if (r == 0) continue;
    const int cs = S.rcs[u], ce = S.rce[u];
    for (int v = S.row_off[r - 1]; v < S.row_off[r]; v++) {
      if (S.rcs[v] > ce) break;
      if (S.rce[v] >= cs) uf_unite(S.parent, u, v);
    }
  }
  __syncthreads();
  // parent := root; cid := is-root flag, then exclusive scan -> component ids
  // in order of first run (= first cell in a row-major scan).
  for (int u = tid; u < nruns; u += blockDim.x) S.cid[u] = uf_find(S.parent, u);
  __syncthreads();
  for (int u = tid; u < nruns; u += blockDim.x) S.parent[u] = S.cid[u];
  __syncthreads();
  for (int u = tid; u < nruns; u += blockDim.x) S.cid[u] = (S.parent[u] == u) ? 1 : 0;
  __syncthreads();
  const int ncomp = block_excl_scan_smem(S.cid, nruns, S.tmp);
  // a component's root is its first run in row-major order, so its top row
  // is the root's row (plain store); the other three sides are 16-bit
  // min / max updates (CAS on the 32-bit word holding the entry)
  for (int q = tid; q < ncomp; q += blockDim.x) {
    S.bc0[q] = SHRT_MAX;
    S.bc1[q] = -1;
    S.br1[q] = -1;
  }
  __syncthreads();
  for (int u = tid; u < nruns; u += blockDim.x) {
    const int root = S.parent[u];
    const int q = S.cid[root];
    if (root == u) S.br0[q] = S.rrow[u];
    atomic_minmax_s16<false>(&S.bc0[q], S.rcs[u]);
    atomic_minmax_s16<true>(&S.bc1[q], S.rce[u]);
    atomic_minmax_s16<true>(&S.br1[q], S.rrow[u]);
  }
  __syncthreads();
  for (int q = tid; q < ncomp; q += blockDim.x) {
    int px0, py0, bw, bh;
    extent(P, S.bc0[q], S.br0[q], S.bc1[q], S.br1[q], px0, py0, bw, bh);
    S.csz[q] = (unsigned char)smallest_size(P, bw, bh);
    S.memb[q] = 0;
  }
  if (tid < kMaxClasses) S.run[tid] = 0;
  __syncthreads();
  const long long* T = P.cost;
  int n = ncomp;
  bool again = n > 0;
  if (ncomp > kCoopMergeMin) {
    // many components: the CTA runs the greedy (same order rules) with block-wide
    // arg-mins; warp 0 then only places the final clusters
    n = coop_merge<FW>(P, S, ncomp, ext_cap);
    again = false;
  }
  if (wid != 0) return true;

  // ---- a3: greedy agglomerative merge, warp 0 ------------
  while (again) {
    again = false;
    int i = 0;
    while (i < n && n >= 2) {
      const int ic0 = S.bc0[i], ir0 = S.br0[i], ic1 = S.bc1[i], ir1 = S.br1[i];
      const int sx = ic0 + ic1, sy = ir0 + ir1;
      // (a) closest neighbour: squared distance of bbox centres (doubled cell
      //     units), ties -> smallest position (R5)
      unsigned long long best = ~0ull;
      for (int j = lane; j < n; j += 32) {
        if (j == i) continue;
        const int dx = sx - (S.bc0[j] + S.bc1[j]);
        const int dy = sy - (S.br0[j] + S.br1[j]);
        const unsigned long long key =
            ((unsigned long long)(unsigned)(dx * dx + dy * dy) << 32) | (unsigned)j;
        best = key < best ? key : best;
      }
      best = warp_min_u64(best);
      const int j = (int)(best & 0xffffffffu);
      // (b) proposed merge and its smallest containing size (R6)
      int m0 = min(ic0, S.bc0[j]), n0 = min(ir0, S.br0[j]);
      int m1 = max(ic1, S.bc1[j]), n1 = max(ir1, S.br1[j]);
      int px0, py0, bw, bh;
      extent(P, m0, n0, m1, n1, px0, py0, bw, bh);
      const int s = smallest_size(P, bw, bh);
      const int ws = P.sw[s], hs = P.sh[s];
      long long sum = T[S.csz[i]] + T[S.csz[j]];
      int before_i = (j < i) ? 1 : 0;
      if (lane == 0) {
        S.memb[i] = 1;
        S.memb[j] = 1;
      }
      // (c) absorb, k ascending, each fitting cluster immediately (R7): a
      //     ballot finds the first fitting k; earlier non-fitting ones can never
      //     fit later because the box only grows.
      int pos = 0;
      while (pos < n) {
        const int q = pos + lane;
        bool fit = false;
        if (q < n && q != i && q != j) {
          int a0 = min(m0, S.bc0[q]), a1 = min(n0, S.br0[q]);
          int a2 = max(m1, S.bc1[q]), a3 = max(n1, S.br1[q]);
          int qx, qy, qw, qh;
          extent(P, a0, a1, a2, a3, qx, qy, qw, qh);
          fit = (qw <= ws) && (qh <= hs);
        }
        const uint32_t msk = __ballot_sync(0xffffffffu, fit);
        if (msk) {
          const int qq = pos + __ffs(msk) - 1;
          m0 = min(m0, S.bc0[qq]);
          n0 = min(n0, S.br0[qq]);
          m1 = max(m1, S.bc1[qq]);
          n1 = max(n1, S.br1[qq]);
          sum += T[S.csz[qq]];
          before_i += (qq < i) ? 1 : 0;
          if (lane == 0) S.memb[qq] = 1;
          pos = qq + 1;
        } else {
          pos += 32;
        }
      }
      __syncwarp();
      // (d) accept iff strictly faster (R8); remove members, append merged (R4)
      if (T[s] < sum) {
        int wpos = 0;
        for (int base = 0; base < n; base += 32) {
          const int q = base + lane;
          bool keep = false;
          int v0 = 0, v1 = 0, v2 = 0, v3 = 0;
          unsigned char vs = 0;
          if (q < n) {
            keep = !S.memb[q];
            v0 = S.bc0[q]; v1 = S.br0[q]; v2 = S.bc1[q]; v3 = S.br1[q]; vs = S.csz[q];
          }
          const uint32_t km = __ballot_sync(0xffffffffu, keep);
          __syncwarp();
          if (keep) {
            const int d = wpos + __popc(km & lanemask_lt());
            S.bc0[d] = v0; S.br0[d] = v1; S.bc1[d] = v2; S.br1[d] = v3; S.csz[d] = vs;
          }
          if (q < n) S.memb[q] = 0;
          wpos += __popc(km);
          __syncwarp();
        }
        if (lane == 0) {
          S.bc0[wpos] = m0; S.br0[wpos] = n0; S.bc1[wpos] = m1; S.br1[wpos] = n1;
          S.csz[wpos] = (unsigned char)s;
        }
        __syncwarp();
        n = wpos + 1;
        i -= before_i;
        again = true;
      } else {
        for (int q = lane; q < n; q += 32) S.memb[q] = 0;
        __syncwarp();
        i++;
      }
    }
  }

  // ---- R11 fallback + a4 placement (R10) into per-frame scratch ----------
  long long est = 0;
  for (int q = lane; q < n; q += 32) est += T[S.csz[q]];
  est = warp_sum_i64(est);
  if (!ws_win) {   // estimate-only mode (window-size selection): est(R_t) after the R11 fallback
    if (lane == 0) *est_out = (n > 0 && est > T[P.full]) ? T[P.full] : est;
    return true;
  }
  int4* out = ws_win + (size_t)f * P.maxc;
  if (n > 0 && est > T[P.full]) {
    if (lane == 0) {
      out[0] = make_int4(0, 0, P.full, 0);
      ws_count[f] = 1;
      for (int kk = 0; kk < P.k; kk++) ws_cls[(size_t)f * P.k + kk] = (kk == P.full) ? 1 : 0;
    }
    return true;
  }
  for (int base = 0; base < n; base += 32) {
    const int q = base + lane;
    int s = -1, x = 0, y = 0;
    if (q < n) {
      s = S.csz[q];
      int px0, py0, bw, bh;
      extent(P, S.bc0[q], S.br0[q], S.bc1[q], S.br1[q], px0, py0, bw, bh);
      x = min(max(px0 - (P.sw[s] - bw) / 2, 0), P.W - P.sw[s]);
      y = min(max(py0 - (P.sh[s] - bh) / 2, 0), P.H - P.sh[s]);
    }
    int rank = 0;
    for (int kk = 0; kk < P.k; kk++) {
      const uint32_t mk = __ballot_sync(0xffffffffu, s == kk);
      if (s == kk) rank = S.run[kk] + __popc(mk & lanemask_lt());
      __syncwarp();
      if (lane == 0) S.run[kk] += __popc(mk);
      __syncwarp();
    }
    if (q < n) out[q] = make_int4(x, y, s, rank);
  }
  __syncwarp();
  if (lane == 0) ws_count[f] = n;
  for (int kk = lane; kk < P.k; kk += 32) ws_cls[(size_t)f * P.k + kk] = S.run[kk];
  return true;
}

__global__ void __launch_bounds__(kFastThreads) plan_fast_kernel(PlanArgs P, const float* __restrict__ scores,
                                                                  uint32_t* __restrict__ mask_out,
                                                                  int4* __restrict__ ws_win, int* __restrict__ ws_count,
                                                                  int* __restrict__ ws_cls, int* __restrict__ q_cnt,
                                                                  int* __restrict__ q_list) {
  plan_frame<false, kFwSmall>(P, blockIdx.x, min(kFastCap, P.maxc), scores, mask_out, ws_win, ws_count, ws_cls, q_cnt,
                          q_list);
}

// Persistent over the frames the fast tier queued (dense / checkerboard grids).
// Shared memory holds min(maxc, kMidCap) runs, so a CTA fits beside the
// persistent gather CTA of the previous batch on the same SM (the pipelined
// step runs plan(i+1) while gather(i) streams); frames with more runs are
// queued for plan_huge_kernel.
__global__ void __launch_bounds__(kPlanThreads) plan_full_kernel(PlanArgs P, const float* __restrict__ scores,
                                                                 uint32_t* __restrict__ mask_out,
                                                                 int4* __restrict__ ws_win, int* __restrict__ ws_count,
                                                                 int* __restrict__ ws_cls, const int* __restrict__ q_cnt,
                                                                 const int* __restrict__ q_list, int cap,
                                                                 int* __restrict__ q2_cnt, int* __restrict__ q2_list) {
  const int nq = *q_cnt;
  for (int qi = blockIdx.x; qi < nq; qi += gridDim.x) {
    plan_frame<false, kFwSmall>(P, q_list[qi], cap, scores, mask_out, ws_win, ws_count, ws_cls, q2_cnt, q2_list);
    __syncthreads();
  }
}

// Persistent over the frames with more than kMidCap runs (up to R*ceil(C/2)):
// the same plan with the run/component arrays in the CTA's global scratch
// slot (gbig + blockIdx.x * slot_bytes).
__global__ void __launch_bounds__(kPlanThreads) plan_huge_kernel(PlanArgs P, const float* __restrict__ scores,
                                                                 uint32_t* __restrict__ mask_out,
                                                                 int4* __restrict__ ws_win, int* __restrict__ ws_count,
                                                                 int* __restrict__ ws_cls, const int* __restrict__ q_cnt,
                                                                 const int* __restrict__ q_list,
                                                                 unsigned char* __restrict__ gbig, size_t slot_bytes) {
  const int nq = *q_cnt;
  unsigned char* slot = gbig + (size_t)blockIdx.x * slot_bytes;
  for (int qi = blockIdx.x; qi < nq; qi += gridDim.x) {
    plan_frame<true, kFwHuge>(P, q_list[qi], P.maxc, scores, mask_out, ws_win, ws_count, ws_cls, nullptr, nullptr, nullptr,
                     slot);
    __syncthreads();
  }
}

// kScanThreads (128, not 1024): a 1024-thread CTA needs ~32 K registers, more
// than a persistent gather CTA leaves of an SM, and would wait for the gather
// to end (so did 256 threads beside an f32 gather and its side CTAs).
__global__ void __launch_bounds__(kScanThreads, kScanMinBlocks) plan_scan_kernel(int F, int k, int* __restrict__ ws_count,
                                                         int* __restrict__ ws_cls, int* __restrict__ frame_off,
                                                         int* __restrict__ class_count, int max_windows,
                                                         int* __restrict__ d_status) {
  __shared__ int tmp[40];
  // frame CSR: copy counts then scan in place in frame_off
  for (int f = threadIdx.x; f < F; f += blockDim.x) frame_off[f] = ws_count[f];
  __syncthreads();
  const int total = block_scan_global(frame_off, F, 1, tmp);
  if (threadIdx.x == 0) {
    frame_off[F] = total;
    if (total > max_windows) set_status(d_status, MP_ERR_CAPACITY);
  }
  for (int kk = 0; kk < k; kk++) {
    const int tot = block_scan_global(ws_cls + kk, F, k, tmp);
    if (threadIdx.x == 0) class_count[kk] = tot;
  }
}

__global__ void __launch_bounds__(256) plan_scatter_kernel(PlanArgs P, int F, const int4* __restrict__ ws_win,
                                                           const int* __restrict__ ws_count,
                                                           const int* __restrict__ ws_cls,
                                                           const int* __restrict__ frame_off,
                                                           mp_window* __restrict__ windows, int max_windows) {
  const int f = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (f >= F) return;
  const int n = ws_count[f];
  const int base = frame_off[f];
  for (int q = lane; q < n; q += 32) {
    const int4 v = ws_win[(size_t)f * P.maxc + q];
    const int idx = base + q;
    if (idx >= max_windows) continue;
    mp_window w;
    w.frame = f;
    w.x = v.x;
    w.y = v.y;
    w.w = P.sw[v.z];
    w.h = P.sh[v.z];
    w.size_idx = v.z;
    w.slot = ws_cls[(size_t)f * P.k + v.z] + v.w;
    windows[idx] = w;
  }
}

// ------------------------------------------------------------------ NEXT-1 proxy sweep
constexpr int kSweepMaxJ = 64;
constexpr int kSweepThreads = 256;
struct SweepThr {
  float v[kSweepMaxJ];   // thresholds in ascending order
  int idx[kSweepMaxJ];   // their positions in the caller's list (output rows)
};

// One CTA per frame, single pass over the score grid: the
// frame's cells are read ONCE and ranked against the J ascending thresholds
// (rank = number of thresholds the score exceeds; NaN -> 0) into shared
// memory; the mask of threshold j is then {rank > j}.  For each threshold the
// frame is planned exactly as in mp_plan_windows (plan_frame, full capacity,
// a1 from the ranks), then the frame's detections are tested against its
// windows.  A threshold whose mask equals the previous one's (no cell has
// rank == j) has the same plan, so its totals are the previous ones (no
// re-plan).  Per-threshold totals are reduced in shared memory and added to
// the output with one int64 atomic per field per CTA.
__global__ void __launch_bounds__(kSweepThreads) proxy_sweep_kernel(PlanArgs P, const float* __restrict__ scores,
                                                                    SweepThr thr, int J,
                                                                    const float4* __restrict__ dets,
                                                                    const int* __restrict__ det_off,
                                                                    int4* __restrict__ ws_win, int* __restrict__ ws_count,
                                                                    int* __restrict__ ws_cls,
                                                                    unsigned long long* __restrict__ out) {
  __shared__ unsigned long long acc[5];
  __shared__ float s_thr[kSweepMaxJ];
  __shared__ int s_hist[kSweepMaxJ + 1];
  const int f = blockIdx.x, tid = threadIdx.x;
  if (tid < J) s_thr[tid] = thr.v[tid];
  if (tid <= J) s_hist[tid] = 0;
  if (tid < 5) acc[tid] = 0;
  __syncthreads();
  // the one pass over the frame's scores: per-cell threshold rank (binary
  // search over the ascending thresholds) + a histogram of the ranks
  const size_t plan_bytes = plan_smem_bytes(P.R, P.words, P.maxc, nullptr, nullptr);
  unsigned char* rk = smem_raw + plan_bytes;
  const int RC = P.R * P.C;
  const float* sc = scores + (size_t)f * RC;
  for (int c = tid; c < RC; c += blockDim.x) {
    const float v = __ldg(sc + c);
    int lo = 0, hi = J;   // number of thresholds t with v > t (NaN: none)
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (v > s_thr[mid]) lo = mid + 1;
      else hi = mid;
    }
    rk[c] = (unsigned char)lo;
    atomicAdd(&s_hist[lo], 1);
  }
  __syncthreads();
  const int d_lo = det_off[f], d_hi = det_off[f + 1];
  for (int j = 0; j < J; j++) {
    // mask(j) = {rank > j}; it differs from mask(j-1) iff some cell has rank j
    const bool same = j > 0 && s_hist[j] == 0;
    if (same) {   // identical plan: the previous threshold's totals (still in acc)
      if (tid < 5 && acc[tid]) atomicAdd(&out[5 * thr.idx[j] + tid], acc[tid]);
      continue;
    }
    __syncthreads();   // (acc read by the previous threshold's atomics above)
    if (tid < 5) acc[tid] = 0;
    __syncthreads();
    plan_frame(P, f, P.maxc, scores, nullptr, ws_win, ws_count, ws_cls, nullptr, nullptr, nullptr, nullptr, rk, j);
    __syncthreads();   // warp 0's scratch writes are visible to the CTA
    const int n = ws_count[f];
    const int4* wl = ws_win + (size_t)f * P.maxc;
    unsigned long long cost = 0, cov = 0, touch = 0;
    for (int q = tid; q < n; q += blockDim.x) cost += (unsigned long long)P.cost[wl[q].z];
    for (int d = d_lo + tid; d < d_hi; d += blockDim.x) {
      const float4 b = dets[d];
      bool in = false, ov = false;
      for (int q = 0; q < n; q++) {
        const int4 w = wl[q];
        const float x0 = (float)w.x, y0 = (float)w.y;
        const float x1 = (float)(w.x + P.sw[w.z]), y1 = (float)(w.y + P.sh[w.z]);
        in |= (b.x >= x0) && (b.z <= x1) && (b.y >= y0) && (b.w <= y1);
        ov |= (b.x < x1) && (b.z > x0) && (b.y < y1) && (b.w > y0);
      }
      cov += in ? 1 : 0;
      touch += ov ? 1 : 0;
    }
    if (cost) atomicAdd(&acc[0], cost);
    if (cov) atomicAdd(&acc[3], cov);
    if (touch) atomicAdd(&acc[4], touch);
    if (tid == 0) {
      acc[1] = n;
      acc[2] = (n == 1 && wl[0].z == P.full) ? 1 : 0;
    }
    __syncthreads();
    if (tid < 5 && acc[tid]) atomicAdd(&out[5 * thr.idx[j] + tid], acc[tid]);
    __syncthreads();   // scratch is reused by the next threshold (acc is kept for an identical next mask)
  }
}

// ------------------------------------------------------------------ NEXT-2 window-size selection
constexpr int kSelThreads = 128;
constexpr int kSelCandPerBlock = 16;

// R13/R14 for S + {candidate}: 1 <= w <= W, 1 <= h <= H, distinct from every
// size of S, T > 0, and strictly monotone in area against every size of S.
__device__ __forceinline__ bool cand_valid(const PlanArgs& P, int w, int h, long long t) {
  if (w < 1 || h < 1 || w > P.W || h > P.H || t <= 0) return false;
  const long long ac = (long long)w * h;
  for (int q = 0; q < P.k; q++) {
    if (P.sw[q] == w && P.sh[q] == h) return false;
    const long long aq = (long long)P.sw[q] * P.sh[q];
    if (aq < ac && !(P.cost[q] < t)) return false;
    if (ac < aq && !(t < P.cost[q])) return false;
  }
  return true;
}

// tot[c] = 0 for valid candidates, INT64_MAX (never the arg-min) and
// *d_status = MP_ERR_INVALID for invalid ones.
__global__ void window_set_init_kernel(PlanArgs P, const mp_size* __restrict__ cand,
                                       const long long* __restrict__ cand_cost, int n_cand,
                                       long long* __restrict__ tot, int* __restrict__ d_status) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n_cand; c += gridDim.x * blockDim.x) {
    const mp_size cd = cand[c];
    const bool ok = cand_valid(P, cd.w, cd.h, cand_cost[c]);
    tot[c] = ok ? 0 : 0x7fffffffffffffffLL;
    if (!ok) set_status(d_status, MP_ERR_INVALID);
  }
}

// grid (F, ceil(n_cand / kSelCandPerBlock)): the CTA plans frame f once per
// candidate size, with S' = S + {candidate} (order re-derived by (area, w, h)),
// in estimate-only mode, and adds est(R(I_f; S')) to tot[c].
__global__ void __launch_bounds__(kSelThreads) window_set_cost_kernel(PlanArgs P, const float* __restrict__ scores,
                                                                      const mp_size* __restrict__ cand,
                                                                      const long long* __restrict__ cand_cost,
                                                                      int n_cand,
                                                                      unsigned long long* __restrict__ tot) {
  __shared__ long long s_est;
  const int f = blockIdx.x;
  const int c0 = blockIdx.y * kSelCandPerBlock, c1 = min(n_cand, c0 + kSelCandPerBlock);
  for (int c = c0; c < c1; c++) {
    const mp_size cd = cand[c];
    const long long ct = cand_cost[c];
    if (!cand_valid(P, cd.w, cd.h, ct)) continue;   // (uniform across the CTA)
    PlanArgs Q = P;
    const int kk = P.k;
    Q.sw[kk] = cd.w;
    Q.sh[kk] = cd.h;
    Q.cost[kk] = ct;
    Q.k = kk + 1;
    // insert the candidate into the (area, w, h) order
    const long long ac = (long long)cd.w * cd.h;
    int pos = kk;
    for (int q = 0; q < kk; q++) {
      const int i = P.order[q];
      const long long ai = (long long)P.sw[i] * P.sh[i];
      if (ac < ai || (ac == ai && (cd.w < P.sw[i] || (cd.w == P.sw[i] && cd.h < P.sh[i])))) {
        pos = q;
        break;
      }
    }
    for (int q = kk; q > pos; q--) Q.order[q] = P.order[q - 1];
    Q.order[pos] = kk;
    plan_frame(Q, f, P.maxc, scores, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, &s_est);
    __syncthreads();
    if (threadIdx.x == 0 && s_est) atomicAdd(&tot[c], (unsigned long long)s_est);
    __syncthreads();
  }
}

// ------------------------------------------------------------------ host side
static bool build_plan_args(const mp_plan_params* p, PlanArgs* A, mp_status* err) {
  *err = MP_ERR_INVALID;
  if (!p || !p->sizes || !p->cost) return false;
  if (p->W < 1 || p->H < 1 || p->W > 16384 || p->H > 16384) return false;
  if (p->cell_w < 1 || p->cell_h < 1 || p->k < 1 || p->k > kMaxClasses) return false;
  if (!(p->b_proxy == p->b_proxy)) return false;   // NaN threshold
  int full = -1;
  for (int i = 0; i < p->k; i++) {
    const mp_size s = p->sizes[i];
    if (s.w < 1 || s.h < 1 || s.w > p->W || s.h > p->H || p->cost[i] <= 0) return false;
    if (s.w == p->W && s.h == p->H) full = i;
    for (int j = 0; j < p->k; j++) {
      if (j == i) continue;
      if (p->sizes[j].w == s.w && p->sizes[j].h == s.h) return false;
      const long long ai = (long long)s.w * s.h, aj = (long long)p->sizes[j].w * p->sizes[j].h;
      if (ai < aj && !(p->cost[i] < p->cost[j])) return false;
    }
  }
  if (full < 0) return false;   // the full frame is always in S (R14)
  A->W = p->W;
  A->H = p->H;
  A->cw = p->cell_w;
  A->ch = p->cell_h;
  A->R = (p->H + p->cell_h - 1) / p->cell_h;
  A->C = (p->W + p->cell_w - 1) / p->cell_w;
  A->words = (A->C + 31) / 32;
  A->k = p->k;
  A->full = full;
  A->b = p->b_proxy;
  // (W, H <= 16384: cell rows / columns fit the planner's int16 runs and boxes)
  if ((long long)A->R * A->C > kMaxCells) {
    *err = MP_ERR_UNSUPPORTED;
    return false;
  }
  A->maxc = A->R * ((A->C + 1) / 2);
  for (int i = 0; i < kMaxClasses; i++) {
    A->order[i] = i;
    A->sw[i] = i < p->k ? p->sizes[i].w : 0;
    A->sh[i] = i < p->k ? p->sizes[i].h : 0;
    A->cost[i] = i < p->k ? p->cost[i] : 0;
  }
  // insertion sort of size indices by (area, w, h)
  for (int a = 1; a < p->k; a++) {
    int v = A->order[a], b = a - 1;
    auto less = [&](int x, int y) {
      long long ax = (long long)A->sw[x] * A->sh[x], ay = (long long)A->sw[y] * A->sh[y];
      if (ax != ay) return ax < ay;
      if (A->sw[x] != A->sw[y]) return A->sw[x] < A->sw[y];
      return A->sh[x] < A->sh[y];
    };
    while (b >= 0 && less(v, A->order[b])) {
      A->order[b + 1] = A->order[b];
      b--;
    }
    A->order[b + 1] = v;
  }
  *err = MP_OK;
  return true;
}

struct PlanWs {
  size_t win_off, count_off, cls_off, q_off, big_off, slot_bytes, total;
};

static int plan_sms() {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) !=
                                                 cudaSuccess || sms < 1) {
    (void)cudaGetLastError();
    return 148;
  }
  return sms;
}

// Global scratch slots of the full tier (one per plan_full CTA) exist only
// when the grid's worst case (maxc runs) exceeds the shared-memory capacity.
static PlanWs plan_ws_layout(const PlanArgs& A, int F) {
  PlanWs L;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  L.win_off = 0;
  L.count_off = al(L.win_off + sizeof(int4) * (size_t)F * A.maxc);
  L.cls_off = al(L.count_off + sizeof(int) * (size_t)F);
  // [0] full-tier queue count, [1] huge-tier queue count, [2..F+1] full-tier
  // frames, [F+2..2F+1] huge-tier frames
  L.q_off = al(L.cls_off + sizeof(int) * (size_t)F * A.k);
  L.big_off = al(L.q_off + sizeof(int) * (size_t)(2 * F + 2));
  L.slot_bytes = A.maxc > kMidCap ? al(plan_smem_bytes(A.R, A.words, A.maxc, nullptr, nullptr)) : 0;
  const size_t slots = (F > 0 && L.slot_bytes) ? (size_t)plan_sms() * kHugeGrid : 0;
  L.total = al(L.big_off + slots * L.slot_bytes) + 256;
  return L;
}

}  // namespace mpk

using namespace mpk;

extern "C" size_t mp_plan_workspace_size(const mp_plan_params* p, int32_t F) {
  PlanArgs A;
  mp_status err;
  if (F < 0 || !build_plan_args(p, &A, &err)) return 0;
  return plan_ws_layout(A, F).total;
}

extern "C" mp_status mp_plan_windows(const mp_plan_params* p, const float* d_scores, int32_t F,
                                     uint32_t* d_mask, mp_window* d_windows, int32_t max_windows,
                                     int32_t* d_frame_off, int32_t* d_class_count, int32_t* d_status,
                                     void* d_ws, size_t ws_bytes, void* stream) {
  PlanArgs A;
  mp_status err;
  if (!build_plan_args(p, &A, &err)) return err;
  if (F < 0 || max_windows < 0 || !d_frame_off || !d_class_count || !d_status) return MP_ERR_INVALID;
  if (F > 0 && !d_scores) return MP_ERR_INVALID;
  if (max_windows > 0 && !d_windows) return MP_ERR_INVALID;
  const PlanWs L = plan_ws_layout(A, F);
  if (ws_bytes < L.total || (!d_ws && L.total > 0)) return MP_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  unsigned char* ws = (unsigned char*)d_ws;
  int4* ws_win = (int4*)(ws + L.win_off);
  int* ws_count = (int*)(ws + L.count_off);
  int* ws_cls = (int*)(ws + L.cls_off);
  int* q_cnt = (int*)(ws + L.q_off);
  int* q2_cnt = q_cnt + 1;
  int* q_list = q_cnt + 2;
  int* q2_list = q_list + F;
  if (F > 0) {
    const int cap_full = A.maxc < kMidCap ? A.maxc : kMidCap;
    const size_t smem = plan_smem_bytes(A.R, A.words, cap_full, nullptr, nullptr);
    if (smem > 227 * 1024) return MP_ERR_UNSUPPORTED;
    const size_t smem_fast = plan_smem_bytes(A.R, A.words, kFastCap < A.maxc ? kFastCap : A.maxc, nullptr, nullptr);
    if (smem_fast > 227 * 1024 || plan_smem_bytes(A.R, A.words, 0, nullptr, nullptr) > 227 * 1024)
      return MP_ERR_UNSUPPORTED;   // (the bit rows of very tall grids)
    MP_CUDA_TRY(cudaMemsetAsync(q_cnt, 0, 2 * sizeof(int), s));
    for (const void* k : {(const void*)plan_fast_kernel, (const void*)plan_full_kernel,
                          (const void*)plan_huge_kernel, (const void*)plan_scan_kernel,
                          (const void*)plan_scatter_kernel})
      MP_CUDA_TRY(prefer_max_shared(k));
    MP_CUDA_TRY(cudaFuncSetAttribute(plan_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem_fast));
    MP_CUDA_TRY(cudaFuncSetAttribute(plan_full_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    PlanArgs Af = A;   // the fast tier lays out shared memory for min(kFastCap, maxc) runs
    plan_fast_kernel<<<F, kFastThreads, smem_fast, s>>>(Af, d_scores, d_mask, ws_win, ws_count, ws_cls, q_cnt,
                                                         q_list);
    MP_CUDA_TRY(cudaGetLastError());
    plan_full_kernel<<<plan_sms() * kFullGrid, kPlanThreads, smem, s>>>(
        A, d_scores, d_mask, ws_win, ws_count, ws_cls, q_cnt, q_list, cap_full, q2_cnt, q2_list);
    MP_CUDA_TRY(cudaGetLastError());
    if (L.slot_bytes) {   // grids whose worst case exceeds the shared-memory tiers
      const size_t smem_huge = plan_smem_bytes(A.R, A.words, 0, nullptr, nullptr);
      // one CTA per global scratch slot the caller's workspace holds (the
      // workspace may have been sized on a device with fewer SMs)
      const size_t slots = (ws_bytes - L.big_off) / L.slot_bytes;
      const int grid = (int)(slots < (size_t)plan_sms() * kHugeGrid ? slots : (size_t)plan_sms() * kHugeGrid);
      if (grid < 1) return MP_ERR_INVALID;
      plan_huge_kernel<<<grid, kPlanThreads, smem_huge, s>>>(
          A, d_scores, d_mask, ws_win, ws_count, ws_cls, q2_cnt, q2_list, ws + L.big_off, L.slot_bytes);
      MP_CUDA_TRY(cudaGetLastError());
    }
  }
  plan_scan_kernel<<<1, kScanThreads, 0, s>>>(F, A.k, ws_count, ws_cls, d_frame_off, d_class_count, max_windows,
                                      d_status);
  MP_CUDA_TRY(cudaGetLastError());
  if (F > 0) {
    plan_scatter_kernel<<<(F + 7) / 8, 256, 0, s>>>(A, F, ws_win, ws_count, ws_cls, d_frame_off, d_windows,
                                                    max_windows);
    MP_CUDA_TRY(cudaGetLastError());
  }
  return MP_OK;
}

#ifdef MP_PLAN_PROF
extern "C" int mp_debug_plan_prof(unsigned long long* out4, int reset) {
  if (cudaMemcpyFromSymbol(out4, g_plan_prof, sizeof(g_plan_prof)) != cudaSuccess) return -1;
  if (reset) {
    unsigned long long z[4] = {0, 0, 0, 0};
    if (cudaMemcpyToSymbol(g_plan_prof, z, sizeof(z)) != cudaSuccess) return -1;
  }
  return 0;
}
#endif

extern "C" size_t mp_proxy_sweep_workspace_size(const mp_plan_params* p, int32_t F) {
  return mp_plan_workspace_size(p, F);
}

extern "C" mp_status mp_proxy_sweep(const mp_plan_params* p, const float* d_scores, int32_t F,
                                    const float* thresholds, int32_t J, const float* d_dets,
                                    const int32_t* d_det_off, mp_sweep_result* d_out, void* d_ws, size_t ws_bytes,
                                    void* stream) {
  PlanArgs A;
  mp_status err;
  if (!build_plan_args(p, &A, &err)) return err;
  if (F < 0 || J < 1 || J > kSweepMaxJ || !thresholds || !d_out || !d_det_off) return MP_ERR_INVALID;
  if (F > 0 && (!d_scores || !d_dets)) return MP_ERR_INVALID;
  for (int j = 0; j < J; j++)
    if (!(thresholds[j] == thresholds[j])) return MP_ERR_INVALID;
  const PlanWs L = plan_ws_layout(A, F);
  if (ws_bytes < L.total || !d_ws) return MP_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  unsigned char* ws = (unsigned char*)d_ws;
  int4* ws_win = (int4*)(ws + L.win_off);
  int* ws_count = (int*)(ws + L.count_off);
  int* ws_cls = (int*)(ws + L.cls_off);
  // thresholds travel in the (graph-capturable) kernel parameter block,
  // sorted ascending (stable: equal thresholds keep their order) with their
  // output rows
  SweepThr th;
  for (int j = 0; j < kSweepMaxJ; j++) {
    th.v[j] = j < J ? thresholds[j] : 0.0f;
    th.idx[j] = j;
  }
  for (int a = 1; a < J; a++) {
    const float v = th.v[a];
    const int ix = th.idx[a];
    int b = a - 1;
    while (b >= 0 && th.v[b] > v) {
      th.v[b + 1] = th.v[b];
      th.idx[b + 1] = th.idx[b];
      b--;
    }
    th.v[b + 1] = v;
    th.idx[b + 1] = ix;
  }
  MP_CUDA_TRY(cudaMemsetAsync(d_out, 0, sizeof(mp_sweep_result) * (size_t)J, s));
  if (F == 0) return MP_OK;
  // planner layout + one rank byte per cell
  const size_t smem = plan_smem_bytes(A.R, A.words, A.maxc, nullptr, nullptr) + (size_t)A.R * A.C;
  if (smem > 227 * 1024) return MP_ERR_UNSUPPORTED;
  MP_CUDA_TRY(cudaFuncSetAttribute(proxy_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  proxy_sweep_kernel<<<F, kSweepThreads, smem, s>>>(A, d_scores, th, J, (const float4*)d_dets, d_det_off, ws_win,
                                                    ws_count, ws_cls, (unsigned long long*)d_out);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" mp_status mp_window_set_cost(const mp_plan_params* p, const float* d_scores, int32_t F,
                                        const mp_size* d_cand, const int64_t* d_cand_cost, int32_t n_cand,
                                        int64_t* d_tot, int32_t* d_status, void* stream) {
  PlanArgs A;
  mp_status err;
  if (!build_plan_args(p, &A, &err)) return err;
  if (A.k >= kMaxClasses) return MP_ERR_UNSUPPORTED;
  if (F < 0 || n_cand < 0 || (n_cand > 0 && (!d_cand || !d_cand_cost || !d_tot || !d_status))) return MP_ERR_INVALID;
  if (F > 0 && !d_scores) return MP_ERR_INVALID;
  if (n_cand == 0) return MP_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t smem = plan_smem_bytes(A.R, A.words, A.maxc, nullptr, nullptr);
  if (smem > 227 * 1024) return MP_ERR_UNSUPPORTED;
  // candidates are validated on the device (R13/R14 against S): no host copy,
  // no synchronisation, graph-capturable
  window_set_init_kernel<<<(n_cand + 255) / 256, 256, 0, s>>>(A, d_cand, (const long long*)d_cand_cost, n_cand,
                                                               (long long*)d_tot, d_status);
  MP_CUDA_TRY(cudaGetLastError());
  if (F == 0) return MP_OK;
  MP_CUDA_TRY(cudaFuncSetAttribute(window_set_cost_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid(F, (n_cand + kSelCandPerBlock - 1) / kSelCandPerBlock);
  window_set_cost_kernel<<<grid, kSelThreads, smem, s>>>(A, d_scores, d_cand, (const long long*)d_cand_cost, n_cand,
                                                         (unsigned long long*)d_tot);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}
