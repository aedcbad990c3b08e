"""Seeded synthetic workload generator (shared by tests and bench; holds none
of the method's arithmetic).

It produces, for a configuration and a clip id:
  * RGB24 frames from a counter-based generator (splitmix64 stream per frame)
    that gives identical bytes in numpy (host) and torch (any device) — so the
    GPU bench can synthesise its frames in HBM while the oracle regenerates any
    sampled frame on the host;
  * traffic-camera-shaped scenes: 3-4 lanes (polylines crossing the frame),
    Poisson spawns, speed 2-8 px/frame x W/1920, size U[smin,smax] times the
    perspective factor (0.4 + 0.6 y/H), aspect h/w U[0.6,1.0], 3 classes;
  * proxy score grids: label = the cell overlaps an object with positive area
    (the proxy's training label of PAPER.md:165); score =
    sigmoid(z), z ~ N(+2,1) if labelled else N(neg_mu,1);
  * stand-in detector outputs for a given window list: per window, each object
    with >= 25% of its area inside emits jittered copies of (object ∩ window)
    in window-local detector-input pixels, plus Poisson false positives.
Seeds: master 210314695; clip seed = splitmix64(master ^ clip); frame seed =
splitmix64(clip seed ^ frame).
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Sequence, Tuple

import numpy as np

MASTER_SEED = 210314695
_M64 = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15
_MIX1 = 0xBF58476D1CE4E5B9
_MIX2 = 0x94D049BB133111EB


def splitmix64(x: int) -> int:
    """One splitmix64 output for integer state x (pure Python ints)."""
    z = (x + _GAMMA) & _M64
    z = ((z ^ (z >> 30)) * _MIX1) & _M64
    z = ((z ^ (z >> 27)) * _MIX2) & _M64
    return z ^ (z >> 31)


def clip_seed(clip: int) -> int:
    return splitmix64(MASTER_SEED ^ clip)


def frame_seed(clip: int, frame: int) -> int:
    return splitmix64(clip_seed(clip) ^ frame)


# --------------------------------------------------------------------------- configs
@dataclasses.dataclass(frozen=True)
class Config:
    """One synthetic workload (BASELINE.json configs)."""
    name: str
    W: int
    H: int
    sizes: Tuple[Tuple[int, int], ...]          # S, full frame last
    frames: int                                 # frames per clip
    obj_range: Tuple[int, int]                  # target objects per frame (clip mean drawn U[lo,hi])
    size_range: Tuple[int, int]                 # object size px before perspective
    lanes: Tuple[int, int] = (3, 4)
    neg_mu: float = -3.0
    cell: int = 32
    scale: float = 0.75                         # detector-input scale s (R15)
    copies: str = "poisson"                     # "poisson": 1+Poisson(1); "bernoulli": 1+Bern(.5)
    fp_rate: float = 0.3                        # false positives per window (Poisson mean)
    clips: int = 1
    b_proxy: float = 0.5
    score_thr: float = 0.25
    iou_thr: float = 0.5

    @property
    def grid(self) -> Tuple[int, int]:
        return (-(-self.H // self.cell), -(-self.W // self.cell))   # (R, C)

    @property
    def cost(self) -> Tuple[int, ...]:
        """T_k = ceil(w/32)*ceil(h/32) + 16 (cell units + per-window overhead)."""
        return tuple(-(-w // 32) * -(-h // 32) + 16 for (w, h) in self.sizes)

    @property
    def out_dims(self) -> Tuple[Tuple[int, int], ...]:
        return tuple((max(1, int(math.floor(self.scale * w + 0.5))),
                      max(1, int(math.floor(self.scale * h + 0.5)))) for (w, h) in self.sizes)

    @property
    def pitch(self) -> int:
        return (3 * self.W + 15) // 16 * 16

    @property
    def proxy_dims(self) -> Tuple[int, int]:
        """Proxy-model input resolution for NEXT-3's full-frame downscale:
        416x256, the larger of P:167's two examples (13x8 output grid)."""
        return (416, 256)

    @property
    def pitch_nv12(self) -> int:
        """NV12 row pitch (bytes, both planes): W rounded up to 16."""
        return (self.W + 15) // 16 * 16


CONFIGS = {
    # BASELINE.json configs[0]: 960x540, 30 frames, one 256x256 window size, <=20 boxes/frame
    "c1_540p": Config("c1_540p", 960, 540, ((256, 256), (960, 540)), 30, (5, 10), (30, 110),
                      copies="bernoulli", fp_rate=0.0),
    # configs[1]: 1080p traffic clip, 1800 frames, sparse, window sizes 256 and 512
    "c2_1080p_sparse": Config("c2_1080p_sparse", 1920, 1080,
                              ((256, 256), (512, 512), (1920, 1080)), 1800, (3, 15), (40, 160)),
    # configs[2]: 1080p dense (>=100 boxes/frame)
    "c3_1080p_dense": Config("c3_1080p_dense", 1920, 1080,
                             ((256, 256), (512, 512), (1920, 1080)), 1800, (100, 150), (30, 90),
                             lanes=(6, 8)),
    # configs[3]: 4K drone view, small objects, three window sizes, high positive fraction
    "c4_4k_drone": Config("c4_4k_drone", 3840, 2160,
                          ((128, 128), (256, 256), (512, 512), (3840, 2160)), 300, (300, 600),
                          (12, 48), lanes=(16, 24), neg_mu=-1.5),
    # configs[4]: 1000 x 1080p clips, threshold sweep (density mixed by clip)
    "c5_1080p_clips": Config("c5_1080p_clips", 1920, 1080,
                             ((256, 256), (512, 512), (1920, 1080)), 1800, (3, 60), (30, 160),
                             clips=1000),
}
B_SWEEP = tuple(round(0.1 * i, 1) for i in range(1, 10))


# --------------------------------------------------------------------------- pixels
def frame_words(H: int, pitch: int) -> int:
    return -(-(H * pitch) // 8)


def frame_pixels_np(seed: int, H: int, pitch: int) -> np.ndarray:
    """uint8 [H][pitch]: byte i = byte (i%8) (little-endian) of the
    (i//8)-th splitmix64 output of the stream started at `seed`."""
    n = frame_words(H, pitch)
    with np.errstate(over="ignore"):
        z = (np.uint64(seed) + (np.arange(1, n + 1, dtype=np.uint64) * np.uint64(_GAMMA)))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_MIX1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_MIX2)
        z = z ^ (z >> np.uint64(31))
    return z.view(np.uint8)[: H * pitch].reshape(H, pitch)


def frame_nv12_np(seed: int, H: int, pitch: int) -> np.ndarray:
    """NV12 frame uint8 [H*3/2][pitch] (rows 0..H-1 = Y plane, rows H.. =
    interleaved U,V): the same splitmix64 byte stream as frame_pixels_np over
    H*3/2 rows, i.e. Y, U and V uniform over 0..255 (values outside the
    limited range exercise the clamp)."""
    return frame_pixels_np(seed, H + H // 2, pitch)


def _s64(x: int) -> int:
    x &= _M64
    return x - (1 << 64) if x >= (1 << 63) else x


def frame_pixels_torch(seeds: Sequence[int], H: int, pitch: int, device="cpu", out=None):
    """Same bytes as frame_pixels_np for each seed, computed with torch int64
    (two's-complement wrap-around) on `device`.  Returns uint8 [n][H][pitch]
    (written into `out` if given)."""
    import torch
    n = frame_words(H, pitch)
    nf = len(seeds)
    if out is None:
        out = torch.empty((nf, H, pitch), dtype=torch.uint8, device=device)
    idx = torch.arange(1, n + 1, dtype=torch.int64, device=device) * _s64(_GAMMA)
    chunk = max(1, (1 << 27) // n)
    m1, m2 = _s64(_MIX1), _s64(_MIX2)

    def lsr(z, s):   # logical shift right on int64
        return (z >> s) & ((1 << (64 - s)) - 1)

    for a in range(0, nf, chunk):
        b = min(nf, a + chunk)
        sd = torch.tensor([_s64(s) for s in seeds[a:b]], dtype=torch.int64, device=device)
        z = sd[:, None] + idx[None, :]
        z = (z ^ lsr(z, 30)) * m1
        z = (z ^ lsr(z, 27)) * m2
        z = z ^ lsr(z, 31)
        by = z.view(torch.uint8).reshape(b - a, n * 8)[:, : H * pitch]
        out[a:b].copy_(by.reshape(b - a, H, pitch))
        del z, by
    return out


# --------------------------------------------------------------------------- scenes
@dataclasses.dataclass
class Scene:
    """Objects of one clip: per-frame boxes (x1,y1,x2,y2) frame px, cls, id."""
    boxes: List[np.ndarray]      # [F] float64 (n,4)
    cls: List[np.ndarray]        # [F] int32 (n,)
    ids: List[np.ndarray]        # [F] int64 (n,)


def _lane(rng, W, H):
    """A polyline crossing the frame: entry on one border, exit on the opposite
    border, one jittered midpoint."""
    if rng.random() < 0.5:   # left -> right
        p0 = (0.0, rng.uniform(0.1, 0.9) * H)
        p2 = (float(W), rng.uniform(0.1, 0.9) * H)
    else:                    # top -> bottom
        p0 = (rng.uniform(0.1, 0.9) * W, 0.0)
        p2 = (rng.uniform(0.1, 0.9) * W, float(H))
    if rng.random() < 0.5:
        p0, p2 = p2, p0
    mid = ((p0[0] + p2[0]) / 2 + rng.normal(0, 0.08 * W), (p0[1] + p2[1]) / 2 + rng.normal(0, 0.08 * H))
    pts = np.array([p0, mid, p2], dtype=np.float64)
    seg = np.linalg.norm(np.diff(pts, axis=0), axis=1)
    return pts, np.concatenate([[0.0], np.cumsum(seg)])


def clip_cost_estimate(cfg: Config, clip: int) -> float:
    """A clip's expected objects per frame (the density `make_scene` draws
    first from the clip seed) — a cheap per-clip cost estimate for
    longest-processing-time sharding, without generating the clip."""
    rng = np.random.default_rng(clip_seed(clip))
    rng.integers(cfg.lanes[0], cfg.lanes[1] + 1)
    return float(rng.uniform(*cfg.obj_range))


def make_scene(cfg: Config, clip: int, n_frames: Optional[int] = None, frame0: int = 0) -> Scene:
    """Objects for frames [frame0, frame0+n_frames) of a clip."""
    F = cfg.frames if n_frames is None else n_frames
    rng = np.random.default_rng(clip_seed(clip))
    n_lanes = int(rng.integers(cfg.lanes[0], cfg.lanes[1] + 1))
    target = rng.uniform(*cfg.obj_range)
    vscale = cfg.W / 1920.0
    lanes = [_lane(rng, cfg.W, cfg.H) for _ in range(n_lanes)]
    mean_speed = 5.0 * vscale
    boxes = [[] for _ in range(F)]
    cls = [[] for _ in range(F)]
    ids = [[] for _ in range(F)]
    oid = 0
    t_end = frame0 + F
    for li, (pts, arc) in enumerate(lanes):
        L = arc[-1]
        life = L / mean_speed
        rate = target / (n_lanes * life)               # spawns per frame on this lane
        lrng = np.random.default_rng(splitmix64(clip_seed(clip) ^ (0x1000 + li)))
        t = -2.0 * life * 2.0                          # warm start
        while True:
            t += lrng.exponential(1.0 / rate)
            if t >= t_end:
                break
            speed = lrng.uniform(2.0, 8.0) * vscale
            size = lrng.uniform(*cfg.size_range)
            aspect = lrng.uniform(0.6, 1.0)
            c = int(lrng.integers(0, 3))
            my_id = oid
            oid += 1
            fa = max(frame0, int(math.ceil(t)))
            fb = min(t_end - 1, int(math.floor(t + L / speed)))
            if fb < fa:
                continue
            fr = np.arange(fa, fb + 1)
            d = speed * (fr - t)
            cx = np.interp(d, arc, pts[:, 0])
            cy = np.interp(d, arc, pts[:, 1])
            w = size * (0.4 + 0.6 * cy / cfg.H)
            h = w * aspect
            x1 = np.clip(cx - w / 2, 0, cfg.W)
            x2 = np.clip(cx + w / 2, 0, cfg.W)
            y1 = np.clip(cy - h / 2, 0, cfg.H)
            y2 = np.clip(cy + h / 2, 0, cfg.H)
            for q, f in enumerate(fr):
                if x2[q] - x1[q] >= 1.0 and y2[q] - y1[q] >= 1.0:
                    boxes[f - frame0].append((x1[q], y1[q], x2[q], y2[q]))
                    cls[f - frame0].append(c)
                    ids[f - frame0].append(my_id)
    return Scene([np.asarray(b, np.float64).reshape(-1, 4) for b in boxes],
                 [np.asarray(c, np.int32) for c in cls],
                 [np.asarray(i, np.int64) for i in ids])


def cell_labels(cfg: Config, boxes: np.ndarray) -> np.ndarray:
    """uint8 [R][C]: 1 iff the cell's pixel region overlaps some box with
    positive area (SPEC.md:72-89 strict positive-area rule)."""
    R, Cc = cfg.grid
    lab = np.zeros((R, Cc), np.uint8)
    cw = cfg.cell
    for x1, y1, x2, y2 in boxes:
        c_lo, c_hi = int(math.floor(x1 / cw)), int(math.ceil(x2 / cw)) - 1
        r_lo, r_hi = int(math.floor(y1 / cw)), int(math.ceil(y2 / cw)) - 1
        c_lo, r_lo = max(c_lo, 0), max(r_lo, 0)
        c_hi, r_hi = min(c_hi, Cc - 1), min(r_hi, R - 1)
        if c_hi >= c_lo and r_hi >= r_lo:
            lab[r_lo:r_hi + 1, c_lo:c_hi + 1] = 1
    return lab


def score_grids(cfg: Config, clip: int, scene: Scene, frame0: int = 0) -> np.ndarray:
    """float32 [F][R][C] proxy scores for the scene's frames."""
    F = len(scene.boxes)
    R, Cc = cfg.grid
    out = np.empty((F, R, Cc), np.float32)
    for i in range(F):
        lab = cell_labels(cfg, scene.boxes[i])
        rng = np.random.default_rng(frame_seed(clip, frame0 + i))
        z = np.where(lab == 1, rng.normal(2.0, 1.0, (R, Cc)), rng.normal(cfg.neg_mu, 1.0, (R, Cc)))
        out[i] = (1.0 / (1.0 + np.exp(-z))).astype(np.float32)
    return out


BOX_DTYPE = np.dtype([("x1", "<f4"), ("y1", "<f4"), ("x2", "<f4"), ("y2", "<f4"),
                      ("score", "<f4"), ("cls", "<i4")])


def standin_boxes(cfg: Config, clip: int, scene: Scene, windows: np.ndarray,
                  frame0: int = 0, extra_edge_cases: bool = False):
    """Stand-in detector output for a window list (int32 [n][7] = frame, x, y,
    w, h, size_idx, slot; frame index relative to the scene's first frame).
    Returns (boxes BOX_DTYPE [n_box], win_box_off int32 [n_win+1]).  Boxes are
    in each window's detector-input pixels; jitter may push them outside
    [0,ow]x[0,oh] (exercising the clip step)."""
    od = cfg.out_dims
    out = []
    off = [0]
    for wi, (f, x, y, w, h, k, _slot) in enumerate(np.asarray(windows).reshape(-1, 7)):
        rng = np.random.default_rng(splitmix64(frame_seed(clip, frame0 + int(f)) ^ (0xB0C5 + wi * 7919)))
        ow, oh = od[k]
        sx, sy = ow / w, oh / h
        ob = scene.boxes[int(f)]
        oc = scene.cls[int(f)]
        rows = []
        if len(ob):
            ix1 = np.maximum(ob[:, 0], x)
            iy1 = np.maximum(ob[:, 1], y)
            ix2 = np.minimum(ob[:, 2], x + w)
            iy2 = np.minimum(ob[:, 3], y + h)
            inter = np.clip(ix2 - ix1, 0, None) * np.clip(iy2 - iy1, 0, None)
            area = (ob[:, 2] - ob[:, 0]) * (ob[:, 3] - ob[:, 1])
            for q in np.nonzero(inter >= 0.25 * area)[0]:
                n = 1 + (int(rng.random() < 0.5) if cfg.copies == "bernoulli" else int(rng.poisson(1.0)))
                base = np.array([(ix1[q] - x) * sx, (iy1[q] - y) * sy, (ix2[q] - x) * sx, (iy2[q] - y) * sy])
                for _ in range(n):
                    j = base + rng.normal(0.0, 1.0, 4)
                    rows.append((j[0], j[1], j[2], j[3], rng.uniform(0.3, 1.0), oc[q]))
        nfp = int(rng.poisson(cfg.fp_rate)) if cfg.fp_rate > 0 else 0
        for _ in range(nfp):
            bw, bh = rng.uniform(8, 60, 2)
            bx, by = rng.uniform(0, max(ow - bw, 1)), rng.uniform(0, max(oh - bh, 1))
            rows.append((bx, by, bx + bw, by + bh, rng.uniform(0.3, 1.0), int(rng.integers(0, 3))))
        if extra_edge_cases:
            rows.append((5.0, 5.0, 5.0, 9.0, 0.9, 0))                 # degenerate (x2 == x1)
            rows.append((1.0, 1.0, 3.0, 3.0, float("nan"), 1))          # NaN score
            rows.append((-10.0, -3.0, 20.0, 12.0, 0.25, 2))             # score == thr (dropped)
            rows.append((2.0, 2.0, 12.0, 12.0, -0.0, 0))                # -0.0 score
            rows.append((float(ow) - 4, 0.0, float(ow) + 30, 9.0, 0.77, 1))  # clipped right edge
        arr = np.zeros(len(rows), BOX_DTYPE)
        if rows:
            a = np.asarray(rows, dtype=np.float64)
            for i, name in enumerate(("x1", "y1", "x2", "y2", "score")):
                arr[name] = a[:, i].astype(np.float32)
            arr["cls"] = a[:, 5].astype(np.int32)
        out.append(arr)
        off.append(off[-1] + len(arr))
    boxes = np.concatenate(out) if out else np.zeros(0, BOX_DTYPE)
    return boxes, np.asarray(off, np.int32)


# --------------------------------------------------------------------------- NEXT-4a
def assign_batch(seed: int, B: int, m_range=(3, 40), n_range=(3, 40), sigma_px: float = 24.0,
                 miss: float = 0.1, spawn: float = 0.1):
    """A batch of B synthetic tracker score matrices p_ij for the
    Hungarian stage: per problem, m track prefixes at uniform positions in a
    1920x1080 frame; each continues into a detection with probability 1-miss
    (jittered by N(0, sigma_px/2)), plus Poisson(spawn*m) new detections; the
    stand-in scorer gives p_ij = exp(-d_ij^2 / (2 sigma_px^2)) * U[0.85, 1]
    (float32).  Sizes m ~ U[m_range], n follows from the model and is clipped
    to n_range.  Returns (list of float32 [m][n] matrices)."""
    rng = np.random.default_rng(splitmix64(seed ^ 0xA551))
    out = []
    for _ in range(B):
        m = int(rng.integers(m_range[0], m_range[1] + 1))
        tp = rng.uniform((0, 0), (1920, 1080), (m, 2))
        keep = rng.random(m) >= miss
        det = tp[keep] + rng.normal(0, sigma_px / 2, (int(keep.sum()), 2))
        new = rng.uniform((0, 0), (1920, 1080), (int(rng.poisson(spawn * m)), 2))
        det = np.concatenate([det, new])
        rng.shuffle(det)
        n = int(np.clip(len(det), n_range[0], n_range[1]))
        if len(det) < n:
            det = np.concatenate([det, rng.uniform((0, 0), (1920, 1080), (n - len(det), 2))])
        det = det[:n]
        d2 = ((tp[:, None, :] - det[None, :, :]) ** 2).sum(-1)
        p = np.exp(-d2 / (2 * sigma_px ** 2)) * rng.uniform(0.85, 1.0, (m, n))
        out.append(p.astype(np.float32))
    return out


# --------------------------------------------------------------------------- NEXT-4b
def lane_paths(seed: int, n_lanes: int = 12, W: int = 1920, H: int = 1080):
    """Synthetic traffic-camera lanes for the refinement stage:
    each lane is a 3-5 point polyline from one frame border to another through
    the interior (a turning movement).  Returns a list of float64 [k][2]."""
    rng = np.random.default_rng(splitmix64(seed ^ 0x7E4E))
    def border_point():
        side = int(rng.integers(0, 4))
        t = rng.uniform(0.1, 0.9)
        return [(t * W, 0.0), (W, t * H), (t * W, float(H)), (0.0, t * H)][side], side
    lanes = []
    for _ in range(n_lanes):
        (a, sa) = border_point()
        (b, sb) = border_point()
        while sb == sa:
            (b, sb) = border_point()
        k = int(rng.integers(1, 4))
        mids = [(rng.uniform(0.25, 0.75) * W, rng.uniform(0.25, 0.75) * H) for _ in range(k)]
        lanes.append(np.asarray([a] + mids + [b], np.float64))
    return lanes


def _walk(lane, speed, rng, jitter):
    """Positions every frame along a lane polyline at `speed` px/frame."""
    seg = np.sqrt((np.diff(lane, axis=0) ** 2).sum(1))
    L = seg.sum()
    s = np.arange(0.0, L, speed)
    cum = np.concatenate([[0], np.cumsum(seg)])
    k = np.clip(np.searchsorted(cum, s, side="right") - 1, 0, len(seg) - 1)
    lam = (s - cum[k]) / np.maximum(seg[k], 1e-12)
    pts = lane[k] + lam[:, None] * (lane[k + 1] - lane[k])
    return pts + rng.normal(0, jitter, pts.shape)


def track_sets(seed: int, n_train: int = 2000, n_query: int = 4000, n_lanes: int = 12, gap: int = 16):
    """Training tracks S* (full-rate walks along the lanes, box 24-60 px) and
    query tracks (a random middle 30-80% of a walk, sampled every `gap`
    frames — a reduced-rate track) as lists of float32 [n][4] boxes.
    Returns (lanes, train boxes, query boxes, query lane ids)."""
    rng = np.random.default_rng(splitmix64(seed ^ 0x7E4F))
    lanes = lane_paths(seed, n_lanes)

    def boxes_of(pts):
        sz = rng.uniform(24, 60)
        b = np.concatenate([pts - sz / 2, pts + sz / 2], 1)
        return b.astype(np.float32)

    train, query, qlane = [], [], []
    for _ in range(n_train):
        li = int(rng.integers(0, n_lanes))
        train.append(boxes_of(_walk(lanes[li], rng.uniform(4, 12), rng, 3.0)))
    for _ in range(n_query):
        li = int(rng.integers(0, n_lanes))
        pts = _walk(lanes[li], rng.uniform(4, 12), rng, 3.0)
        n = len(pts)
        a = int(rng.uniform(0.1, 0.35) * n)
        b = max(a + 2, int(rng.uniform(0.65, 0.9) * n))
        q = pts[a:b:gap]
        if len(q) < 2:
            q = pts[a:b][[0, -1]]
        query.append(boxes_of(q))
        qlane.append(li)
    return lanes, train, query, np.asarray(qlane)


# --------------------------------------------------------------------------- configs[4] clip pools
def clip_pool(cfg: Config, pool: int) -> List[Tuple[Scene, np.ndarray]]:
    """The `pool` distinct generated clips the configs[4] sweep draws on:
    (scene, score grids) of clip ids 0..pool-1.  Clip c of the 1000-clip job
    uses pool entry c mod pool (host generation of 1000 full clips would take
    ~25 min; the kernels keep nothing from one clip to the next, so reusing
    a clip's data costs the same work as a new clip)."""
    out = []
    for c in range(pool):
        sc = make_scene(cfg, c)
        out.append((sc, score_grids(cfg, c, sc)))
    return out


def standin_boxes_torch(cfg: Config, clip: int, obj_boxes, obj_cls, obj_off, windows, device):
    """Vectorised stand-in detector on the device (torch, untimed input
    generation for the configs[4] sweep): per window, ONE jittered copy
    (sigma = 1 detector px) of (object ∩ window) for every object of the
    window's frame with >= 25 % of its area inside, score U[0.3, 1], cls =
    the object's class — the same model as `standin_boxes` without the
    Poisson extra copies and false positives.  obj_boxes float64 [n_obj, 4]
    (frame px), obj_cls int32 [n_obj], obj_off int64 [F+1] (per-frame CSR),
    windows int32 [n_win, 7] (device).  Returns (boxes float32 [n_box, 6]
    with cls bits in column 5, win_box_off int32 [n_win+1])."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(clip_seed(clip) & ((1 << 63) - 1))
    n_win = int(windows.shape[0])
    if n_win == 0:
        return torch.zeros((1, 6), dtype=torch.float32, device=device), torch.zeros(1, dtype=torch.int32, device=device)
    ob = torch.as_tensor(obj_boxes, dtype=torch.float64, device=device)
    oc = torch.as_tensor(obj_cls, dtype=torch.int32, device=device)
    off = torch.as_tensor(obj_off, dtype=torch.int64, device=device)
    cnt = off[1:] - off[:-1]
    kmax = int(cnt.max().item()) if len(cnt) else 0
    w = windows.to(torch.int64)
    fr = w[:, 0]
    if kmax == 0:
        return torch.zeros((1, 6), dtype=torch.float32, device=device), torch.zeros(n_win + 1, dtype=torch.int32,
                                                                                    device=device)
    j = torch.arange(kmax, device=device)
    valid = j[None, :] < cnt[fr][:, None]                                   # [n_win, kmax]
    idx = (off[fr][:, None] + j[None, :]).clamp(max=max(len(ob) - 1, 0))
    b = ob[idx]                                                              # [n_win, kmax, 4]
    x, y, ww, hh = (w[:, i].to(torch.float64)[:, None] for i in (1, 2, 3, 4))
    ix1, iy1 = torch.maximum(b[..., 0], x), torch.maximum(b[..., 1], y)
    ix2, iy2 = torch.minimum(b[..., 2], x + ww), torch.minimum(b[..., 3], y + hh)
    inter = (ix2 - ix1).clamp(min=0) * (iy2 - iy1).clamp(min=0)
    area = (b[..., 2] - b[..., 0]) * (b[..., 3] - b[..., 1])
    keep = valid & (inter >= 0.25 * area)
    wi, oj = torch.nonzero(keep, as_tuple=True)                              # window-major order
    od = torch.as_tensor(cfg.out_dims, dtype=torch.float64, device=device)[w[wi, 5]]
    sx, sy = od[:, 0] / ww[wi, 0], od[:, 1] / hh[wi, 0]
    loc = torch.stack([(ix1[wi, oj] - x[wi, 0]) * sx, (iy1[wi, oj] - y[wi, 0]) * sy,
                       (ix2[wi, oj] - x[wi, 0]) * sx, (iy2[wi, oj] - y[wi, 0]) * sy], 1)
    loc = loc + torch.randn(loc.shape, generator=g, dtype=torch.float64, device=device)
    score = 0.3 + 0.7 * torch.rand(len(wi), generator=g, dtype=torch.float64, device=device)
    n_box = len(wi)
    out = torch.empty((max(n_box, 1), 6), dtype=torch.float32, device=device)
    if n_box:
        out[:n_box, :4] = loc.to(torch.float32)
        out[:n_box, 4] = score.to(torch.float32)
        out[:n_box, 5] = oc[idx[wi, oj]].view(torch.float32)
    wbo = torch.zeros(n_win + 1, dtype=torch.int32, device=device)
    wbo[1:] = torch.cumsum(torch.bincount(wi, minlength=n_win), 0).to(torch.int32)
    return out, wbo
