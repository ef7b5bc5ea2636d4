"""Seeded synthetic profiling tables (the input recipe of DESIGN.md §4).

This module is the ONE thing the oracle side and the CUDA side share: it makes
inputs and holds none of the method's arithmetic (no labelling, binning,
histograms, splits or tree walks).  It has two implementations of the same
counter-based recipe:

* ``generate()`` — numpy, on the host (tests, the oracle, e2e host buffers);
* ``generate_device()`` — ``synth/synth.cu`` (libsynth.so), writing straight
  into device memory for the bench's 1e8-row tables.

Both produce byte-identical float32 tables (tests/test_synth.py checks it on
the GPU).  Every random draw is a pure function of (seed, row, column):

    h   = splitmix64(seed ^ splitmix64(row * 0x9E3779B97F4A7C15 + col))
    u24 = h >> 40                          (24 random bits)
    feature f of row i = grid_f[(u24(seed, i, f) * G_f) >> 24]
    noise factor of variant v = 1 + a * (2 * u24(seed, i, 1000 + v) / 2^24 - 1)

and each variant's time is a closed-form cost model evaluated
in IEEE double with one rounding per operation (no FMA: numpy never fuses, the
device uses __dmul_rn/__dadd_rn/__ddiv_rn), then rounded to float32.

Feature grids follow the inputs of Table 3: geometric trip counts
(XSBench-style 10000*2^k), small categorical resources, flags and distractors.
The variants follow the paper's three use-cases: host vs device
offload (C1), num_threads (C2), GPU block size (C3) and their product (C4).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsynth.so")

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def _geom(lo: float, hi_exp: float, k: int) -> np.ndarray:
    """k points lo * 2^(hi_exp * j/(k-1)), rounded to float32 (host table)."""
    j = np.arange(k, dtype=np.float64)
    return (lo * np.power(2.0, hi_exp * j / (k - 1))).astype(np.float32)


def _lin(start: float, step: float, k: int) -> np.ndarray:
    return (start + step * np.arange(k, dtype=np.float64)).astype(np.float32)


@dataclass
class Config:
    name: str
    cid: int          # cost-model id shared with synth.cu
    N: int            # rows of the full table (BASELINE.json configs)
    F: int
    V: int
    D: int            # max depth
    grids: list = field(default_factory=list)
    seed: int = 1
    regions: int = 1  # C2: region = row mod 3 (R15)

    @property
    def grid_table(self):
        off = np.zeros(self.F + 1, np.int32)
        for f, g in enumerate(self.grids):
            off[f + 1] = off[f] + len(g)
        flat = np.concatenate(self.grids).astype(np.float32)
        return flat, off


def _c3_grids():
    return [
        _geom(1024.0, 20.0, 256),          # f0 trip count N: 1K .. 1G (geometric, 256 pts)
        _lin(16.0, 8.0, 30),               # f1 registers / thread: 16..248
        _lin(0.0, 4.0, 25),                # f2 shared KB / block: 0..96
        _geom(1.0, 10.0, 256),             # f3 flops / iteration: 1..1024
        _geom(4.0, 8.0, 256),              # f4 bytes / iteration: 4..1024
        _lin(0.0, 0.125, 256),             # f5..f7 distractors
        _lin(-16.0, 0.125, 256),
        _lin(100.0, 1.0, 256),
    ]


CONFIGS = {
    # C1: 1 region, host vs GPU offload, feature = trip count
    "C1": Config("C1", 1, 512, 1, 2, 4, [_geom(128.0, 17.0, 64)], seed=1),
    # C2: 3 regions, num_threads variants {1..64} (P:364-374 style), 4 features
    "C2": Config("C2", 2, 100_000, 4, 7, 8,
                 [_geom(64.0, 20.0, 256), _geom(8.0, 8.0, 9), _lin(0.0, 1.0 / 64.0, 33),
                  _lin(1.0, 1.0, 8)], seed=2, regions=3),
    # C3: GPU thread-block size {32..1024}, 8 features, 256 bins
    "C3": Config("C3", 3, 1_000_000, 8, 6, 12, _c3_grids(), seed=3),
    # C4: offload x threads x block size, 48 classes, 16 features
    "C4": Config("C4", 4, 100_000_000, 16, 48, 12,
                 _c3_grids() + [
                     _lin(8.0, 8.0, 16),            # f8 host cores 8..128
                     _lin(0.0, 1.0, 2),             # f9 data resident on device
                     _geom(1.0, 12.0, 64),          # f10 transfer bytes / iteration
                     _lin(0.0, 1.0, 2),             # f11 NUMA-remote flag
                     _lin(0.0, 0.25, 256),          # f12..f15 distractors
                     _lin(-1.0, 0.0078125, 256),
                     _geom(0.001, 16.0, 256),
                     _lin(7.0, 3.0, 200),
                 ], seed=4),
}


# ------------------------------------------------------------------ RNG --
def _splitmix64(z):
    z = (z + np.uint64(GOLDEN)) & np.uint64(M64)
    z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & np.uint64(M64)
    z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & np.uint64(M64)
    return z ^ (z >> np.uint64(31))


def u24(seed: int, rows: np.ndarray, col: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        r = rows.astype(np.uint64) * np.uint64(GOLDEN) + np.uint64(col)
        h = _splitmix64(np.uint64(seed) ^ _splitmix64(r))
    return (h >> np.uint64(40)).astype(np.uint64)


# ------------------------------------------------------------ cost models --
def _costs(cfg: Config, x: list, rows: np.ndarray) -> list:
    """Per-variant cost (float64), one IEEE rounding per written operation."""
    d = np.float64
    if cfg.cid == 1:
        N = x[0]
        return [N * d(1.0) + d(2000.0), N * d(0.02) + d(30000.0)]
    if cfg.cid == 2:
        N, m, s, cls = x
        r = (rows % 3).astype(np.int64)
        w = np.array([1.0, 2.5, 0.6])[r]
        o = np.array([3000.0, 1500.0, 6000.0])[r]
        out = []
        for v in range(cfg.V):
            p = d(float(1 << v))
            a = d(1.0) - s
            b = a / p
            c = s + b
            t1 = N * w
            t1 = t1 * c
            t2 = o * cls
            t2 = t2 * p
            bwp = np.minimum(p * d(8.0), d(96.0))
            t3 = N * m
            t3 = t3 / bwp
            out.append((t1 + t2) + t3)
        return out
    if cfg.cid in (3, 4):
        N, regs, smem, flops, byts = x[0], x[1], x[2], x[3], x[4]
        w1 = flops * d(0.5)
        w2 = byts * d(0.25)
        work = N * (w1 + w2)
        cap = d(65536.0) / regs
        sm = smem / d(32.0)
        sm = d(1.0) + sm
        if cfg.cid == 3:
            out = []
            for v in range(cfg.V):
                T = d(float(32 << v))
                conc = np.minimum(T, cap)
                t = work / conc
                g = d(2000.0) * T
                g = g * sm
                out.append(t + g)
            return out
        cores, res, xfer, numa = x[8], x[9], x[10], x[11]
        out = []
        for v in range(cfg.V):
            dev = v // 24
            th = d(float(8 << ((v // 6) % 4)))   # 8,16,32,64
            blk = d(float(32 << (v % 6)))        # 32..1024
            if dev == 0:  # host: th threads, schedule chunk = blk
                t = work / np.minimum(th, cores)
                nf = numa * d(0.25)
                nf = d(1.0) + nf
                t = t * nf
                s1 = N / blk
                s1 = s1 * d(40.0)
                t = t + s1
                s2 = blk * (w1 + w2)   # tail imbalance of one chunk
                t = t + s2
                t = t + th * d(800.0)
            else:         # device: block blk, teams multiplier th/8
                mm = th / d(8.0)
                conc = np.minimum(blk, cap)
                conc = conc * mm
                conc = conc * d(16.0)
                t = work / conc
                g = d(2000.0) * blk
                g = g * sm
                g = g / mm
                t = t + g
                xr = d(1.0) - res
                xb = N * xfer
                xb = xb / d(25.0)
                xb = xb * xr
                t = t + xb
                t = t + d(20000.0)
                t = t + mm * d(3000.0)
            out.append(t)
        return out
    raise ValueError(cfg.cid)


def generate(cfg: Config | str, row0: int, n: int, seed: int | None = None,
             noise: float = 0.05, times: bool = True):
    """Host table rows [row0, row0+n): (features f32 [n][F], times f32 [n][V]).
    times=False skips the cost models (selection inputs): times is None."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    seed = cfg.seed if seed is None else seed
    rows = np.arange(row0, row0 + n, dtype=np.uint64)
    X = np.empty((n, cfg.F), np.float32)
    for f, g in enumerate(cfg.grids):
        idx = (u24(seed, rows, f) * np.uint64(len(g))) >> np.uint64(24)
        X[:, f] = g[idx.astype(np.int64)]
    if not times:
        return X, None
    x64 = [X[:, f].astype(np.float64) for f in range(cfg.F)]
    costs = _costs(cfg, x64, rows.astype(np.int64))
    T = np.empty((n, cfg.V), np.float32)
    for v, c in enumerate(costs):
        if noise:
            u = u24(seed, rows, 1000 + v).astype(np.float64) * np.float64(2.0 ** -24)
            fac = np.float64(2.0) * u
            fac = fac - np.float64(1.0)
            fac = np.float64(noise) * fac
            fac = np.float64(1.0) + fac
            c = c * fac
        T[:, v] = c.astype(np.float32)
    return X, T


# ------------------------------------------------------ device generator --
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            raise RuntimeError("synth/libsynth.so not built: run __graft_entry__.build()")
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        L.synth_generate.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_int, ctypes.c_int, P, P, ctypes.c_double, P, P, P]
        L.synth_generate.restype = ctypes.c_int
        _lib = L
    return _lib


def generate_device(cfg: Config | str, row0: int, n: int, feat_ptr: int, times_ptr: int,
                    grid_dev_ptr: int, off_dev_ptr: int, stream: int = 0,
                    seed: int | None = None, noise: float = 0.05) -> None:
    """Write rows [row0, row0+n) into device buffers feat [n][F] f32, times [n][V] f32.
    grid_dev_ptr / off_dev_ptr: device copies of ``cfg.grid_table``.  times_ptr may be 0."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    seed = cfg.seed if seed is None else seed
    rc = _load().synth_generate(cfg.cid, seed, row0, n, cfg.F, cfg.V, grid_dev_ptr, off_dev_ptr,
                                noise, feat_ptr, times_ptr, stream)
    if rc != 0:
        raise RuntimeError(f"synth_generate failed: {rc}")


def region_rows(cfg: Config, r: int) -> np.ndarray:
    """Global row ids of region r (C2: region = row mod 3)."""
    return np.arange(r, cfg.N, cfg.regions, dtype=np.int64)


def random_tree(cfg: Config | str, depth: int, seed: int = 6):
    """SURVEY §8(d) C5 worst case: a complete tree of the given depth, BFS order;
    internal node k splits on feature u24(seed, k, 0) % F at the midpoint of two
    adjacent grid values of that feature; leaf labels u24(seed, k, 1) % V.
    Returns a dict of numpy columns (feature, left, right, label, depth, threshold)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    n = (1 << (depth + 1)) - 1
    k = np.arange(n, dtype=np.uint64)
    internal = k < np.uint64((1 << depth) - 1)
    feat = (u24(seed, k, 0) % np.uint64(cfg.F)).astype(np.int32)
    thr = np.zeros(n, np.float64)
    for f in range(cfg.F):
        g = cfg.grids[f].astype(np.float64)
        sel = np.nonzero(internal & (feat == f))[0]
        if len(g) < 2:
            feat[sel] = (f + 1) % cfg.F
            continue
        j = (u24(seed, sel.astype(np.uint64), 2) % np.uint64(len(g) - 1)).astype(np.int64)
        thr[sel] = (g[j] + g[j + 1]) / 2
    # features whose grid has < 2 values were remapped above; recompute their thresholds
    for f in range(cfg.F):
        g = cfg.grids[f].astype(np.float64)
        sel = np.nonzero(internal & (feat == f) & (thr == 0))[0]
        if len(sel) and len(g) >= 2:
            j = (u24(seed, sel.astype(np.uint64), 2) % np.uint64(len(g) - 1)).astype(np.int64)
            thr[sel] = (g[j] + g[j + 1]) / 2
    left = np.where(internal, 2 * k.astype(np.int64) + 1, -1).astype(np.int32)
    right = np.where(internal, 2 * k.astype(np.int64) + 2, -1).astype(np.int32)
    label = (u24(seed, k, 1) % np.uint64(cfg.V)).astype(np.int32)
    dep = np.floor(np.log2(k.astype(np.float64) + 1)).astype(np.int32)
    return dict(feature=np.where(internal, feat, -1).astype(np.int32), left=left, right=right,
                label=label, depth=dep, threshold=np.where(internal, thr, 0.0))
