"""Synthetic inputs for the benchmark configurations (BASELINE.json configs 1-5).

Host-side (numpy) input synthesis, following the reference generators
(workloads.py:29-67) and SURVEY §8.2 (simulated LiDAR for cfg3).  Value
distributions follow cli.py:349-352: features / grad_out ~ N(0,1), weights
N(0,1)/sqrt(27·Cin).
"""

from __future__ import annotations

import numpy as np


def random_points(rng, count, sigma=1.0):
    """Gaussian world points (workloads.py:29-31)."""
    return rng.normal(0.0, sigma, size=(count, 3))


def sphere_shell_coords(res, band=1.5):
    """Voxels within ``band`` of a sphere of radius 0.35·res centred in [0,res)³ (workloads.py:34-67).

    Enumeration order differs from the reference; the build dedupes and sorts, so the
    resulting grid is identical.
    """
    res = int(res)
    radius = 0.35 * res
    ctr = (res - 1) / 2.0
    nl = (res + 7) // 8
    ax = np.arange(nl) * 8
    lo = np.stack(np.meshgrid(ax, ax, ax, indexing="ij"), -1).reshape(-1, 3)
    dist = np.sqrt(((lo + 3.5 - ctr) ** 2).sum(1))
    lo = lo[np.abs(dist - radius) <= band + np.sqrt(3.0) * 4.0]
    cube = np.stack(np.meshgrid(np.arange(8), np.arange(8), np.arange(8), indexing="ij"), -1).reshape(-1, 3)
    out = []
    for s in range(0, len(lo), 4096):
        blk = (lo[s:s + 4096, None, :] + cube[None]).reshape(-1, 3)
        r = np.sqrt(((blk - ctr) ** 2).sum(1))
        out.append(blk[np.abs(r - radius) <= band])
    return np.concatenate(out) if out else np.zeros((0, 3), np.int64)


def lidar_scan_points(seed, beams=128, azimuths=2048, height=1.73, wall=40.0, noise=0.02, boxes=30):
    """Simulated spinning LiDAR scan: ground plane, r=40 m wall, 30 boxes."""
    rng = np.random.default_rng(seed)
    el = np.deg2rad(np.linspace(-24.8, 2.0, beams))
    az = np.linspace(0.0, 2 * np.pi, azimuths, endpoint=False) + rng.uniform(0, 2 * np.pi / azimuths)
    E, A = np.meshgrid(el, az, indexing="ij")
    d = np.stack([np.cos(E) * np.cos(A), np.cos(E) * np.sin(A), np.sin(E)], -1).reshape(-1, 3)
    o = np.array([0.0, 0.0, height])
    t = np.full(len(d), np.inf)
    dn = d[:, 2] < 0
    t[dn] = -height / d[dn, 2]
    t = np.minimum(t, wall / np.maximum(np.hypot(d[:, 0], d[:, 1]), 1e-9))
    r = rng.uniform(6.0, 35.0, boxes)
    a = rng.uniform(0, 2 * np.pi, boxes)
    cen = np.stack([r * np.cos(a), r * np.sin(a), np.zeros(boxes)], 1)
    half = np.concatenate([rng.uniform(1, 3, (boxes, 2)), rng.uniform(0.8, 2.5, (boxes, 1))], 1)
    for cc, hh in zip(cen, half):
        blo = cc - hh
        bhi = cc + hh
        blo[2] = 0.0
        bhi[2] = 2 * hh[2]
        with np.errstate(divide="ignore", invalid="ignore"):
            ta = (blo - o) / d
            tb = (bhi - o) / d
        tmin = np.nanmax(np.minimum(ta, tb), 1)
        tmax = np.nanmin(np.maximum(ta, tb), 1)
        hit = (tmax >= tmin) & (tmin > 0)
        t = np.where(hit, np.minimum(t, tmin), t)
    return o + d * t[:, None] + rng.normal(0, noise, (len(d), 3))


def conv_tensors(rng, n_in, n_out, cin, cout):
    """(features, weights, grad_out) float32 with the reference CLI distributions (cli.py:349-352)."""
    f = rng.normal(size=(n_in, cin)).astype(np.float32)
    w = (rng.normal(size=(cout, cin, 3, 3, 3)) / np.sqrt(27 * cin)).astype(np.float32)
    go = rng.normal(size=(n_out, cout)).astype(np.float32)
    return f, w, go
