"""CPU model of k_push's gather on the L1 data pipe: a
quarter-warp of a warp-wide LDG.128 takes one wavefront per distinct 128-byte
line on each of the 8 sixteen-byte chunk positions of a line (address bits
4-6; measured with tools/microbench/ldg256.cu).  Builds cell-sorted markers of the paper's density on the
class-A grid (bin key order of H-4 with the mu sub-bins), ages them by
`--age` RK2 half-steps of parallel streaming, and counts the wavefronts of
the 6 x 8 gather loads per marker for field-record layouts:
  interleaved48 : node n of interval k at 48 * (k gstride + n), pair j, j+1 = 96 B
                  (gstride = mgrid padded to --gstride-res mod 8; -1: mgrid)
  pair128       : the pair (j, j+1) of interval k as one 128-byte line
  interleaved48_f32 / pair64_f32 : the same in fp32 (3 LDG.128 per pair)

  python tools/push_l1_sim.py --size A --ncell 400 --age 1 --gstride-res 3
"""
import argparse
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1510_05546_b200 as G  # noqa: E402  (host geometry only)
import synth  # noqa: E402

TWO_PI = 2 * math.pi


def markers(size, ncell_ring, seed, age, nmu=4):
    p = G.gtcp_default_params(size)
    geo = G.gtcp_geometry(p)
    mt, ig, qt = geo["mtheta"], geo["igrid"], geo["qtinv"]
    cfg = synth.config(size)
    M, K = p.mpsi, p.mzetamax
    dr = (p.a1 - p.a0) / M
    rng = np.random.default_rng(seed)
    out = []
    i = M // 2  # a mid ring
    c = np.arange(ncell_ring) % mt[i]
    for k in range(2):
        C, Kk = np.meshgrid(c, [k], indexing="ij")
        C = np.repeat(C.ravel(), cfg["micell"])
        n = len(C)
        r = p.a0 + (i + rng.random(n)) * dr
        zeta = (k + rng.random(n)) * TWO_PI / K
        alpha = (C + rng.random(n)) / mt[i] * TWO_PI
        theta = np.mod(alpha + zeta * qt[i], TWO_PI)
        B = 1.0 / (1.0 + r / p.R0 * np.cos(theta))
        mu = rng.exponential(1.0, n) / B
        vpar = rng.standard_normal(n)
        mb = sum((mu >= -math.log(1 - b / nmu)).astype(int) for b in range(1, nmu))
        key = ((ig[i] + C) * K + k) * nmu + mb
        # age: parallel streaming since the bin (field-line following)
        dz = vpar * B / p.R0 * (0.5 * p.dt) * age
        zeta = np.mod(zeta + dz, TWO_PI)
        theta = np.mod(theta + dz * qt[i], TWO_PI)
        out.append((key, r, theta, zeta, mu, B))
    key, r, theta, zeta, mu, B = (np.concatenate(x) for x in zip(*out))
    o = np.lexsort((rng.random(len(key)), key))
    return p, geo, r[o], theta[o], zeta[o], mu[o], B[o]


def records(p, geo, r, theta, zeta, mu, B, res=3):
    """Per marker the 8 (point, ring) global node-pair indices (k gstride + igrid_m + j)."""
    mt, ig, qt = geo["mtheta"], geo["igrid"], geo["qtinv"]
    M, K, mg = p.mpsi, p.mzetamax, geo["mgrid"]
    if res >= 0:
        mg += ((res - mg % 8) % 8 + 8) % 8
    dr = (p.a1 - p.a0) / M
    rho = np.sqrt(2 * mu / B) / p.omega0
    k = np.minimum(np.floor(zeta * K / TWO_PI).astype(int), K - 1)
    rec = []
    for l in range(4):
        rl = r + (rho if l == 0 else -rho if l == 2 else 0)
        tl = theta + (rho / r if l == 1 else -rho / r if l == 3 else 0)
        rl = np.clip(rl, p.a0, p.a1)
        x = (rl - p.a0) / dr
        i = np.clip(np.floor(x).astype(int), 0, M - 1)
        for mm in range(2):
            m = i + mm
            s = (tl - zeta * qt[m]) / TWO_PI
            s = (s - np.floor(s)) * mt[m]
            j = np.minimum(np.floor(s).astype(int), mt[m] - 1)
            rec.append(k * mg + ig[m] + j)
    return np.stack(rec, 1)  # [n, 8]


def wavefronts(rec, layout):
    n = (len(rec) // 32) * 32
    rec = rec[:n].reshape(-1, 32, 8)
    if layout == "interleaved48":
        base, nchunk = rec * 48, 6
    elif layout == "pair128":
        base, nchunk = rec * 128, 6
    elif layout == "interleaved48_f32":
        base, nchunk = rec * 24, 3
    elif layout == "pair64_f32":
        base, nchunk = rec * 64, 3
    tot = 0
    for c in range(nchunk):
        addr = base + 16 * c  # [warps, 32, 8]
        lines, pos = addr // 128, (addr // 16) % 8
        for qw in range(4):
            ql = lines[:, 8 * qw:8 * qw + 8, :]  # [warps, 8 lanes, 8 records]
            qp = pos[:, 8 * qw:8 * qw + 8, :]
            worst = np.zeros(ql.shape[0:1] + ql.shape[2:], np.int64)
            for b in range(8):  # distinct lines on chunk position b
                key = np.where(qp == b, ql, -1)
                srt = np.sort(key, axis=1)
                nd = (np.diff(srt, axis=1) != 0) & (srt[:, 1:] >= 0)
                cnt = nd.sum(axis=1) + (srt[:, 0] >= 0)
                worst = np.maximum(worst, cnt)
            tot += int(worst.sum())
    nldg = rec.shape[0] * 8 * nchunk
    return tot / nldg, tot / rec.shape[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", default="A")
    ap.add_argument("--ncell", type=int, default=400)
    ap.add_argument("--age", type=float, default=1.0)
    ap.add_argument("--gstride-res", type=int, default=3, help="interval stride residue mod 8 (-1: mgrid)")
    a = ap.parse_args()
    p, geo, *st = markers(a.size, a.ncell, 1, a.age)
    rec = records(p, geo, *st, res=a.gstride_res)
    for lay in ("interleaved48", "pair128", "interleaved48_f32", "pair64_f32"):
        per_ldg, per_warp = wavefronts(rec, lay)
        print(f"{lay:18s} {per_ldg:5.2f} wavefronts per LDG.128, {per_warp:6.1f} per warp-marker")


if __name__ == "__main__":
    main()
