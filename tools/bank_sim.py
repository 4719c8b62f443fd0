"""CPU model of k_deposit_tiled's shared-memory bank conflicts: builds one
tile (window layout exactly as the kernel), a cell-sorted marker set of the
paper's density, and counts, for every ATOMS instruction of every warp, the
wavefronts (max lanes on one bank) of the lane-rotated slot order.
Used to compare window layouts / rotations without the GPU.

  python tools/bank_sim.py --size A            # mzetamax 64
  python tools/bank_sim.py --size B --mzetamax 16
"""
import argparse
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1510_05546_b200 as G  # noqa: E402  (host geometry only; no GPU needed)
import synth  # noqa: E402

TWO_PI = 2 * math.pi


def build(size, mzetamax, ring_frac, tile_max, nmu, seed, layout):
    over = {"mzetamax": mzetamax} if mzetamax else {}
    cfg = synth.config(size, **over)
    p = G.gtcp_default_params(size, **over)
    g = G.gtcp_geometry(p)
    M, P = p.mpsi, p.mzetamax
    mt, ig, qt = np.array(g["mtheta"]), np.array(g["igrid"]), np.array(g["qtinv"])
    a0, a1 = p.a0, p.a1
    dr = (a1 - a0) / M
    om = p.omega0
    dz = TWO_PI / P
    rho_cut = 3.0 / om
    i = int(ring_frac * M)
    ncell = max(1, tile_max // (cfg["micell"] * P))
    c0 = mt[i] // 3
    c1 = c0 + ncell - 1
    rng = np.random.default_rng(seed)
    # markers: micell per (cell, plane), uniform in the cell, mu ~ Exp(1)/B
    n_per = cfg["micell"]
    C, K = np.meshgrid(np.arange(c0, c1 + 1), np.arange(P), indexing="ij")
    C = np.repeat(C.ravel(), n_per)
    K = np.repeat(K.ravel(), n_per)
    n = len(C)
    r = a0 + (i + rng.random(n)) * dr
    zeta = (K + rng.random(n)) * dz
    alpha = (C + rng.random(n)) / mt[i] * TWO_PI
    theta = np.mod(alpha + zeta * qt[i], TWO_PI)
    invB = 1.0 + r / p.R0 * np.cos(theta)
    mu = rng.exponential(1.0, n) * invB
    mb = np.zeros(n, np.int64)
    for b in range(1, nmu):
        mb += mu >= -math.log(1 - b / nmu)
    key = ((ig[i] + C) * P + K) * nmu + mb
    order = np.lexsort((rng.random(n), key))
    r, zeta, theta, invB, mu, K = r[order], zeta[order], theta[order], invB[order], mu[order], K[order]
    # streaming since the bin: `age` stages of parallel motion (v_par ~ N(0, 1),
    # zeta advances v_par B / R0 per unit time, theta follows the field line)
    age = layout.get("age", 0.0)
    if age:
        vpar = rng.standard_normal(n)
        dzeta = vpar / p.R0 * (0.5 * p.dt) * age
        zeta = zeta + dzeta
        theta = np.mod(theta + dzeta * qt[i], TWO_PI)
        K = np.clip(np.floor(zeta / dz).astype(np.int64), 0, P - 1)
        zeta = np.clip(zeta, 0, P * dz - 1e-12)
    rho = np.sqrt(2.0 * mu * invB) / om
    # window (kernel: win_halo / win_width / js)
    h = min(int(math.ceil(rho_cut / dr)) + 1, 7)
    m_lo, m_hi = max(0, i - h), min(M, i + 1 + h)
    nr = m_hi - m_lo + 1
    W = np.zeros(nr, np.int64)
    js = np.zeros((P + 1, nr), np.int64)
    half0 = 0.5 * (c1 + 1 - c0) / mt[i]
    fc = 0.5 * (c0 + c1 + 1) / mt[i]
    hw = np.zeros(nr)
    for q in range(nr):
        m = m_lo + q
        dq = (qt[i] - qt[m]) / TWO_PI
        rm = a0 + m * dr
        thm = rho_cut / rm / TWO_PI if i - 1 <= m <= i + 2 else 0.0
        hw[q] = half0 + dz * abs(dq) + thm + 1.0 / mt[m]
        W[q] = min(int(math.ceil(2 * hw[q] * mt[m])) + 2, mt[m])
        for kk in range(P + 1):
            f = fc + kk * dz * dq - hw[q]
            f -= math.floor(f)
            js[kk, q] = min(max(int(math.floor(f * mt[m])), 0), mt[m] - 1)
    col = np.zeros(nr, np.int64)
    S = 0
    for q in range(nr):
        col[q] = S
        S += W[q] + 1 + layout.get("ring_gap", 0)
        if layout.get("ring_align"):
            S += (-S) % layout["ring_align"]
    pad = layout.get("pad", 4)  # kPlanePad of the kernel (GTCP_PLANE_PAD)
    if pad is not None:
        S += (pad - (S & 31) + 32) & 31
    return dict(n=n, r=r, zeta=zeta, theta=theta, rho=rho, K=K, mt=mt, qt=qt, a0=a0, a1=a1, dr=dr, M=M,
                m_lo=m_lo, nr=nr, W=W, js=js, col=col, S=S)


def lane_addresses(T, p0, lq, mq, kq, t, rot):
    """word address of the lo limb touched by each of the 32 lanes (markers p0..p0+31)."""
    b = np.arange(32)
    pidx = p0 + b
    b2, b3, b4 = (b >> 2) & 1, (b >> 3) & 1, (b >> 4) & 1
    l = (lq + b) & 3 if rot else np.full(32, lq)
    mm = (mq ^ b2) if rot else np.full(32, mq)
    kko = (kq ^ b3) if rot else np.full(32, kq)
    nd = (t ^ b4) if rot else np.full(32, t)
    r, th, z, rho = T["r"][pidx], T["theta"][pidx], T["zeta"][pidx], T["rho"][pidx]
    sr = np.where(l == 0, 1, np.where(l == 2, -1, 0))
    st = np.where(l == 1, 1, np.where(l == 3, -1, 0))
    rl = np.clip(r + sr * rho, T["a0"], T["a1"])
    tl = th + st * rho / r
    ir = np.clip(np.floor((rl - T["a0"]) / T["dr"]).astype(np.int64), 0, T["M"] - 1)
    m = ir + mm
    q = m - T["m_lo"]
    inband = (q >= 0) & (q < T["nr"])
    qc = np.where(inband, q, 0)
    mtm = T["mt"][m]
    sl = (tl - z * T["qt"][m]) / TWO_PI
    sl = (sl - np.floor(sl)) * mtm
    j = np.minimum(np.floor(sl).astype(np.int64), mtm - 1)
    j1 = np.where(j + 1 == mtm, 0, j + 1)
    jn = np.where(nd == 1, j1, j)
    row = T["K"][pidx] + kko
    jsv = T["js"][row, qc]
    du = np.mod(jn - jsv, mtm)
    Wq = np.where(inband, T["W"][qc], 0)
    addr = row * T["S"] + T["col"][qc] + np.minimum(du, Wq)
    return np.where(inband, addr, -1 - b)  # out of band: trash slot (distinct dummy)


def wavefronts(addr, distinct=False):
    """max over banks of the lanes (or, distinct=True, of the distinct words) on one bank"""
    if distinct:
        addr = np.unique(addr)
    bank = np.mod(addr, 32)
    return np.bincount(bank, minlength=32).max()


def run(T, rot=True, warps=400, seed=0):
    rng = np.random.default_rng(seed)
    nw = T["n"] // 32
    ws = rng.choice(nw, size=min(warps, nw), replace=False)
    tot, cnt = 0, 0
    for w in ws:
        for lq in range(4):
            for mq in range(2):
                for kq in range(2):
                    for t in range(2):
                        tot += wavefronts(lane_addresses(T, w * 32, lq, mq, kq, t, rot))
                        cnt += 1
    return tot / cnt


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", default="A")
    ap.add_argument("--mzetamax", type=int, default=None)
    ap.add_argument("--nmu", type=int, default=4)
    a = ap.parse_args()
    for frac in (0.3, 0.6, 0.9):
        T = build(a.size, a.mzetamax, frac, 8192, a.nmu, 1, {"pad": 4})
        print(f"ring {frac:.1f}: S={T['S']} nr={T['nr']} W={list(T['W'])} wavefronts/ATOMS rot={run(T):.2f} "
              f"norot={run(T, rot=False):.2f}")


def lane_addresses_v(T, pidx, lq, mq, kq, t, bits):
    """variant: bits = (l_shift, mm_bit, kk_bit, nd_bit) of the lane rotation."""
    b = np.arange(32)
    ls, mb_, kb, nb = bits
    l = (lq + (b >> ls)) & 3
    mm = mq ^ ((b >> mb_) & 1)
    kko = kq ^ ((b >> kb) & 1)
    nd = t ^ ((b >> nb) & 1)
    r, th, z, rho = T["r"][pidx], T["theta"][pidx], T["zeta"][pidx], T["rho"][pidx]
    sr = np.where(l == 0, 1, np.where(l == 2, -1, 0))
    st = np.where(l == 1, 1, np.where(l == 3, -1, 0))
    rl = np.clip(r + sr * rho, T["a0"], T["a1"])
    tl = th + st * rho / r
    ir = np.clip(np.floor((rl - T["a0"]) / T["dr"]).astype(np.int64), 0, T["M"] - 1)
    m = ir + mm
    q = m - T["m_lo"]
    inband = (q >= 0) & (q < T["nr"])
    qc = np.where(inband, q, 0)
    mtm = T["mt"][m]
    sl = (tl - z * T["qt"][m]) / TWO_PI
    sl = (sl - np.floor(sl)) * mtm
    j = np.minimum(np.floor(sl).astype(np.int64), mtm - 1)
    j1 = np.where(j + 1 == mtm, 0, j + 1)
    jn = np.where(nd == 1, j1, j)
    row = T["K"][pidx] + kko
    jsv = T["js"][row, qc]
    du = np.mod(jn - jsv, mtm)
    Wq = np.where(inband, T["W"][qc], 0)
    addr = row * T["S"] + T["col"][qc] + np.minimum(du, Wq)
    return np.where(inband, addr, -1 - b)


def run_v(T, bits, mapping="contig", warps=300, seed=0, distinct=False):
    rng = np.random.default_rng(seed)
    n = T["n"]
    nw = n // 32
    ws = rng.choice(nw, size=min(warps, nw), replace=False)
    tot = cnt = same = 0
    for w in ws:
        b = np.arange(32)
        if mapping == "contig":
            pidx = w * 32 + b
        elif mapping == "strided":  # lane b takes marker w + b * (n // 32)
            pidx = w + b * nw
        elif mapping.startswith("span"):  # "spanS": lane b -> span (b % S), consecutive markers by b // S
            S = int(mapping[4:])
            span = n // S
            pidx = (b % S) * span + (w % (span // (32 // S))) * (32 // S) + b // S
        else:  # "groupG": G consecutive markers per lane group, 32/G groups spread over the tile
            G = int(mapping[5:])
            ng = 32 // G
            span = n // ng
            pidx = (w % (span // G)) * G + (b % G) + (b // G) * span
        for lq in range(4):
            for mq in range(2):
                for kq in range(2):
                    for t in range(2):
                        a = lane_addresses_v(T, pidx, lq, mq, kq, t, bits)
                        tot += wavefronts(a, distinct)
                        same += 32 - len(np.unique(a))
                        cnt += 1
    return tot / cnt, same / cnt
