"""Mutation check of the oracle's pins: apply plausible mistakes to a scratch
copy of oracle/gtcp_oracle.c and confirm that the CPU pin suite
(`pytest -m "not gpu"` over tests/test_oracle_*.py) fails for every one.

  python tools/oracle_mutation_check.py

Each mutation is (name, old text, new text) on the oracle source; the check
copies the repo to a temp dir, applies one mutation, rebuilds the oracle there
and runs the oracle pin tests.  Exit 0 iff every mutation is caught."""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MUTATIONS = [
    ("smooth theta weights (1/3,1/3,1/3)",
     "dst[j] = 0.25 * src[(j - 1 + mt) % mt] + 0.5 * src[j] + 0.25 * src[(j + 1) % mt];",
     "dst[j] = (1.0/3) * src[(j - 1 + mt) % mt] + (1.0/3) * src[j] + (1.0/3) * src[(j + 1) % mt];"),
    ("smooth radial weights (1/3,1/3,1/3)",
     "0.25 * ring_interp(p, &g, src, i - 1, th, zeta_k) +\n                    0.5 * src[g.igrid[i] + j] +\n"
     "                    0.25 * ring_interp(p, &g, src, i + 1, th, zeta_k);",
     "(1.0/3) * ring_interp(p, &g, src, i - 1, th, zeta_k) +\n                    (1.0/3) * src[g.igrid[i] + j] +\n"
     "                    (1.0/3) * ring_interp(p, &g, src, i + 1, th, zeta_k);"),
    ("gyro operator radius 1/Omega0",
     "double rhoG = sqrt(2.0) / p->omega0;", "double rhoG = 1.0 / p->omega0;"),
    ("gyro operator theta offset rho_G (not rho_G/r)",
     "plane_interp(p, g, in, r, th + rhoG / r, zeta_k) +", "plane_interp(p, g, in, r, th + rhoG, zeta_k) +"),
    ("seam rotation dropped in plane_value",
     "while (k >= K) { k -= K; j = (j + g->itran[i]) % mt; }", "while (k >= K) { k -= K; j = j % mt; }"),
    ("seam rotation dropped in plane_value (k < 0)",
     "while (k < 0) { k += K; j = ((j - g->itran[i]) % mt + mt) % mt; }", "while (k < 0) { k += K; }"),
    ("reflection replaced by clamping (outer)",
     "if (r > p->a1) { r = 2.0 * p->a1 - r; refl = 1; }", "if (r > p->a1) { r = p->a1; refl = 1; }"),
    ("reflection replaced by clamping (inner)",
     "if (r < p->a0) { r = 2.0 * p->a0 - r; refl = 1; }", "if (r < p->a0) { r = p->a0; refl = 1; }"),
    ("radial windows not snapped to nearest (floor)",
     "int32_t b = (int32_t)floor((rk - p->a0) / dr + 0.5);", "int32_t b = (int32_t)floor((rk - p->a0) / dr);"),
    ("radial destination: boundary ring to inner window",
     "if (r >= p->a0 + bound[k] * dr) d = k;", "if (r > p->a0 + bound[k] * dr) d = k;"),
    ("deposit gyro-point theta offset rho (not rho/r)",
     "double pdt[4] = {0.0, rho / r, 0.0, -rho / r};", "double pdt[4] = {0.0, rho, 0.0, -rho};"),
    ("field g_theta one-sided",
     "double gt = (pl[g.igrid[i] + (j + 1) % mt] - pl[g.igrid[i] + (j - 1 + mt) % mt]) / (2.0 * dth);",
     "double gt = (pl[g.igrid[i] + (j + 1) % mt] - pl[g.igrid[i] + j]) / dth;"),
    ("push: weight drive sign flipped (-v_E,r kappa)",
     "(vEr * kappa - (vpar * (B / p->R0) * gp + vdr * gr + vdt * gt / r));",
     "(-vEr * kappa - (vpar * (B / p->R0) * gp + vdr * gr + vdt * gt / r));"),
    ("push: mirror force dropped",
     "double vdot = -mu * B * B * B * r * st / (q * p->R0 * p->R0);", "double vdot = 0.0;"),
    ("push: dB/dtheta sign flipped",
     "double dBdt = B * B * (r / p->R0) * st;", "double dBdt = -B * B * (r / p->R0) * st;"),
    ("push: curvature drift without the mirror part (v_par^2 only)",
     "double Cd = (vpar * vpar + mu * B) / (p->omega0 * p->R0);", "double Cd = (vpar * vpar) / (p->omega0 * p->R0);"),
    ("push: kappa without the energy dependence",
     "double kappa = orc_prof(r) * (p->rln + (Ekin - 1.5) * p->rlt) / p->R0;",
     "double kappa = orc_prof(r) * (p->rln + p->rlt) / p->R0;"),
    ("marker density: divided by mtheta + 1 (duplicate node counted)",
     "nm[i] = s / ((double)p->mzetamax * g.mtheta[i]);", "nm[i] = s / ((double)p->mzetamax * (g.mtheta[i] + 1));"),
    ("marker density: seam plane included in the mean",
     "        for (int32_t k = 0; k < p->mzetamax; k++)\n            for (int32_t j = 0; j < g.mtheta[i]; j++)\n                s += grid",
     "        for (int32_t k = 0; k <= p->mzetamax; k++)\n            for (int32_t j = 0; j < g.mtheta[i]; j++)\n                s += grid"),
    ("field g_r neighbour rings at the same label (not physical theta)",
     "gr = (ring_interp(p, &g, pl, i + 1, th, zeta_k) -\n                          ring_interp(p, &g, pl, i - 1, th, zeta_k)) / (2.0 * dr);",
     "gr = (ring_interp(p, &g, pl, i + 1, j * TWO_PI / g.mtheta[i + 1], 0.0) -\n"
     "                          ring_interp(p, &g, pl, i - 1, j * TWO_PI / g.mtheta[i - 1], 0.0)) / (2.0 * dr);"),
]


def main():
    tests = sorted(os.path.join("tests", f) for f in os.listdir(os.path.join(ROOT, "tests"))
                   if f.startswith("test_oracle_"))
    src_rel = os.path.join("oracle", "gtcp_oracle.c")
    base = open(os.path.join(ROOT, src_rel)).read()
    missed = []
    for name, old, new in MUTATIONS:
        assert base.count(old) == 1, f"mutation anchor not found once: {name}"
        with tempfile.TemporaryDirectory() as d:
            for sub in ("oracle", "tests", "synth"):
                shutil.copytree(os.path.join(ROOT, sub), os.path.join(d, sub),
                                ignore=shutil.ignore_patterns("_build", "__pycache__"))
            shutil.copy(os.path.join(ROOT, "pytest.ini"), d)
            with open(os.path.join(d, src_rel), "w") as f:
                f.write(base.replace(old, new))
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "not gpu", "-p", "no:cacheprovider"]
                               + tests, cwd=d, capture_output=True, text=True)
            caught = r.returncode != 0
            fails = [ln for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
            print(f"{'caught' if caught else 'MISSED'}: {name}" + (f"  <- {fails[0][7:]}" if fails else ""))
            if not caught:
                missed.append(name)
    print(f"{len(MUTATIONS) - len(missed)}/{len(MUTATIONS)} mutations caught")
    return 1 if missed else 0


if __name__ == "__main__":
    sys.exit(main())
