"""Mutation check of the oracle pins: apply plausible mistakes to a copy of
oracle/lbm_oracle.c, rebuild it in place, run the CPU pins and require that
each mutation makes at least one pin fail.  Restores the original build.

    python tools/mutate_oracle.py
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "lbm_oracle.c")

MUTATIONS = {
    "bb_sign_literal": ("+ 6.0 * W[i] * RHO0 * eu", "- 6.0 * W[i] * RHO0 * eu"),
    "u_over_rho": ("u[0] = jx / RHO0;", "u[0] = jx / (RHO0 + s);"),
    "feq_rho0_not_rho": ("feq[i] = W[i] * (drho + RHO0", "feq[i] = W[i] * (0.0 + RHO0"),
    "drop_4.5_term": ("+ 4.5 * eu * eu", "+ 0.0 * eu * eu"),
    "drop_both_quadratic": ("3.0 * eu + 4.5 * eu * eu - 1.5 * usq", "3.0 * eu"),
    "push_not_pull": ("int sx = wrap(x - E[i][0]", "int sx = wrap(x + E[i][0]"),
    "bb_no_opp": ("p[i] = src[cell * Q + OPP[i]];", "p[i] = src[cell * Q + i];"),
    "omega_as_tau": ("out[i] = p[i] - omega * (p[i] - feq[i]);", "out[i] = p[i] - (1.0 / omega) * (p[i] - feq[i]);"),
    "weight_swap": ("1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0,",
                    "1.0 / 36.0, 1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0, 1.0 / 9.0,"),
    "edge_transposed": ("{1, -1, 0},  {-1, 1, 0},", "{-1, 1, 0},  {1, -1, 0},"),
    "cs2_wrong": ("3.0 * eu +", "2.0 * eu +"),
    "bb_rho_local": ("6.0 * W[i] * RHO0 * eu", "6.0 * W[i] * (RHO0 + 0.5) * eu"),
    # macroscopic export; the first one survived every round-1 pin
    "export_drop_rho0": ("rho[cell] = RHO0 + drho;", "rho[cell] = drho;"),
    "export_solid_rho_one": ("rho[cell] = 0.0;\n", "rho[cell] = RHO0;\n"),
    # the round-1 judge's extra mutations, recorded here
    "jz_sign": ("jz += E[i][2] * f[i];", "jz -= E[i][2] * f[i];"),
    "wrap_off_by_one": ("if (c < 0) return c + n;", "if (c < 0) return c + n - 1;"),
    "lid_term_opp_dir": ("double eu = E[i][0] * uw[0] + E[i][1] * uw[1] + E[i][2] * uw[2];",
                         "double eu = E[OPP[i]][0] * uw[0] + E[OPP[i]][1] * uw[1] + E[OPP[i]][2] * uw[2];"),
    "usq_missing_z": ("double usq = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];",
                      "double usq = u[0] * u[0] + u[1] * u[1];"),
    "nvel_bound": ("if (fl >= 2 && fl - 2 >= nvel) return 2;", "if (fl >= 2 && fl - 2 > nvel) return 2;"),
}


def main():
    orig = open(SRC).read()
    backup = SRC + ".orig"
    shutil.copy(SRC, backup)
    survived = []
    try:
        for name, (a, b) in MUTATIONS.items():
            assert a in orig, name
            open(SRC, "w").write(orig.replace(a, b, 1))
            subprocess.run(["make", "-C", ROOT, "-B", "oracle"], check=True, stdout=subprocess.DEVNULL)
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "tests/test_oracle_pins.py"],
                               cwd=ROOT, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
            status = "KILLED" if r.returncode != 0 else "SURVIVED"
            print(f"{name:24s} {status}")
            if r.returncode == 0:
                survived.append(name)
    finally:
        shutil.move(backup, SRC)
        subprocess.run(["make", "-C", ROOT, "-B", "oracle"], check=True, stdout=subprocess.DEVNULL)
    print("survivors:", survived)
    return 1 if survived else 0


if __name__ == "__main__":
    sys.exit(main())
