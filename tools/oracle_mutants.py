#!/usr/bin/env python
"""Mutation check of the oracle's pins: apply each plausible slip to a scratch copy of
oracle/cc_oracle.c and run the CPU pins (tests/test_oracle_*.py) against it.  Every mutant must
be killed (at least one failing test).  Usage: python tools/oracle_mutants.py [name ...]"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# name: (original text, mutated text) -- each a single plausible mistake
MUTANTS = {
    "band_4xi": ("double s = 2.0 * sqrt(3.0) * xi;", "double s = 4.0 * xi;"),
    "band_sqrt3xi": ("double s = 2.0 * sqrt(3.0) * xi;", "double s = sqrt(3.0) * xi;"),
    "mu_sqrt3": ("t->mu = 2.0 * sqrt(3.0) * t->eps_q;", "t->mu = sqrt(3.0) * t->eps_q;"),
    "eps_q_2m": ("t->eps_q = 2.0 * xi / (ldexp(1.0, c->m) - 1.0);", "t->eps_q = 2.0 * xi / ldexp(1.0, c->m);"),
    "xip_m1": ("t->xip_f = rd32_sum(xi * (1.0 - ldexp(1.0, -c->m)), 0.0);",
               "t->xip_f = rd32_sum(xi * (1.0 - ldexp(1.0, 1 - c->m)), 0.0);"),
    "adam_eps_in_sqrt": ("float den = sqrtf(vh) + eps;", "float den = sqrtf(vh + eps);"),
    "adam_no_bc1": ("float mh = *m / bc1;", "float mh = *m;"),
    "adam_no_bc2": ("float vh = *v / bc2;", "float vh = *v;"),
    "adam_beta_swap": ("*m = b1 * *m + omb1 * g[q];", "*m = b2 * *m + omb2 * g[q];"),
    "broken_ge": ("if (d > t->c_b) { *e = d - t->c_b; return 1; }", "if (d >= t->c_b) { *e = d - t->c_b; return 1; }"),
    "false_lt": ("if (d <= t->c_f) { *e = d - t->c_f; return 1; }", "if (d < t->c_f) { *e = d - t->c_f; return 1; }"),
    "grad_sign": ("g[0] = g[0] + k * r[0];", "g[0] = g[0] - k * r[0];"),
    "grad_no2": ("float two_e = 2.0f * e;", "float two_e = e;"),
    "coincident_dir": ("g[0] = g[0] + (i_is_lower ? two_e : -two_e);", "g[0] = g[0] + (i_is_lower ? -two_e : two_e);"),
    "band_lower_closed": ("if (t.lo2 < d2_ && d2_ <= t.hi2) {", "if (t.lo2 <= d2_ && d2_ <= t.hi2) {"),
    "link_strict": ("uint8_t f_ = (uint8_t)((d2_ <= t.b2 ? 1 : 0)", "uint8_t f_ = (uint8_t)((d2_ < t.b2 ? 1 : 0)"),
    "no_min_image": ("if (d > t->hLf) d = d - t->Lf;", "if (d > t->Lf) d = d - t->Lf;"),
    "proj_plain_round": ("box[6 * e + 2 * q + 1] = rd32_sum((double)o[q], (double)t.xip_f);",
                         "box[6 * e + 2 * q + 1] = (float)((double)o[q] + (double)t.xip_f);"),
    "proj_around_dec": ("const float o[3] = {x[i], y[i], z[i]};", "const float o[3] = {xh[i], yh[i], zh[i]};"),
    "stop_rounded_sum": ("const int loss_le = xsum_cmp(&loss, c->eps_loss) <= 0;\n            if (c->stop_mode == 0",
                         "const int loss_le = xsum_value(&loss) <= c->eps_loss;\n            if (c->stop_mode == 0"),
    "stop_after_update": ("if (c->stop_mode == 0 && act == 0) break;", "if (c->stop_mode == 0 && act == 0 && t_it > 1) break;"),
    "fof_strict": ("if (dist2(x[i], y[i], z[i], x[j], y[j], z[j], &t, per) <= t.b2) uf_union(par, sz, i, j);",
                   "if (dist2(x[i], y[i], z[i], x[j], y[j], z[j], &t, per) < t.b2) uf_union(par, sz, i, j);"),
    "edit_step": ("return ldexp((double)(float)c->xi, 1 - c->m);", "return ldexp((double)(float)c->xi, -c->m);"),
    "edit_flag_order": ("flags[k / 8] |= (uint8_t)(1u << (k % 8));", "flags[k / 8] |= (uint8_t)(0x80u >> (k % 8));"),
}


def run(name, old, new):
    src = open(os.path.join(ROOT, "oracle", "cc_oracle.c")).read()
    assert src.count(old) >= 1, f"{name}: pattern not found"
    with tempfile.TemporaryDirectory(prefix=f"mut_{name}_") as d:
        for sub in ("oracle", "tests", "synth"):
            shutil.copytree(os.path.join(ROOT, sub), os.path.join(d, sub),
                            ignore=shutil.ignore_patterns("*.so", "__pycache__"))
        shutil.copy(os.path.join(ROOT, "pytest.ini"), d)
        with open(os.path.join(d, "oracle", "cc_oracle.c"), "w") as f:
            f.write(src.replace(old, new, 1))
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider"] +
                           sorted(os.path.join("tests", t) for t in os.listdir(os.path.join(d, "tests"))
                                  if t.startswith("test_oracle_")),
                           cwd=d, capture_output=True, text=True, timeout=1800)
        killed = r.returncode != 0
        first = next((ln for ln in r.stdout.splitlines() if ln.startswith("FAILED")), "")
        return killed, first


def main():
    names = sys.argv[1:] or list(MUTANTS)
    alive = []
    for n in names:
        killed, first = run(n, *MUTANTS[n])
        print(f"{n:22s} {'killed' if killed else 'ALIVE'}  {first[:110]}", flush=True)
        if not killed:
            alive.append(n)
    print(f"{len(names) - len(alive)}/{len(names)} mutants killed" + (f"; alive: {alive}" if alive else ""))
    return 1 if alive else 0


if __name__ == "__main__":
    sys.exit(main())
