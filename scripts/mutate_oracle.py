"""Mutation check for the oracle pins: apply plausible mistakes to a temp copy of
oracle/hht_oracle.c, rebuild, run tests/test_oracle_pins.py, and require every mutant to fail.
Usage: python scripts/mutate_oracle.py   (CPU only; ~5 min)"""
import os, shutil, subprocess, sys, tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = open(os.path.join(ROOT, "oracle", "hht_oracle.c")).read()
MUTANTS = {
    "tie_on_line_counts_below": ("return F_scaled < 0;", "return F_scaled <= 0;"),
    "swap_i_j": ("const int64_t m_scaled = -scale + 2 * i;", "const int64_t m_scaled = -scale + 2 * j;"),
    "drop_ex_term": ("b_scaled + ex * m_scaled - scale * ey", "b_scaled - scale * ey"),
    "wrong_b_extent": ("-(int64_t)N * scale + 3 * (int64_t)N * j", "-(int64_t)N * scale + 2 * (int64_t)N * j"),
    "bit_order_ne_se": ("if (ne) code |= 8;", "if (ne) code |= 1;"),
    "no_beta_swap": ("if (half == ORACLE_BETA) { *ex = y; *ey = x; }", "if (0) { *ex = y; *ey = x; }"),
    "non_strict_threshold": ("if (nv > r->T) {", "if (nv >= r->T) {"),
    "quad_order_swapped": ("da[4] = {1, 0, 0, 1}", "da[4] = {0, 1, 0, 1}"),
    "vote_rule_only_zero": ("return code != 0 && code != 15;", "return code != 0;"),
    "children_use_all_points": ("visit(k, l + 1, 2 * a + da[q], 2 * c + dc[q], voters, nv);",
                                "visit(k, l + 1, 2 * a + da[q], 2 * c + dc[q], cand, ncand);"),
    # FHT circumcircle, lattice units (variant 1)
    "circle_radius_s_not_s_over_sqrt2": ("(__int128)2 * s * s * (4 * ex * ex", "(__int128)4 * s * s * (4 * ex * ex"),
    "circle_centre_at_sw_corner": ("const int64_t i2 = 2 * a * s + s, j2 = 2 * c * s + s;",
                                   "const int64_t i2 = 2 * a * s, j2 = 2 * c * s;"),
    "circle_drop_ex_term": ("- 2 * ex * i2 - 3 * (int64_t)N * j2", "- 3 * (int64_t)N * j2"),
    # FHT circumcircle, (m, b) units (variant 2)
    "circle_mb_drop_width": ("(4 + 9 * (__int128)N * N)", "(9 * (__int128)N * N)"),
    "circle_mb_no_slope_norm": ("(__int128)(1 + ex * ex)", "(__int128)(1 + ex)"),
    "circle_mb_centre_m_at_corner": ("const __int128 m2 = -sc + 2 * (__int128)i2;",
                                     "const __int128 m2 = -sc + 2 * (__int128)(i2 - s);"),
}
ok = True
for name, (a, b) in MUTANTS.items():
    assert a in SRC, name
    tmp = tempfile.mkdtemp()
    shutil.copytree(os.path.join(ROOT, "oracle"), os.path.join(tmp, "oracle"))
    for f in ("tests", "paper_1007_0547_b200"):
        shutil.copytree(os.path.join(ROOT, f), os.path.join(tmp, f),
                        ignore=shutil.ignore_patterns("*.so", "__pycache__"))
    p = os.path.join(tmp, "oracle", "hht_oracle.c")
    open(p, "w").write(SRC.replace(a, b, 1))   # first occurrence only
    so = os.path.join(tmp, "oracle", "liboracle.so")
    if os.path.exists(so):
        os.remove(so)
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "tests/test_oracle_pins.py"],
                       cwd=tmp, capture_output=True, text=True)
    killed = r.returncode == 1 and " failed" in r.stdout   # a failing pin, not a build/collection error
    ok &= killed
    print(f"{name:28s} {'killed' if killed else 'SURVIVED'}")
    shutil.rmtree(tmp)
sys.exit(0 if ok else 1)
