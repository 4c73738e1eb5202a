"""Mutation check of the oracle pins (VERDICT r1 "Next round" item 1): apply one plausible slip at a time to
a COPY of oracle/oracle.cpp, build it to a temporary library, run the pin tests that should catch it with
ORACLE_LIB pointing at the mutant, and record whether they went red.  The tree's oracle.cpp is never
modified.  usage: python tools/mutate_oracle.py [out.txt]   (prints one line per mutant; exit 1 if any survives)
"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "oracle.cpp")
T_CTL = "tests/test_oracle_control.py"
T_ARG = "tests/test_oracle_argmin.py"

# (name, rule, [(old, new), ...], pytest selectors)
MUTANTS = [
    ("batch: double and halve swapped", "M16(ii)",
     [("? std::min(32u, 2 * I.B) : std::max(1u, I.B / 2)", "? std::max(1u, I.B / 2) : std::min(32u, 2 * I.B)")],
     [T_CTL + "::test_batch_control_sequence"]),
    ("batch: calm halves B instead of reset", "M16(ii)",
     [("else if (calm) nb = I.B_default;", "else if (calm) nb = std::max(1u, I.B / 2);")],
     [T_CTL + "::test_batch_control_sequence"]),
    ("batch: window p99 rank floor(0.99 n)", "M16(ii) / R-SLO",
     [("uint32_t k99 = (uint32_t)((99ull * w_n + 99) / 100);", "uint32_t k99 = (uint32_t)((99ull * w_n) / 100);")],
     [T_CTL + "::test_batch_control_sequence"]),
    ("batch: Q threshold ignores q_hi", "M16(ii)",
     [("(I.w_qint > (uint64_t)cand.q_hi * W)", "(I.w_qint > (uint64_t)W)")],
     [T_CTL + "::test_batch_control_limits"]),
    ("batch: dwell ignored", "M16(ii)",
     [("if (nb != I.B && q - I.q_last_B >= (int64_t)cand.dwell)", "if (nb != I.B)")],
     [T_CTL + "::test_batch_control_dwell_two"]),
    ("select: SMALL and LARGE swapped", "M16(iii)",
     [("if (b1000 >= (u128)cand.hi * W || viol) ns = small_i;", "if (b1000 >= (u128)cand.hi * W || viol) ns = large_i;"),
      ("else if (b1000 <= (u128)cand.lo * W && !viol) ns = large_i;",
       "else if (b1000 <= (u128)cand.lo * W && !viol) ns = small_i;")],
     [T_CTL + "::test_model_selection_by_busy"]),
    ("select: busy of the LARGE instance, not the selected one", "M16(iii)",
     [("u128 b1000 = (u128)inst[cur].w_busy * 1000u;", "u128 b1000 = (u128)inst[large_i].w_busy * 1000u;")],
     [T_CTL + "::test_model_selection_by_busy"]),
    ("select: violation ignored", "M16(iii)",
     [("if (b1000 >= (u128)cand.hi * W || viol) ns = small_i;", "if (b1000 >= (u128)cand.hi * W) ns = small_i;")],
     [T_CTL + "::test_model_selection_by_violation"]),
    ("select: hi bound exclusive", "M16(iii)",
     [("if (b1000 >= (u128)cand.hi * W || viol)", "if (b1000 > (u128)cand.hi * W || viol)")],
     [T_CTL + "::test_model_selection_by_busy"]),
    ("RR: counter pre-incremented", "M11",
     [("return f + (rr[role]++ % n);", "return f + (++rr[role] % n);")],
     [T_CTL + "::test_rr_rotates_per_opening"]),
    ("RR: one counter for every role", "M11",
     [("return f + (rr[role]++ % n);", "return f + (rr[0]++ % n);")],
     [T_CTL + "::test_rr_counter_is_per_role"]),
    ("route override also replaces FIXED", "M11",
     [("if ((pol == ORC_JSQ || pol == ORC_RR) && cand.route_override != ORC_ROUTE_NONE)",
       "if (cand.route_override != ORC_ROUTE_NONE)")],
     [T_CTL + "::test_route_override"]),
    ("LOAD metric: busy time used", "M16(i) LOAD",
     [("u += cand.metric_load ? I.w_lint : I.w_busy;", "u += I.w_busy;")],
     [T_CTL + "::test_load_metric_band"]),
    ("LOAD metric: in-flight messages not counted", "M15 LOAD",
     [("I.w_lint += (uint64_t)I.load() * dt;", "I.w_lint += (uint64_t)(I.load() - I.inflight) * dt;")],
     [T_CTL + "::test_load_metric_band"]),
    ("truncation: an event at max_ticks is not processed", "M1 / M12",
     [("if (G.max_ticks && t_next > G.max_ticks)", "if (G.max_ticks && t_next >= G.max_ticks)")],
     [T_CTL + "::test_truncation_ht1"]),
    ("overflow: inbox capacity off by one", "M14",
     [("if (inst[dest].inbox.size() >= P.roles[0].inbox_cap)", "if (inst[dest].inbox.size() > P.roles[0].inbox_cap)")],
     [T_CTL + "::test_overflow_inbox"]),
    ("overflow: wait capacity off by one", "M14",
     [("if (I.wait.size() >= R.wait_cap)", "if (I.wait.size() > R.wait_cap)")],
     [T_CTL + "::test_overflow_wait_and_flight"]),
    ("sum_ff over saturated values", "M19 / R-SAT",
     [("S.sum_ff += ffl;", "S.sum_ff += f32;")],
     [T_CTL + "::test_saturated_latencies"]),
    ("saturation count strict", "M18 / R-SAT",
     [("if (e2e >= 0xFFFFFFFFull || ffl >= 0xFFFFFFFFull) S.n_saturated++;",
       "if (e2e > 0xFFFFFFFFull || ffl > 0xFFFFFFFFull) S.n_saturated++;")],
     [T_CTL + "::test_saturated_latencies"]),
    ("argmin: goodput ranked by completions", "M20 / R-KEYS",
     [("uint64_t na = obj == ORC_OBJ_GOODPUT ? a.good : a.completed;", "uint64_t na = a.completed;"),
      ("uint64_t nb = obj == ORC_OBJ_GOODPUT ? b.good : b.completed;", "uint64_t nb = b.completed;")],
     [T_ARG + "::test_group_argmin_brute_force_random"]),
    ("argmin: large-model items minimised", "M20 / R-KEYS",
     [("if (a.large != b.large) return a.large > b.large;", "if (a.large != b.large) return a.large < b.large;")],
     [T_ARG + "::test_group_argmin_brute_force_random"]),
    ("argmin: infeasible ranked by p99 before drops", "M20 / R-KEYS",
     [("if (a.dropped != b.dropped) return a.dropped < b.dropped;\n      }",
       "if (a.p != b.p) return a.p < b.p;\n      }")],
     [T_ARG + "::test_group_argmin_brute_force_random"]),
    ("argmin: latency ranks drops after the percentile", "M20 / R-KEYS",
     [("      if (a.dropped != b.dropped) return a.dropped < b.dropped;\n      if (a.p != b.p) return a.p < b.p;",
       "      if (a.p != b.p) return a.p < b.p;\n      if (a.dropped != b.dropped) return a.dropped < b.dropped;")],
     [T_ARG + "::test_group_argmin_brute_force_random"]),
    ("argmin: zero makespan ties every rate", "R-RATE0",
     [("  if (ma == 0) { na = 0; ma = 1; }\n  if (mb == 0) { nb = 0; mb = 1; }\n", "")],
     [T_ARG + "::test_group_argmin_brute_force_random"]),
    ("rows: pooled percentile at the bin's upper edge", "M18 / M20 pooled rows",
     [("if (cum >= k) return bin_lo(b);", "if (cum >= k) return bin_lo(b + 1);")],
     [T_ARG + "::test_pooled_percentile_brute_force", T_ARG + "::test_row_argmin_pooled_records"]),
    ("rows: pooled percentile rank floor(q n)", "M18 pooled rows",
     [("const uint64_t k = (num * n + 99) / 100;\n  uint64_t cum = 0;", "const uint64_t k = (num * n) / 100 + 1;\n  uint64_t cum = 0;")],
     [T_ARG + "::test_pooled_percentile_brute_force"]),
    ("cell series: integral of the JSQ load instead of Q", "M15 / R-CSER",
     [("e[0] += I.w_qint;", "e[0] += I.w_lint;")],
     ["tests/test_oracle_cellseries.py::test_ht9_cell_series_hand_values"]),
    ("rows: bad = any overflow (truncated ignored)", "M20 / R-KEYS",
     [("k.bad = q[1] != q[0];", "k.bad = q[2] != 0;")],
     [T_ARG + "::test_row_argmin_brute_force_random"]),
]


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else None
    src = open(SRC).read()
    tmp = tempfile.mkdtemp()
    lines, survived = [], 0
    for name, rule, reps, tests in MUTANTS:
        m = src
        for old, new in reps:
            assert m.count(old) == 1, (name, old)
            m = m.replace(old, new)
        cpp = os.path.join(tmp, "oracle_mut.cpp")
        lib = os.path.join(tmp, "liboracle_mut_%d.so" % len(lines))
        open(cpp, "w").write(m)
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-I", os.path.join(ROOT, "oracle"),
                               "-o", lib, cpp, "-lpthread"])
        env = dict(os.environ, ORACLE_LIB=lib)
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider"] + tests, cwd=ROOT,
                           env=env, capture_output=True, text=True)
        killed = r.returncode != 0
        survived += not killed
        tail = [x for x in r.stdout.splitlines() if x.strip()][-1:] or [""]
        lines.append("%-8s %-50s %-22s %s | %s" % ("KILLED" if killed else "SURVIVED", name, rule,
                                                  " ".join(t.split("::")[-1] for t in tests), tail[0]))
        print(lines[-1], flush=True)
    # the unmutated oracle passes the same tests
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", T_CTL, T_ARG], cwd=ROOT,
                       capture_output=True, text=True)
    lines.append("baseline (unmutated oracle): %s" % [x for x in r.stdout.splitlines() if x.strip()][-1])
    print(lines[-1])
    if out:
        open(out, "w").write("\n".join(lines) + "\n")
    return 1 if survived or r.returncode else 0


if __name__ == "__main__":
    sys.exit(main())
