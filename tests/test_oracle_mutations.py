"""Mutation check of the oracle's pins: each case applies ONE plausible one-line mistake to
oracle/sae_oracle.cpp (a dropped term, a wrong index, a wrong queue, a missing step),
builds the mutated oracle into a temporary library and runs the pins against it with
ORACLE_LIB; the named pin must fail.  A pin table row is only as good as the mistakes it
catches (DESIGN.md §2 lists the pins and the mutations each one kills)."""
import os
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "sae_oracle.cpp")

# (id, function mutated, exact original text, mutated text, pin test that must fail)
MUTATIONS = [
    ("ghost_no_expiry", "ghost_push",
     "if (it != R.gmap.end() && it->second.second == os) R.gmap.erase(it);",
     "if (false) R.gmap.erase(it);", "test_golden_trace[ghost_fifo]"),
    ("ghost_slot_index", "ghost_push",
     "size_t slot = (size_t)(s % R.cfg.ghost_capacity);",
     "size_t slot = (size_t)(s % (R.cfg.ghost_capacity - 1));", "test_golden_trace[ghost_fifo]"),
    ("mae_current_tau", "orc_admit O9",
     "if (g->second.first < 5) R.ts_mae[g->second.first]++;",
     "if (tau[j] < 5) R.ts_mae[tau[j]]++;", "test_golden_trace[ghost_fifo]"),
    ("ts_ev_skips_ef", "evict_one",
     "if (b.tau < 5) R.ts_ev[b.tau]++;",
     "if (b.tau < 5 && b.q != Q_EF) R.ts_ev[b.tau]++;", "test_golden_trace[ghost_fifo]"),
    ("qe_counts_ef", "evict_one",
     "if (b.q != Q_EF) R.qe[b.q - 1]++;",
     "R.qe[b.q == Q_EF ? 0 : b.q - 1]++;", "test_golden_trace[ghost_fifo]"),
    ("no_k_chunking", "evict_k",
     "uint64_t m = std::min(remaining, to_cross);",
     "uint64_t m = remaining;", "test_golden_trace[k_crossing]"),
    ("k_trigger_offset", "evict_one",
     "if (R.E % R.cfg.K == 0) learn(R);",
     "if (R.E % R.cfg.K == 1) learn(R);", "test_golden_trace[k_crossing]"),
    ("qh_new_queue", "orc_admit O7",
     "R.qh[b.q - 1]++;",
     "R.qh[(q[j] == Q_EF ? Q_CHAT : q[j]) - 1]++;", "test_golden_trace[hit_statistics]"),
    ("ts_hit_old_tau", "orc_admit O7",
     "if (tau[j] < 5) R.ts_hit[tau[j]]++;",
     "if (b.tau < 5) R.ts_hit[b.tau]++;", "test_golden_trace[hit_statistics]"),
    ("ts_acc_prompt_types_only", "orc_admit O6",
     "if (tau[j] < 5) R.ts_acc[tau[j]]++;",
     "if (tau[j] < 5 && j > 0) R.ts_acc[tau[j]]++;", "test_golden_trace[hit_statistics]"),
    ("bin_denominator", "orc_admit O6/O7",
     "return std::min<uint32_t>(cfg.n_bins - 1, (cfg.n_bins * j) / omax);",
     "return std::min<uint32_t>(cfg.n_bins - 1, (cfg.n_bins * j) / (omax + 1));",
     "test_golden_trace[hit_statistics]"),
    ("interval_no_eps_clamp", "orc_admit O7",
     "iv.push_back(ln(dt));",
     "iv.push_back(ln(now - b.last));", "test_golden_trace[hit_statistics]"),
    ("untempl_ignores_mt", "orc_admit O4",
     "bool untempl = !mt && spb == 0;",
     "bool untempl = spb == 0;", "test_golden_trace[hit_statistics]"),
    ("orphan_not_refreshed", "orc_admit O8",
     "    b.last = now;\n    b.q = q[j]; b.tau = tau[j]; b.ob = j; b.omax = omax;\n  }\n  // O9",
     "    b.q = q[j]; b.tau = tau[j]; b.ob = j; b.omax = omax;\n  }\n  // O9",
     "test_golden_trace[orphan_refresh]"),
    ("relative_pow_times_T", "learn_queues (relative)",
     "double pw = (x == 0.0) ? 0.0 : exp_(ln(x) / p.T);",
     "double pw = (x == 0.0) ? 0.0 : exp_(ln(x) * p.T);", "test_golden_trace[relative_rule]"),
    ("relative_mean_over_all", "learn_queues (relative)",
     "double Ebar = sum / (double)nd;",
     "double Ebar = sum / 3.0;", "test_golden_trace[relative_rule_undefined]"),
    ("alpha_index", "score",
     "int qi = b.q - 1;",
     "int qi = b.q % 3;", "test_golden_trace[route_alpha]"),
    ("w_by_queue", "score",
     "return ((R.par.alpha[qi] * R.par.w[b.tau]) * p) / dt;",
     "return ((R.par.alpha[qi] * R.par.w[b.q]) * p) / dt;", "test_golden_trace[route_w]"),
    ("mu_index", "score",
     "p = survival(dt, R.par.mu[qi], R.par.sigma[qi], R.cfg.z_cut);",
     "p = survival(dt, R.par.mu[0], R.par.sigma[qi], R.cfg.z_cut);", "test_golden_trace[route_mu]"),
    ("sigma_index", "score",
     "p = survival(dt, R.par.mu[qi], R.par.sigma[qi], R.cfg.z_cut);",
     "p = survival(dt, R.par.mu[qi], R.par.sigma[0], R.cfg.z_cut);", "test_golden_trace[route_sigma]"),
    ("omax_is_np", "orc_admit O4 (A8)",
     "uint32_t omax = std::max<uint32_t>(np - 1, 1);",
     "uint32_t omax = std::max<uint32_t>(np, 1);", "test_golden_trace[route_position]"),
    ("classify_chat_needs_mt", "classify",
     "if (mt || cid) return Q_CHAT;",
     "if (mt) return Q_CHAT;", "test_classify_full_truth_table"),
    ("classify_agent_after_chat", "classify",
     "if (mt && ag) return Q_AGENT;\n  if (mt || cid) return Q_CHAT;",
     "if (mt || cid) return Q_CHAT;\n  if (mt && ag) return Q_AGENT;", "test_classify_full_truth_table"),
    ("classify_sys_not_struct", "classify",
     "if (is_struct || tau == T_SYS) return Q_STRUCT;",
     "if (is_struct) return Q_STRUCT;", "test_classify_full_truth_table"),
]


def _run(case, tmp):
    mid, _, old, new, pin = case
    src = open(SRC).read()
    assert src.count(old) == 1, "mutation %s: original text not found exactly once" % mid
    path = os.path.join(tmp, mid + ".cpp")
    open(path, "w").write(src.replace(old, new))
    so = os.path.join(tmp, mid + ".so")
    sys.path.insert(0, ROOT)
    from oracle.oracle import CXXFLAGS
    subprocess.check_call(["g++", *CXXFLAGS, "-o", so, path])
    env = dict(os.environ, ORACLE_LIB=so, PYTHONDONTWRITEBYTECODE="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_oracle_golden.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    return mid, pin, r.returncode, r.stdout


def test_every_mutation_is_caught():
    src = open(SRC).read()
    for mid, _, old, _, _ in MUTATIONS:
        assert src.count(old) == 1, (mid, "original text must occur exactly once")
    with tempfile.TemporaryDirectory() as tmp:
        with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
            results = list(ex.map(lambda c: _run(c, tmp), MUTATIONS))
    missed = []
    for mid, pin, rc, out in results:
        if rc == 0 or ("FAILED tests/test_oracle_golden.py::" + pin) not in out:
            missed.append((mid, pin, rc, out[-600:]))
    assert not missed, missed
