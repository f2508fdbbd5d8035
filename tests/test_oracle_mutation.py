"""Mutation check of the oracle's pins: plausible slips in oracle/geot_oracle.c
(a dropped term, a wrong sign or index, a missing reset, a transposed operand)
are compiled into throwaway copies, and the pins of tests/test_oracle.py must
FAIL on every one of them.  A mutant that no pin catches would mean the oracle
could silently carry that mistake into every parity test.  No GPU needed."""
import json
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

import oracle
import test_oracle as T

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, original text, mutated text) — each original must occur in the source
MUTANTS = [
    ("absum_no_reset", "            ab[f] = 0.0;\n", ""),
    ("absum_no_fabs", "ab[f] += fabs(v);", "ab[f] += v;"),
    ("absum_unweighted", "ab[f] += fabs(v);", "ab[f] += fabs(get_value(j->X, j->dtype, row * F + f));"),
    ("sum_no_reset", "            acc[f] = 0.0;\n", ""),
    ("sum_sign", "acc[f] += v;", "acc[f] -= v;"),
    ("max_flipped", "v > acc[f]", "v < acc[f]"),
    ("mean_count_plus_one", "acc[f] / (double)count;", "acc[f] / (double)(count + 1);"),
    ("row_transposed", "row * F + f", "f * F + row"),
    ("fused_ignores_src", "j->src_idx ? get_index(j->src_idx, j->itype, e) : e", "e"),
    ("weight_dropped", "if (j->w) v = we * v;", ""),
    ("offsets_shifted", "if (s >= 0 && s < S) counts[s] += 1;", "if (s > 0 && s < S) counts[s - 1] += 1;"),
    ("empty_not_zero", "y = 0.0; /* empty", "y = -0.0; /* empty"),
    ("bf16_truncates", "u += 0x7FFFu + lsb;", "u += 0;"),
    ("bf16_round_half_up", "u += 0x7FFFu + lsb;", "u += 0x8000u;"),
    ("partition_no_plus_one", "get_index(idx, itype, tp - 1) + 1", "get_index(idx, itype, tp - 1)"),
    ("exact_split_no_plus_one", "seg_bounds[p] = tp == 0 ? 0 : before + 1;", "seg_bounds[p] = tp == 0 ? 0 : before;"),
    ("exact_split_keys_swapped", "keys[2 * p] = before;", "keys[2 * p] = at;"),
    ("validate_unsorted_missed", "get_index(idx, itype, e - 1) > s", "get_index(idx, itype, e - 1) > s + 1"),
]


def _pins(golden):
    """The oracle's pins (no GPU), as zero-argument callables."""
    pins = []
    for name in ("W1", "W2"):
        for op in ("sum", "mean", "max"):
            pins.append(lambda name=name, op=op: T.test_worked_examples(golden, name, op))
        pins.append(lambda name=name: T.test_worked_offsets_counts_partition(golden, name))
    pins += [lambda: T.test_spec_hand_cases(golden), lambda: T.test_spec_pr_group_sums(golden)]
    for op in ("sum", "mean", "max"):
        pins.append(lambda op=op: T.test_brute_force_random_tiny(op))
        pins.append(lambda op=op: T.test_brute_force_fused_and_weighted(op))
    pins += [T.test_brute_force_bf16_inputs, T.test_identity_index_gives_X, T.test_single_segment_is_column_sum,
             T.test_fused_identity_src_equals_unfused, T.test_fused_equals_gather_then_reduce,
             T.test_weighted_is_dense_matmul, T.test_invariants_random, T.test_integer_mode_exact_long_segment,
             T.test_rounding_to_dtype_matches_torch, T.test_bf16_rne_ties_oracle, T.test_offsets_match_searchsorted,
             T.test_partition_invariants, T.test_validate_bits, T.test_empty_inputs,
             T.test_absum_single_segment_is_numpy_abs_column_sum, T.test_absum_equals_sum_for_nonnegative_inputs,
             T.test_absum_signed_brute_force, T.test_absum_fused_and_weighted,
             T.test_absum_bounds_sum_and_empty_rows_zero, T.test_partition_exact_invariants]
    pins += [lambda name=name: T.test_partition_exact_worked(golden, name) for name in ("W1", "W2")]
    return pins


@pytest.fixture(scope="module")
def golden_all():
    d = os.path.join(ROOT, "tests", "golden")
    return {n[:-5]: json.load(open(os.path.join(d, n))) for n in os.listdir(d) if n.endswith(".json")}


def test_pins_pass_on_the_real_oracle(golden_all):
    for pin in _pins(golden_all):
        pin()


_RUNNER = r"""
import json, os, sys
sys.path[:0] = [sys.argv[2], os.path.join(sys.argv[2], "tests")]
import numpy as np
import oracle, test_oracle_mutation as M
d = os.path.join(sys.argv[2], "tests", "golden")
golden = {n[:-5]: json.load(open(os.path.join(d, n))) for n in os.listdir(d) if n.endswith(".json")}
caught = 0
with oracle.use_library(sys.argv[1]):
    for pin in M._pins(golden):
        try:
            with np.errstate(all="ignore"):
                pin()
        except Exception:  # any failure of a pin counts
            caught += 1
            break  # one failing pin is enough
print("caught", caught)
"""


@pytest.mark.parametrize("name,orig,mut", MUTANTS, ids=[m[0] for m in MUTANTS])
def test_every_mutant_is_caught(name, orig, mut):
    src = open(oracle._SRC).read()
    assert orig in src, f"mutation site of {name} no longer in geot_oracle.c"
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, f"{name}.c")
        open(c, "w").write(src.replace(orig, mut))
        so = oracle.build(force=True, src=c, out=os.path.join(d, f"lib_{name}.so"))
        # in a child process: a mutant may also crash (that counts as caught)
        r = subprocess.run([sys.executable, "-c", _RUNNER, so, ROOT], capture_output=True, text=True, timeout=600)
    assert r.returncode <= 0, f"pin runner failed for {name}: {r.stderr[-2000:]}"  # < 0: killed by a signal
    if r.returncode == 0:
        n = int(r.stdout.split("caught")[-1])
        assert n > 0, f"mutant {name!r} passes every oracle pin"
