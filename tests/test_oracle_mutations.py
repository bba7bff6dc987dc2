"""Mutation check of the oracle pins (SURVEY.md §4 'Mutation'): each plausible mistake,
injected into a copy of oracle/ovs_oracle.cpp, must make tests/test_oracle_pins.py fail."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "ovs_oracle.cpp")

MUTATIONS = {
    "splitter_rank_off_by_one": ("S[q] = T[(uint64_t)(q + 1) * s - 1];", "S[q] = T[(uint64_t)(q + 1) * s - 2 + (q == 0)];"),
    "tie_rule_le": ("return ta < tb;", "return ta <= tb;"),
    "tie_dropped": ("return ta < tb;", "return false;"),
    "unstable_bucket_sort": ("std::stable_sort(y.begin() + start[j]", "std::sort(y.begin() + start[j]"),
    "dro_sample_position": ("return (j + 1) * q + std::min(j + 1, rho) - 1;", "return (j + 1) * q + std::min(j, rho) - 1;"),
    "dro_split_side": ("return lex_less(s.key, s.tag, e.key, e.tag);", "return !lex_less(e.key, e.tag, s.key, s.tag);"),
    "sample_with_replacement": ("if (seen.insert(c).second) I.push_back(c);", "seen.insert(c); I.push_back(c);"),
    "merge_tie_higher_k": ("return A.k > B.k;", "return A.k < B.k;"),
}


@pytest.mark.parametrize("name", sorted(MUTATIONS))
def test_mutation_is_caught(name, tmp_path):
    old, new = MUTATIONS[name]
    src = open(SRC).read()
    assert src.count(old) >= 1, name
    mut = tmp_path / "mut.cpp"
    mut.write_text(src.replace(old, new))
    lib = tmp_path / "libmut.so"
    subprocess.check_call(["g++", "-O1", "-std=c++17", "-fPIC", "-shared", "-o", str(lib), str(mut)])
    env = dict(os.environ, OVS_ORACLE_LIB=str(lib))
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", os.path.join(ROOT, "tests", "test_oracle_pins.py"),
                        "-k", "not inclusion and not claim1 and not lemma1"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode != 0, f"mutation {name} survived:\n{r.stdout[-2000:]}"
