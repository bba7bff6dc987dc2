"""Pins of the CPU oracle against things other than itself (CPU-only, `-m "not gpu"`).

Each test names what it pins and the passage it follows.  A plausible mistake in the
oracle (a dropped tie-break, an off-by-one splitter rank, a wrong sample size, an unstable
bucket sort, a wrong DRO sample position) fails at least one of them; see
tests/test_oracle_mutations.py for the mutation check itself.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import ovs_inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- RNG (reading Q1)
def test_splitmix64_published_vectors(orc):
    g = gold("splitmix64_seed1234567.json")
    got = [str(orc.splitmix64(g["seed"], 0, j)) for j in range(5)]
    assert got == g["outputs"]


def test_input_generator_matches_published_vectors():
    g = gold("splitmix64_seed1234567.json")
    u = ovs_inputs.data_u64(g["seed"], 0, 5)
    assert [str(int(x)) for x in u] == g["outputs"]


def test_draw_index_closed_forms(orc):
    # floor(u n / 2^64): exact at the ends and at u = 2^63 (n/2), checked with Python big ints
    rng = np.random.default_rng(0)
    for n in [1, 2, 3, 7, 1000, 2**20, 2**27, 2**40 - 3]:
        assert orc.draw_index(0, n) == 0
        assert orc.draw_index(2**64 - 1, n) == n - 1
        assert orc.draw_index(2**63, n) == n // 2
        for u in rng.integers(0, 2**63, 20, dtype=np.uint64):
            u = int(u) * 2 + 1
            assert orc.draw_index(u, n) == (u * n) >> 64


def test_ros_sample_is_first_distinct_draws(orc):
    """I = the first ps-1 distinct indices of the stream (Q1-Q3; P:565-567 'sp-1 keys selected
    uniformly at random')."""
    for (n, p, s, seed) in [(1000, 8, 16, 3), (100, 10, 10, 5), (50, 7, 7, 1), (2**20, 64, 32, 1)]:
        I, draws = orc.ros_sample_indices(n, p, s, seed)
        assert len(I) == p * s - 1
        assert len(set(I.tolist())) == len(I)
        assert int(I.max()) < n
        seen, ref = set(), []
        for j in range(draws):
            c = (orc.splitmix64(seed, 1, j) * n) >> 64
            if c not in seen:
                seen.add(c)
                ref.append(c)
        assert ref == I.tolist()  # the last draw was the (ps-1)-th distinct one
        assert len(ref) == p * s - 1


def test_ros_sample_inclusion_frequency(orc):
    """Uniformity: each index's inclusion frequency over 1000 seeds matches
    Binomial(1000, (ps-1)/n); chi-square on the counts and a 5.5-sigma max check."""
    n, p, s, trials = 10_000, 8, 64, 1000
    m = p * s - 1
    hits = np.zeros(n, dtype=np.int64)
    for seed in range(trials):
        I, _ = orc.ros_sample_indices(n, p, s, seed + 1)
        hits[I.astype(np.int64)] += 1
    q = m / n
    mu, sd = trials * q, math.sqrt(trials * q * (1 - q))
    assert np.abs(hits - mu).max() < 5.5 * sd
    chi2 = (((hits - mu) ** 2) / (mu * (1 - q))).sum()
    # n-1 degrees of freedom: mean 9999, sd ~ 141
    assert abs(chi2 - (n - 1)) < 6 * math.sqrt(2 * (n - 1))


# ---------------------------------------------------------------- sorted output = library sort
DISTS_SMALL = ["u32_u31", "i32_uniform", "i32_gauss", "i32_few", "f64_uniform", "f64_normal", "u16key",
               "u32_const", "u32_few4"]


@pytest.mark.parametrize("dist", DISTS_SMALL)
@pytest.mark.parametrize("method", ["ros", "sqran", "dro"])
def test_output_equals_numpy_stable_sort(orc, dist, method):
    n = 20_000
    x = ovs_inputs.keys(dist, n, seed=11)
    v = ovs_inputs.index_values(n)
    if method == "ros":
        res = orc.ros_sort(x, 16, 32, seed=3, vals=v)
    elif method == "sqran":
        res = orc.sqran_literal(x, 16, 32, seed=3, vals=v)
    else:
        res = orc.dro_sort(x, 16, 2, vals=v)
    order = np.argsort(x, kind="stable")
    np.testing.assert_array_equal(res.keys, x[order])
    np.testing.assert_array_equal(res.vals, v[order])  # stability
    assert int(res.counts.sum()) == n


# ---------------------------------------------------------------- closed forms
def _rank_splitters(x, p, s):
    """Exhaustive sample (ps-1 = n): splitter q is the element of rank (q+1)s in (key, index) order."""
    order = sorted(range(len(x)), key=lambda i: (x[i], i))
    return [(x[order[(q + 1) * s - 1]], order[(q + 1) * s - 1]) for q in range(p - 1)]


@pytest.mark.parametrize("n,p,s", [(7, 2, 4), (7, 4, 2), (8, 3, 3), (5, 2, 3), (6, 7, 1)])
def test_ros_exhaustive_sample_closed_form(orc, n, p, s):
    """ps-1 = n: T is the whole input; counts = [s,...,s,s-1] (PAPER.md:569-571 ranks i*s)."""
    assert p * s - 1 == n
    multisets = [list(range(n)), [0, 1] * (n // 2) + [1] * (n % 2), [3] * n]
    for ms in multisets:
        for perm in set(itertools.permutations(ms)):
            x = np.array(perm, dtype=np.uint32)
            for method in (orc.ros_sort, orc.sqran_literal):
                res = method(x, p, s, seed=9)
                assert [(int(k), int(t)) for k, t in zip(res.split_keys, res.split_tags)] == \
                    _rank_splitters(perm, p, s)
                assert res.counts.tolist() == [s] * (p - 1) + [s - 1]
                assert res.keys.tolist() == sorted(perm)


def _baseline_sizes(n, p):
    return [n // p + (1 if k < n % p else 0) for k in range(p)]


@pytest.mark.parametrize("n,p,r", [(1000, 4, 1), (1003, 5, 2), (4096, 8, 3), (777, 3, 5), (64, 4, 1)])
def test_dro_sorted_reverse_constant_closed_forms(orc, n, p, r):
    """Sorted input: bucket j = X_j, so counts = m_j; reverse: m_{p-1-j}; constant: the tags
     order the keys, so counts = m_j (SURVEY.md §8(c) closed forms)."""
    m = _baseline_sizes(n, p)
    base = ovs_inputs.keys("i32_uniform", n, seed=5)
    srt = np.sort(base)
    for padded in (False, True):
        assert orc.dro_sort(srt, p, r, padded=padded).counts.tolist() == m
        assert orc.dro_sort(srt[::-1].copy(), p, r, padded=padded).counts.tolist() == m[::-1]
        assert orc.dro_sort(np.full(n, 7, np.int32), p, r, padded=padded).counts.tolist() == m


def test_paper_worked_examples(orc):
    ex = gold("paper_examples.json")
    for c in ex["lemma1"]:
        assert orc.lemma1_bound(c["n"], c["p"], c["r"]) == c["n_max"], c["cite"]
    d = ex["dro_regular_sample"]
    res = orc.dro_sort(np.array(d["keys"], np.uint32), d["p"], d["r"])
    assert [[int(k), int(t)] for k, t in zip(res.split_keys, res.split_tags)] == d["splitters"]
    assert res.counts.tolist() == d["counts"]
    d = ex["ros_select_splitters"]
    for f in (orc.ros_sort, orc.sqran_literal):
        res = f(np.array(d["keys"], np.uint32), d["p"], d["s"], d["seed"])
        assert [[int(k), int(t)] for k, t in zip(res.split_keys, res.split_tags)] == d["splitters"]
        assert res.counts.tolist() == d["counts"]


# ---------------------------------------------------------------- brute force on tiny inputs
def _brute_counts(x, S, p, tags):
    """Classify every element by a linear scan over the splitters with the (key, tag) order."""
    cnt = [0] * p
    for i, k in enumerate(x):
        b = sum(1 for (sk, st) in S if (sk, st) < (k, tags[i]))
        cnt[b] += 1
    return cnt


def _dro_tags(x, p):
    """DRO tag of each ORIGINAL element: start_k + position in the stably sorted X_k."""
    n = len(x)
    tags = [0] * n
    start = 0
    for m in _baseline_sizes(n, p):
        idx = sorted(range(start, start + m), key=lambda i: x[i])  # Python sort is stable
        for t, i in enumerate(idx):
            tags[i] = start + t
        start += m
    return tags


def test_brute_force_all_permutations(orc):
    """n <= 7, all permutations of distinct and duplicate multisets, p in {1,2,3}, s/r small:
    output = sorted; splitters = the (q+1)s-th smallest of the sample; counts = linear-scan
    classification of every key against the splitters."""
    for ms in ([0, 1, 2, 3, 4, 5], [1, 1, 2, 2, 2, 3], [4, 4, 4, 4, 4, 4, 4], [0, 9, 9, 1, 1, 5, 5]):
        n = len(ms)
        for perm in set(itertools.permutations(ms)):
            x = np.array(perm, dtype=np.int32)
            for p, s in [(1, 3), (2, 1), (2, 2), (3, 2), (2, 3)]:
                if p * s - 1 > n:
                    continue
                res = orc.ros_sort(x, p, s, seed=n + p + s)
                assert res.keys.tolist() == sorted(perm)
                if p > 1:
                    I, _ = orc.ros_sample_indices(n, p, s, n + p + s)
                    T = sorted((perm[i], int(i)) for i in I)
                    S = [T[(q + 1) * s - 1] for q in range(p - 1)]
                    assert [(int(k), int(t)) for k, t in zip(res.split_keys, res.split_tags)] == S
                    assert res.counts.tolist() == _brute_counts(perm, S, p, list(range(n)))
                else:
                    assert res.counts.tolist() == [n]
            for p, r in [(2, 1), (3, 1)]:
                if r * p > n // p:
                    continue
                res = orc.dro_sort(x, p, r)
                assert res.keys.tolist() == sorted(perm)
                S = [(int(k), int(t)) for k, t in zip(res.split_keys, res.split_tags)]
                assert res.counts.tolist() == _brute_counts(perm, S, p, _dro_tags(perm, p))
                assert max(res.counts) <= orc.lemma1_bound(n, p, r)


# ---------------------------------------------------------------- two independent ROS algorithms
@pytest.mark.parametrize("dist", ["u32_u31", "i32_few", "u32_few4", "u32_const", "f64_normal", "u16key"])
@pytest.mark.parametrize("p,s", [(2, 5), (16, 8), (64, 32)])
def test_sqran_literal_equals_partition_first(orc, dist, p, s):
    """Algorithm 2 as written (sort first, split by binary search, p-way merge) and the
    partition-first ROS give identical splitters, counts and stable output (Q2)."""
    n = 30_011
    x = ovs_inputs.keys(dist, n, seed=17)
    v = ovs_inputs.index_values(n)
    a = orc.ros_sort(x, p, s, seed=4, vals=v)
    b = orc.sqran_literal(x, p, s, seed=4, vals=v)
    np.testing.assert_array_equal(a.split_keys, b.split_keys)
    np.testing.assert_array_equal(a.split_tags, b.split_tags)
    np.testing.assert_array_equal(a.counts, b.counts)
    np.testing.assert_array_equal(a.keys, b.keys)
    np.testing.assert_array_equal(a.vals, b.vals)


# ---------------------------------------------------------------- Lemma 1
def test_lemma1_bound_random_instances(orc):
    """>= 500 random DRO instances: max bucket <= Lemma 1's n_max, and <= the
    proof's own sx + px - x before its last relaxation."""
    rng = np.random.default_rng(1)
    dists = ["u32_u31", "u32_few4", "u32_const", "i32_sorted", "i32_reverse", "i32_gauss", "u16key"]
    done = 0
    while done < 520:
        p = int(rng.integers(2, 24))
        r = int(rng.integers(1, 6))
        n = int(rng.integers(r * p * p, r * p * p * 8 + 2))
        dist = dists[done % len(dists)]
        x = ovs_inputs.keys(dist, n, seed=done + 100)
        for padded in (False, True):
            res = orc.dro_sort(x, p, r, padded=padded)
            mx = int(res.counts.max())
            assert mx <= orc.lemma1_bound(n, p, r)
            s = r * p
            xx = -(-(-(-n // p)) // s)
            assert mx <= s * xx + p * xx - xx
            assert mx <= orc.tight_bound(n, p, r)
        done += 1


def _dro_brute_counts(x, p, r):
    """Algorithm 1's split re-derived in plain Python from the paper (independent of the
    oracle): baseline split (Q8), stable sort of every X_k, balanced regular sample of s = rp
    segment ends with tags start_k + position (Q6, Q9), T sorted by (key, tag),
    S[q] = T[(q+1)rp - 1], counts by a linear scan in (key, tag) order."""
    n, s = len(x), r * p
    tags = _dro_tags(x, p)
    T = []
    start = 0
    for m in _baseline_sizes(n, p):
        xs = sorted(x[start:start + m])
        q, rho = m // s, m % s
        for j in range(s):
            e = (j + 1) * q + min(j + 1, rho) - 1
            T.append((xs[e], start + e))
        start += m
    T.sort()
    S = [T[(q + 1) * r * p - 1] for q in range(p - 1)]
    return _brute_counts(list(x), S, p, tags)


def test_tight_bound_attained_reading_q10(orc):
    """The tight form s*x + (p-1)(x-1) of Lemma 1's count (reading Q10; proof at P:430-476) is
    never exceeded (test_lemma1_bound_random_instances) and is attained exactly on hill-climbed
    inputs (tests/golden/dro_tight_instances.json, written by tools/gen_tight_instance.py): their
    largest bucket, re-derived by brute force from Algorithm 1, equals oracle.tight_bound, so a
    formula one too large or too small fails here or there."""
    d = gold("dro_tight_instances.json")
    assert len(d["instances"]) >= 5
    for inst in d["instances"]:
        n, p, r = inst["n"], inst["p"], inst["r"]
        x = [int(v) for v in inst["keys"]]
        assert len(x) == n
        mx = max(_dro_brute_counts(x, p, r))
        assert mx == inst["max_bucket"] == inst["tight_bound"] == orc.tight_bound(n, p, r)
        assert mx <= orc.lemma1_bound(n, p, r)
        res = orc.dro_sort(np.array(x, dtype=np.int32), p, r)
        assert int(res.counts.max()) == mx


def test_dro_parameter_errors(orc):
    x = np.arange(100, dtype=np.uint32)
    with pytest.raises(orc.OracleError) as e:
        orc.dro_sort(x, 8, 2)  # r p = 16 > floor(100/8) = 12
    assert e.value.code == orc.ESAMPLE
    with pytest.raises(orc.OracleError) as e:
        orc.ros_sort(x, 11, 10, seed=1)  # ps - 1 = 109 > 100
    assert e.value.code == orc.ESAMPLE
    with pytest.raises(orc.OracleError) as e:
        orc.ros_sort(x, 0, 10, seed=1)
    assert e.value.code == orc.EINVAL
    res = orc.ros_sort(np.zeros(0, np.uint32), 4, 2, seed=1)
    assert res.counts.tolist() == [0, 0, 0, 0]


def test_claim1_montecarlo_reported(orc):
    """Claim 1 as a statistic: n=10^5, p=16, s=ceil(lg^2 n);
    fraction of trials with any bucket > 1.5 (n-p+1)/p must be <= 5%."""
    n, p = 100_000, 16
    s = math.ceil(math.log2(n) ** 2)
    bad = 0
    for t in range(100):
        x = ovs_inputs.keys("u32", n, seed=1000 + t)
        res = orc.ros_sort(x, p, s, seed=t + 1)
        if res.counts.max() > 1.5 * (n - p + 1) / p:
            bad += 1
    assert bad <= 5


# ---------------------------------------------------------------- DRO sample positions (Q9)
def test_dro_positions_partition_into_even_segments(orc):
    """Balanced reading of P:263-265: the s = rp sample positions cut X_k into s segments whose
    sizes differ by at most one (larger first), the last position is the maximum."""
    for n, p, r in [(1000, 4, 1), (1003, 5, 2), (10_007, 7, 3), (2**16 + 5, 16, 4)]:
        for k in range(p):
            m = n // p + (1 if k < n % p else 0)
            e = orc.dro_sample_positions(n, p, r, k).astype(np.int64)
            sizes = np.diff(np.concatenate([[-1], e]))
            assert e[-1] == m - 1
            assert sizes.min() >= m // (r * p) and sizes.max() <= -(-m // (r * p))
            assert np.all(np.diff(sizes) <= 0)
            assert sizes.sum() == m


def test_dro_worked_positions(orc):
    ex = gold("paper_examples.json")
    d = ex["dro_balanced_positions"]
    res = orc.dro_sort(np.array(d["keys"], np.int32), d["p"], d["r"])
    assert [[int(k), int(t)] for k, t in zip(res.split_keys, res.split_tags)] == d["splitters"]
    assert res.counts.tolist() == d["counts"]
    d = ex["dro_padded_positions"]
    e = orc.dro_sample_positions(d["n"], d["p"], d["r"], 0, padded=True)
    s = d["p"] * d["r"]
    assert e.tolist() == [min((j + 1) * d["x"], 1000) - 1 for j in range(s - 1)] + [999]


def test_empty_input_reading_q26(orc):
    """DESIGN.md Q26: n = 0 sorts nothing; all p counts are 0 and the (undrawn) splitters are reported as 0."""
    for dt in (np.uint32, np.int32, np.float64):
        x = np.empty(0, dt)
        for res in (orc.ros_sort(x, 4, 2, 1), orc.dro_sort(x, 4, 2),
                    orc.ros_sort(x, 4, 2, 1, vals=np.empty(0, np.uint32))):
            assert len(res.keys) == 0
            assert res.counts.tolist() == [0, 0, 0, 0]
            assert not np.any(res.split_keys) and not np.any(res.split_tags)


# ---------------------------------------------------------------- 32-byte string keys (f3)
@pytest.mark.parametrize("dist", ["s32", "s32_prefix", "s32_few"])
def test_strings_sorted_like_python_bytes(orc, dist):
    """memcmp order of 32-byte keys = Python's bytes order (a library sort): the ROS,
    literal SqRan and DRO outputs equal sorted(bytes)."""
    n = 20_000
    x = ovs_inputs.keys(dist, n, seed=11)
    ref = sorted(bytes(v) for v in x)
    for res in (orc.ros_sort(x, 16, 8, 2), orc.sqran_literal(x, 16, 8, 2), orc.dro_sort(x, 16, 3)):
        assert [bytes(v) for v in res.keys] == ref
        assert int(res.counts.sum()) == n
    a, b = orc.ros_sort(x, 16, 8, 2), orc.sqran_literal(x, 16, 8, 2)
    np.testing.assert_array_equal(a.split_tags, b.split_tags)
    np.testing.assert_array_equal(a.counts, b.counts)


@pytest.mark.parametrize("n,p,s", [(7, 2, 4), (8, 3, 3), (63, 4, 16)])
def test_strings_exhaustive_sample_closed_form(orc, n, p, s):
    """ps - 1 = n: T is every string, splitter q is the string of rank (q+1)s in (bytes, index)
    order and the counts are [s, ..., s, s-1] (closed form)."""
    x = ovs_inputs.keys("s32_few", n, seed=5)
    res = orc.ros_sort(x, p, s, 3)
    order = sorted(range(n), key=lambda i: (bytes(x[i]), i))
    idx = [order[(q + 1) * s - 1] for q in range(p - 1)]
    assert res.split_tags.tolist() == idx
    assert [bytes(v) for v in res.split_keys] == [bytes(x[i]) for i in idx]
    assert res.counts.tolist() == [s] * (p - 1) + [s - 1]


@pytest.mark.parametrize("dist", ["u32_u31", "i32_few", "f64_normal", "u16key", "s32_prefix"])
@pytest.mark.parametrize("threads", [1, 3, 8])
def test_mcran_equals_sqran(orc, dist, threads):
    """McRan (Algorithm 2 with the per-sequence and per-bucket steps on t threads) gives
    the same splitters, counts and stable output as the sequential literal SqRan."""
    n = 40_003
    x = ovs_inputs.keys(dist, n, seed=23)
    v = ovs_inputs.index_values(n)
    a = orc.sqran_literal(x, 32, 16, 5, vals=v)
    b = orc.mcran_sort(x, 32, 16, 5, threads, vals=v)
    assert a.keys.tobytes() == b.keys.tobytes()
    np.testing.assert_array_equal(a.vals, b.vals)
    np.testing.assert_array_equal(a.split_tags, b.split_tags)
    np.testing.assert_array_equal(a.counts, b.counts)
