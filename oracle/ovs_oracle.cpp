// ovs_oracle.cpp — plain, slow, single-threaded CPU oracle of the paper's oversampling
// sorts (arXiv 1608.08648).  TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load this library.  It shares no
// code, header, table or constant generator with the CUDA path (paper_1608_08648_b200/csrc).
//
// Citations: "P:n" = /root/reference/PAPER.md line n (LaTeX source of the paper);
// "Q<k>" = a reading of an ambiguous passage, listed in DESIGN.md §3.
//
// What is computed:
//   ROS  — random oversampling, partition-first ("traditional", P:86-91, P:120-127,
//          P:615-620): sample ps-1 keys uniformly at random, sort the sample, splitters are
//          the (i*s)-th smallest, every key is binary-searched over the p-1
//          splitters with the duplicate tie-break of P:533-537, the p sequences
//          are formed and each is sorted; the concatenation is the output.
//   SqRan literal — Algorithm 2 as written: cross-check of ROS.
//   DRO  — Algorithm 1 (SqDet) as written with regular oversampling.
//
// Parity pins of every function live in tests/test_oracle_*.py (none of them is a re-typing
// of the formulas here): SplitMix64 published vectors, numpy stable sort, brute force over
// all permutations of tiny inputs, closed forms (exhaustive sample, sorted/reverse/constant
// DRO inputs), Lemma 1, and agreement of the two independent ROS algorithms.
#include <algorithm>
#include <atomic>
#include <thread>
#include <cstdint>
#include <cstring>
#include <queue>
#include <unordered_set>
#include <vector>
#ifdef EINVAL  // <thread> pulls in errno.h; the oracle's status codes are its own
#undef EINVAL
#endif

namespace {

enum { OK = 0, EINVAL = 1, EDTYPE = 2, ESAMPLE = 3 };
enum { DT_U32 = 0, DT_I32 = 1, DT_F64 = 2, DT_S32 = 3 };

// 32-byte string keys in memcmp order: the paper's own workload, "keys ... random strings of
// 32 bytes" compared as byte strings.  Every algorithm below is
// written against operator< only, so the same code sorts them.
struct S32 { unsigned char b[32]; };
inline bool operator<(const S32& a, const S32& b) { return std::memcmp(a.b, b.b, 32) < 0; }
enum { DRO_PADDED_POSITIONS = 1u };

// ---- counter-based random stream (reading Q1) -------------------------------------------
// H(seed, stream, j) = the (stream*2^40 + j)-th output of SplitMix64 seeded with `seed`
// (Steele, Lea, Flood 2014): state advances by GAMMA, output = mix64(state).
constexpr uint64_t GAMMA = 0x9e3779b97f4a7c15ULL;
constexpr uint64_t STREAM_SAMPLE = 1;

uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
uint64_t H(uint64_t seed, uint64_t stream, uint64_t j) {
    return mix64(seed + GAMMA * ((stream << 40) + j + 1));
}
// index in [0, n): floor(u * n / 2^64), exact 128-bit product
uint64_t draw_index(uint64_t u, uint64_t n) {
    return (uint64_t)(((unsigned __int128)u * (unsigned __int128)n) >> 64);
}

// ---- tagged records and the duplicate tie-break (reading Q5/Q6) -------------
template <class K> struct Rec { K key; uint64_t tag; };

// strict lexicographic (key, tag) order: "first a comparison of the two keys, and if the
// comparison is not resolved that way the use of sequence identifiers or array indexes"
template <class K> bool lex_less(K ka, uint64_t ta, K kb, uint64_t tb) {
    if (ka < kb) return true;
    if (kb < ka) return false;
    return ta < tb;
}
template <class K> bool rec_less(const Rec<K>& a, const Rec<K>& b) {
    return lex_less(a.key, a.tag, b.key, b.tag);
}

// element of the input carried through the algorithms
template <class K> struct Item { K key; uint32_t val; uint64_t tag; };

// ---- R1: the ROS sample index set I (readings Q1-Q3) --------------------------
// I = the first ps-1 DISTINCT values of c_j = floor(H(seed,1,j) * n / 2^64), j = 0,1,2,...
// returned in draw order.
std::vector<uint64_t> ros_sample_indices(uint64_t n, uint64_t m, uint64_t seed, uint64_t* draws) {
    std::vector<uint64_t> I;
    I.reserve(m);
    std::unordered_set<uint64_t> seen;
    seen.reserve(2 * m + 16);
    uint64_t j = 0;
    while (I.size() < m) {
        uint64_t c = draw_index(H(seed, STREAM_SAMPLE, j), n);
        ++j;
        if (seen.insert(c).second) I.push_back(c);
    }
    if (draws) *draws = j;
    return I;
}

template <class K>
void write_report(const std::vector<Rec<K>>& S, K* sk, uint64_t* st) {
    for (size_t q = 0; q < S.size(); ++q) {
        if (sk) sk[q] = S[q].key;
        if (st) st[q] = S[q].tag;
    }
}

// plain stable sort by key of (key, val) — the p == 1 degenerate case
template <class K>
void plain_stable_sort(const K* x, const uint32_t* v, uint64_t n, K* out, uint32_t* outv) {
    std::vector<Item<K>> a(n);
    for (uint64_t i = 0; i < n; ++i) a[i] = {x[i], v ? v[i] : 0u, i};
    std::stable_sort(a.begin(), a.end(), [](const Item<K>& A, const Item<K>& B) { return A.key < B.key; });
    for (uint64_t i = 0; i < n; ++i) {
        out[i] = a[i].key;
        if (outv) outv[i] = a[i].val;
    }
}

// ---- ROS, partition-first (R0-R8 of SURVEY.md §8(c)) -------------------------------------
template <class K>
int ros_sort(const K* x, const uint32_t* v, uint64_t n, uint32_t p, uint32_t s, uint64_t seed,
             K* out, uint32_t* outv, K* sk, uint64_t* st, uint64_t* counts) {
    if (p == 0) return EINVAL;
    // R0
    if (n == 0) {
        if (counts) for (uint32_t j = 0; j < p; ++j) counts[j] = 0;
        return OK;
    }
    if (p == 1) {
        plain_stable_sort(x, v, n, out, outv);
        if (counts) counts[0] = n;
        return OK;
    }
    if (s == 0) return ESAMPLE;
    const uint64_t m = (uint64_t)p * s - 1;  // sample size ps-1 (Q3)
    if (m > n) return ESAMPLE;
    // R1
    std::vector<uint64_t> I = ros_sample_indices(n, m, seed, nullptr);
    // R2: T = [(x[i], i)], sorted by (key, i) ("Sort T"; tags P:524-532)
    std::vector<Rec<K>> T(m);
    for (uint64_t t = 0; t < m; ++t) T[t] = {x[I[t]], I[t]};
    std::sort(T.begin(), T.end(), rec_less<K>);
    // R3: S[q] = (q+1)s-th smallest = T[(q+1)s - 1] (Q4)
    std::vector<Rec<K>> S(p - 1);
    for (uint32_t q = 0; q + 1 < p; ++q) S[q] = T[(uint64_t)(q + 1) * s - 1];
    write_report(S, sk, st);
    // R4: b(i) = #{q : S[q] <lex (x[i], i)} — binary search over the splitters
    std::vector<uint32_t> b(n);
    std::vector<uint64_t> cnt(p, 0);
    for (uint64_t i = 0; i < n; ++i) {
        Rec<K> e{x[i], i};
        b[i] = (uint32_t)(std::lower_bound(S.begin(), S.end(), e, rec_less<K>) - S.begin());
        cnt[b[i]]++;  // R5
    }
    // R5: bucket starts = exclusive prefix sum of the counts
    std::vector<uint64_t> start(p + 1, 0);
    for (uint32_t j = 0; j < p; ++j) start[j + 1] = start[j] + cnt[j];
    // R6: stable counting scatter ("the p output sequences that will be formed")
    std::vector<Item<K>> y(n);
    std::vector<uint64_t> cur(start.begin(), start.end() - 1);
    for (uint64_t i = 0; i < n; ++i) y[cur[b[i]]++] = {x[i], v ? v[i] : 0u, i};
    // R7: sort each sequence independently (stable: equal keys keep input order)
    for (uint32_t j = 0; j < p; ++j)
        std::stable_sort(y.begin() + start[j], y.begin() + start[j + 1],
                         [](const Item<K>& A, const Item<K>& B) { return A.key < B.key; });
    // R8: concatenation
    for (uint64_t i = 0; i < n; ++i) {
        out[i] = y[i].key;
        if (outv) outv[i] = y[i].val;
    }
    if (counts) for (uint32_t j = 0; j < p; ++j) counts[j] = cnt[j];
    return OK;
}

// ---- baseline split of Algorithms 1/2 step 1 (Q8) ------------------
inline uint64_t seq_len(uint64_t n, uint64_t p, uint64_t k) { return n / p + (k < n % p ? 1 : 0); }
inline uint64_t seq_start(uint64_t n, uint64_t p, uint64_t k) { return k * (n / p) + std::min(k, n % p); }

// Step 1 (BaselineSorting): each X_k stably sorted by key; element at sorted position t of
// X_k carries val and tag.  `tag_mode` 0: tag = start_k + t (DRO, Q6); 1: original index.
template <class K>
std::vector<Item<K>> baseline_sorting(const K* x, const uint32_t* v, uint64_t n, uint32_t p, int tag_mode) {
    std::vector<Item<K>> X(n);
    for (uint64_t i = 0; i < n; ++i) X[i] = {x[i], v ? v[i] : 0u, i};
    for (uint32_t k = 0; k < p; ++k) {
        uint64_t a = seq_start(n, p, k), m = seq_len(n, p, k);
        std::stable_sort(X.begin() + a, X.begin() + a + m,
                         [](const Item<K>& A, const Item<K>& B) { return A.key < B.key; });
        if (tag_mode == 0)
            for (uint64_t t = 0; t < m; ++t) X[a + t].tag = a + t;
    }
    return X;
}

// Step 4: bound[k][j] = #{t : (X_k[t], tag) <=lex S[j]}, by binary
// search of each splitter into the sorted X_k (X_k is sorted by (key, tag)).
template <class K>
std::vector<uint64_t> split_bounds(const std::vector<Item<K>>& X, uint64_t n, uint32_t p,
                                   const std::vector<Rec<K>>& S) {
    std::vector<uint64_t> bnd((uint64_t)p * (p + 1));
    for (uint32_t k = 0; k < p; ++k) {
        uint64_t a = seq_start(n, p, k), m = seq_len(n, p, k);
        auto first = X.begin() + a, last = X.begin() + a + m;
        bnd[(uint64_t)k * (p + 1) + 0] = 0;
        for (uint32_t j = 0; j + 1 < p; ++j) {
            auto it = std::upper_bound(first, last, S[j], [](const Rec<K>& s, const Item<K>& e) {
                return lex_less(s.key, s.tag, e.key, e.tag);
            });
            bnd[(uint64_t)k * (p + 1) + j + 1] = (uint64_t)(it - first);
        }
        bnd[(uint64_t)k * (p + 1) + p] = m;
    }
    return bnd;
}

// Step 5: Y_j = p-way merge of X_{0,j},...,X_{p-1,j}; stability is
// "resolved by the merging algorithm itself": ties go to the lower k.
template <class K>
void merge_buckets(const std::vector<Item<K>>& X, uint64_t n, uint32_t p, const std::vector<uint64_t>& bnd,
                   K* out, uint32_t* outv, uint64_t* counts) {
    uint64_t o = 0;
    struct Head { K key; uint32_t k; uint64_t pos, end; };
    auto worse = [](const Head& A, const Head& B) {  // priority_queue keeps the max on top
        if (B.key < A.key) return true;
        if (A.key < B.key) return false;
        return A.k > B.k;
    };
    for (uint32_t j = 0; j < p; ++j) {
        std::priority_queue<Head, std::vector<Head>, decltype(worse)> pq(worse);
        uint64_t nj = 0;
        for (uint32_t k = 0; k < p; ++k) {
            uint64_t a = seq_start(n, p, k);
            uint64_t lo = a + bnd[(uint64_t)k * (p + 1) + j], hi = a + bnd[(uint64_t)k * (p + 1) + j + 1];
            nj += hi - lo;
            if (lo < hi) pq.push({X[lo].key, k, lo, hi});
        }
        while (!pq.empty()) {
            Head h = pq.top();
            pq.pop();
            out[o] = X[h.pos].key;
            if (outv) outv[o] = X[h.pos].val;
            ++o;
            if (++h.pos < h.end) {
                h.key = X[h.pos].key;
                pq.push(h);
            }
        }
        if (counts) counts[j] = nj;
    }
}

// ---- SqRan, literal Algorithm 2 ----------------------------------------------
// The sample is the same index set I over ORIGINAL positions (reading Q2); each sampled key
// is tagged with its original index, which orders equal keys exactly as (seq id, index) does.
template <class K>
int sqran_literal(const K* x, const uint32_t* v, uint64_t n, uint32_t p, uint32_t s, uint64_t seed,
                  K* out, uint32_t* outv, K* sk, uint64_t* st, uint64_t* counts) {
    if (p == 0) return EINVAL;
    if (n == 0) {
        if (counts) for (uint32_t j = 0; j < p; ++j) counts[j] = 0;
        return OK;
    }
    if (p == 1) {
        plain_stable_sort(x, v, n, out, outv);
        if (counts) counts[0] = n;
        return OK;
    }
    if (s == 0) return ESAMPLE;
    const uint64_t m = (uint64_t)p * s - 1;
    if (m > n) return ESAMPLE;
    // step 1: BaselineSorting, tags = original index
    std::vector<Item<K>> X = baseline_sorting(x, v, n, p, 1);
    // step 2: sample ps-1 keys uniformly at random from the keys of all X_k; sort T
    std::vector<uint64_t> I = ros_sample_indices(n, m, seed, nullptr);
    std::vector<Rec<K>> T(m);
    for (uint64_t t = 0; t < m; ++t) T[t] = {x[I[t]], I[t]};
    std::sort(T.begin(), T.end(), rec_less<K>);
    // step 3: splitters = (i*s)-th smallest, 1 <= i <= p-1
    std::vector<Rec<K>> S(p - 1);
    for (uint32_t q = 0; q + 1 < p; ++q) S[q] = T[(uint64_t)(q + 1) * s - 1];
    write_report(S, sk, st);
    // step 4: split the sorted X_k around S
    std::vector<uint64_t> bnd = split_bounds(X, n, p, S);
    // step 5: merge, concatenate
    merge_buckets(X, n, p, bnd, out, outv, counts);
    return OK;
}

// ---- McRan: Algorithm 2 with its independent work spread over t threads -------------------
// The paper's multi-core variant: the p BaselineSorting sorts of step 1 (P:664-668,
// "the p sorts ... over m cores"), the p binary-search splits of step 4 and the p bucket merges of
// step 5 run on t std::threads; the sample, its sort and the splitters are the sequential steps.
// Same results as sqran_literal (tests/test_oracle_pins.py); timed by bench.py as the multi-core CPU
// baseline.
template <class F>
void parallel_for(uint32_t count, uint32_t threads, F&& f) {
    std::atomic<uint32_t> next{0};
    std::vector<std::thread> ts;
    for (uint32_t t = 0; t < std::max<uint32_t>(threads, 1); ++t)
        ts.emplace_back([&] {
            for (uint32_t i; (i = next++) < count;) f(i);
        });
    for (auto& th : ts) th.join();
}

template <class K>
int mcran_sort(const K* x, const uint32_t* v, uint64_t n, uint32_t p, uint32_t s, uint64_t seed, uint32_t threads,
               K* out, uint32_t* outv, K* sk, uint64_t* st, uint64_t* counts) {
    if (p == 0) return EINVAL;
    if (n == 0) {
        if (counts) for (uint32_t j = 0; j < p; ++j) counts[j] = 0;
        return OK;
    }
    if (p == 1) {
        plain_stable_sort(x, v, n, out, outv);
        if (counts) counts[0] = n;
        return OK;
    }
    if (s == 0) return ESAMPLE;
    const uint64_t m = (uint64_t)p * s - 1;
    if (m > n) return ESAMPLE;
    // step 1 in parallel: X_k stably sorted, tags = original index
    std::vector<Item<K>> X(n);
    for (uint64_t i = 0; i < n; ++i) X[i] = {x[i], v ? v[i] : 0u, i};
    parallel_for(p, threads, [&](uint32_t k) {
        uint64_t a = seq_start(n, p, k), mk = seq_len(n, p, k);
        std::stable_sort(X.begin() + a, X.begin() + a + mk,
                         [](const Item<K>& A, const Item<K>& B) { return A.key < B.key; });
    });
    // steps 2-3: the sample (same index set I), sorted; splitters
    std::vector<uint64_t> I = ros_sample_indices(n, m, seed, nullptr);
    std::vector<Rec<K>> T(m);
    for (uint64_t t = 0; t < m; ++t) T[t] = {x[I[t]], I[t]};
    std::sort(T.begin(), T.end(), rec_less<K>);
    std::vector<Rec<K>> S(p - 1);
    for (uint32_t q = 0; q + 1 < p; ++q) S[q] = T[(uint64_t)(q + 1) * s - 1];
    write_report(S, sk, st);
    // step 4 in parallel: split every X_k around S by binary search
    std::vector<uint64_t> bnd((uint64_t)p * (p + 1));
    parallel_for(p, threads, [&](uint32_t k) {
        uint64_t a = seq_start(n, p, k), mk = seq_len(n, p, k);
        auto first = X.begin() + a, last = X.begin() + a + mk;
        bnd[(uint64_t)k * (p + 1)] = 0;
        for (uint32_t j = 0; j + 1 < p; ++j) {
            auto it = std::upper_bound(first, last, S[j], [](const Rec<K>& sp, const Item<K>& e) {
                return lex_less(sp.key, sp.tag, e.key, e.tag);
            });
            bnd[(uint64_t)k * (p + 1) + j + 1] = (uint64_t)(it - first);
        }
        bnd[(uint64_t)k * (p + 1) + p] = mk;
    });
    // step 5 in parallel: bucket j = the p-way merge of its runs (ties to the lower k), at its offset
    std::vector<uint64_t> start(p + 1, 0);
    for (uint32_t j = 0; j < p; ++j) {
        uint64_t nj = 0;
        for (uint32_t k = 0; k < p; ++k) nj += bnd[(uint64_t)k * (p + 1) + j + 1] - bnd[(uint64_t)k * (p + 1) + j];
        start[j + 1] = start[j] + nj;
        if (counts) counts[j] = nj;
    }
    struct Head { K key; uint32_t k; uint64_t pos, end; };
    parallel_for(p, threads, [&](uint32_t j) {
        auto worse = [](const Head& A, const Head& B) {
            if (B.key < A.key) return true;
            if (A.key < B.key) return false;
            return A.k > B.k;
        };
        std::priority_queue<Head, std::vector<Head>, decltype(worse)> pq(worse);
        for (uint32_t k = 0; k < p; ++k) {
            uint64_t a = seq_start(n, p, k);
            uint64_t lo = a + bnd[(uint64_t)k * (p + 1) + j], hi = a + bnd[(uint64_t)k * (p + 1) + j + 1];
            if (lo < hi) pq.push({X[lo].key, k, lo, hi});
        }
        uint64_t o = start[j];
        while (!pq.empty()) {
            Head h = pq.top();
            pq.pop();
            out[o] = X[h.pos].key;
            if (outv) outv[o] = X[h.pos].val;
            ++o;
            if (++h.pos < h.end) {
                h.key = X[h.pos].key;
                pq.push(h);
            }
        }
    });
    return OK;
}

// ---- DRO regular sample position (reading Q9) ----------------------------------
// Position (0-based, in the sorted X_k of m keys) of the j-th of the s = rp samples.
// Balanced (default): X_k is cut into s segments, the first (m mod s) of ceil(m/s) keys and
// the rest of floor(m/s) keys; the sample is each segment's last key, so j = s-1 is the max.
// Padded (flag): the Lemma 1 proof's virtual padding, segments of
// x = ceil(ceil(n/p)/s) keys, positions past the end clamped to the maximum.
uint64_t dro_position(uint64_t m, uint64_t s, uint64_t j, uint32_t flags, uint64_t xpad) {
    if (flags & DRO_PADDED_POSITIONS) return (j + 1 == s) ? m - 1 : std::min((j + 1) * xpad, m) - 1;
    uint64_t q = m / s, rho = m % s;
    return (j + 1) * q + std::min(j + 1, rho) - 1;  // end of the j-th balanced segment
}

// ---- DRO = SqDet, literal Algorithm 1 ----------------------------------------
template <class K>
int dro_sort(const K* x, const uint32_t* v, uint64_t n, uint32_t p, uint32_t r, uint32_t flags,
             K* out, uint32_t* outv, K* sk, uint64_t* st, uint64_t* counts) {
    if (p == 0) return EINVAL;
    if (n == 0) {
        if (counts) for (uint32_t j = 0; j < p; ++j) counts[j] = 0;
        return OK;
    }
    if (p == 1) {
        plain_stable_sort(x, v, n, out, outv);
        if (counts) counts[0] = n;
        return OK;
    }
    if (r == 0) return ESAMPLE;
    const uint64_t s = (uint64_t)r * p;  // "Let r = ceil(omega_n) and s = rp"
    if (s > n / p) return ESAMPLE;       // distinct sample positions in every X_k (Q16)
    // step 1: BaselineSorting, tag = start_k + position (Q6)
    std::vector<Item<K>> X = baseline_sorting(x, v, n, p, 0);
    // step 2: T_k = rp-1 evenly spaced keys of X_k + its maximum (reading Q9)
    std::vector<Rec<K>> T;
    T.reserve(s * p);
    const uint64_t xpad = ((n + p - 1) / p + s - 1) / s;  // x = ceil(ceil(n/p)/s)
    for (uint32_t k = 0; k < p; ++k) {
        uint64_t a = seq_start(n, p, k), mk = seq_len(n, p, k);
        for (uint64_t j = 0; j < s; ++j) {
            uint64_t e = dro_position(mk, s, j, flags, xpad);
            T.push_back({X[a + e].key, X[a + e].tag});
        }
    }
    // "Merge all T_k into a sorted sequence T of rp^2 keys"
    std::sort(T.begin(), T.end(), rec_less<K>);
    // step 3: S = the (i*s)-th smallest keys of T, s = rp (Q4)
    std::vector<Rec<K>> S(p - 1);
    for (uint32_t q = 0; q + 1 < p; ++q) S[q] = T[(uint64_t)(q + 1) * s - 1];
    write_report(S, sk, st);
    // step 4: split by binary search
    std::vector<uint64_t> bnd = split_bounds(X, n, p, S);
    // step 5: merge each bucket, concatenate
    merge_buckets(X, n, p, bnd, out, outv, counts);
    return OK;
}

template <class F>
int dispatch(int dtype, F&& f) {
    switch (dtype) {
        case DT_U32: return f((uint32_t*)nullptr);
        case DT_I32: return f((int32_t*)nullptr);
        case DT_F64: return f((double*)nullptr);
        case DT_S32: return f((S32*)nullptr);
        default: return EDTYPE;
    }
}

}  // namespace

extern "C" {

int orc_version(void) { return 1; }

uint64_t orc_splitmix64(uint64_t seed, uint64_t stream, uint64_t j) { return H(seed, stream, j); }

uint64_t orc_draw_index(uint64_t u, uint64_t n) { return draw_index(u, n); }

// I in draw order; returns the number of draws consumed in *draws (may be NULL).
int orc_ros_sample_indices(uint64_t n, uint32_t p, uint32_t s, uint64_t seed, uint64_t* out_idx, uint64_t* draws) {
    if (p < 2 || s == 0) return EINVAL;
    uint64_t m = (uint64_t)p * s - 1;
    if (m > n) return ESAMPLE;
    std::vector<uint64_t> I = ros_sample_indices(n, m, seed, draws);
    std::memcpy(out_idx, I.data(), m * sizeof(uint64_t));
    return OK;
}

// positions of the s = r p regular samples of sequence k (DRO step 2), 0-based within X_k
int orc_dro_sample_positions(uint64_t n, uint32_t p, uint32_t r, uint32_t flags, uint32_t k, uint64_t* out) {
    if (p < 2 || r == 0 || k >= p) return EINVAL;
    const uint64_t s = (uint64_t)r * p;
    if (s > n / p) return ESAMPLE;
    const uint64_t xpad = ((n + p - 1) / p + s - 1) / s;
    for (uint64_t j = 0; j < s; ++j) out[j] = dro_position(seq_len(n, p, k), s, j, flags, xpad);
    return OK;
}

int orc_ros_sort(int dtype, const void* keys, const uint32_t* vals, uint64_t n, uint32_t p, uint32_t s,
                 uint64_t seed, void* out_keys, uint32_t* out_vals, void* split_keys, uint64_t* split_tags,
                 uint64_t* counts) {
    return dispatch(dtype, [&](auto* tag) {
        using K = std::remove_pointer_t<decltype(tag)>;
        return ros_sort<K>((const K*)keys, vals, n, p, s, seed, (K*)out_keys, out_vals, (K*)split_keys,
                           split_tags, counts);
    });
}

int orc_sqran_literal(int dtype, const void* keys, const uint32_t* vals, uint64_t n, uint32_t p, uint32_t s,
                      uint64_t seed, void* out_keys, uint32_t* out_vals, void* split_keys, uint64_t* split_tags,
                      uint64_t* counts) {
    return dispatch(dtype, [&](auto* tag) {
        using K = std::remove_pointer_t<decltype(tag)>;
        return sqran_literal<K>((const K*)keys, vals, n, p, s, seed, (K*)out_keys, out_vals, (K*)split_keys,
                                split_tags, counts);
    });
}

int orc_mcran_sort(int dtype, const void* keys, const uint32_t* vals, uint64_t n, uint32_t p, uint32_t s,
                   uint64_t seed, uint32_t threads, void* out_keys, uint32_t* out_vals, void* split_keys,
                   uint64_t* split_tags, uint64_t* counts) {
    return dispatch(dtype, [&](auto* tag) {
        using K = std::remove_pointer_t<decltype(tag)>;
        return mcran_sort<K>((const K*)keys, vals, n, p, s, seed, threads, (K*)out_keys, out_vals, (K*)split_keys,
                             split_tags, counts);
    });
}

int orc_dro_sort(int dtype, const void* keys, const uint32_t* vals, uint64_t n, uint32_t p, uint32_t r,
                 uint32_t flags, void* out_keys, uint32_t* out_vals, void* split_keys, uint64_t* split_tags,
                 uint64_t* counts) {
    return dispatch(dtype, [&](auto* tag) {
        using K = std::remove_pointer_t<decltype(tag)>;
        return dro_sort<K>((const K*)keys, vals, n, p, r, flags, (K*)out_keys, out_vals, (K*)split_keys,
                           split_tags, counts);
    });
}

}  // extern "C"
