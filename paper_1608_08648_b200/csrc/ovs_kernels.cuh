// ovs_kernels.cuh — sm_100a kernels of the partition-first oversampling sort.
//
// Citations: "P:n" = /root/reference/PAPER.md line n.  "§8(a) aN" = SURVEY.md hot-path row.
// Design notes: all ranking inside a CTA uses shared-memory atomics
// (measured on B200: random-address ATOMS run at LDS speed, ~9 lanes/clk/SM, while
// __match_any_sync runs at 0.5 lanes/clk/SM — tools/ubench, profiles/r01_ubench.txt), so no
// kernel uses warp-match ranking.  Placement inside a bucket run is therefore not in input
// order; determinism of the OUTPUT comes from the bucket sorter, which orders every bucket
// totally: by key (keys-only: the sorted multiset is unique) or by (key, original index)
// (key-value: that is exactly the stable order).  Splitters and bucket counts never
// depend on placement order.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <type_traits>

namespace ovs {
// internal linkage: every translation unit gets its own copy of the kernels it launches
namespace {

typedef uint32_t u32;
typedef uint64_t u64;
typedef uint16_t u16;

// ------------------------------------------------------------------ programmatic dependent launch
// First statement of every kernel (see launch() in ovs_engine.cuh): allow the next kernel on the
// stream to be scheduled once all CTAs of this one have started, then wait until the previous
// kernel has completed and its memory is visible.  Both are no-ops without the PDL attribute,
// which launch() sets only with -DOVS_PDL=1 (measured: no gain over plain stream order, and
// CUDA-graph replay already removes the launch gaps).
#ifndef OVS_PDL
#define OVS_PDL 0
#endif
#ifndef OVS_WC_BFLUSH  // write-combining scatter: completed sectors flushed per bucket (0: per key)
#define OVS_WC_BFLUSH 1
#endif
#define PDL_PROLOGUE() asm volatile("griddepcontrol.launch_dependents;\n\tgriddepcontrol.wait;" ::: "memory")

// ------------------------------------------------------------------ key codecs
// Keys are compared as "ordered bits": an order-preserving map to unsigned integers
// (native < on u32; sign flip on i32; IEEE total order on f64 without NaN / -0, reading Q18).
enum { DT_U32 = 0, DT_I32 = 1, DT_F64 = 2, DT_U64 = 3 /* internal, identity */,
       DT_S32 = 4 /* 32-byte strings: the key word is the big-endian 8-byte prefix */ };

template <int DT> struct Codec;
template <> struct Codec<DT_U32> {
    typedef u32 U;
    __device__ __forceinline__ static U ord(U b) { return b; }
    __device__ __forceinline__ static U raw(U o) { return o; }
};
template <> struct Codec<DT_I32> {
    typedef u32 U;
    __device__ __forceinline__ static U ord(U b) { return b ^ 0x80000000u; }
    __device__ __forceinline__ static U raw(U o) { return o ^ 0x80000000u; }
};
template <> struct Codec<DT_F64> {
    typedef u64 U;
    __device__ __forceinline__ static U ord(U b) { return (b >> 63) ? ~b : (b | 0x8000000000000000ull); }
    __device__ __forceinline__ static U raw(U o) { return (o >> 63) ? (o & 0x7fffffffffffffffull) : ~o; }
};
template <> struct Codec<DT_U64> {
    typedef u64 U;
    __device__ __forceinline__ static U ord(U b) { return b; }
    __device__ __forceinline__ static U raw(U o) { return o; }
};

template <> struct Codec<DT_S32> {
    typedef u64 U;
    __device__ __forceinline__ static U ord(U b) { return b; }
    __device__ __forceinline__ static U raw(U o) { return o; }
};
// a 64-bit word of a string record as a big-endian number (memcmp order = integer order)
__device__ __forceinline__ u64 bswap64(u64 x) {
    const u32 lo = (u32)x, hi = (u32)(x >> 32);
    return ((u64)__byte_perm(lo, 0, 0x0123) << 32) | __byte_perm(hi, 0, 0x0123);
}
// the key word of item i: the ordered key (x holds keys) or, for strings (x holds the 32-byte
// records as 4 words each), the big-endian prefix
template <int DT>
__device__ __forceinline__ typename Codec<DT>::U load_key(const typename Codec<DT>::U* x, u64 i) {
    if constexpr (DT == DT_S32) return bswap64(x[4 * i]);
    else return Codec<DT>::ord(x[i]);
}

template <class U> __device__ __host__ __forceinline__ U umax_of() { return (U)~(U)0; }
template <class U> __device__ __forceinline__ u32 bitlen(U x) {
    return x == 0 ? 0u : (u32)(8 * sizeof(U)) - (sizeof(U) == 8 ? __clzll((long long)x) : __clz((int)x));
}

// ------------------------------------------------------------------ device status bits
enum : u32 {
    ST_SAMPLE_SHORT = 1u,   // fewer than ps-1 distinct candidates were drawn (never observed)
    ST_BUCKET_OVER = 2u,    // a bucket larger than the on-chip capacity reached the sorter
    ST_LIST_OVER = 4u,      // a work list overflowed its capacity
};
// status[0]: bits of the current call (zeroed when the call starts); status[1]: sticky bits of
// every call since the caller last reset them (ovs_device_status), so graph replays are checkable
__device__ __forceinline__ void st_set(u32* status, u32 bit) {
    atomicOr(status, bit);
    atomicOr(status + 1, bit);
}

// ------------------------------------------------------------------ counter-based RNG
// H(seed, stream, j) = SplitMix64 output number stream*2^40 + j (reading Q1).
__device__ __forceinline__ u64 mix64(u64 z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ u64 rng_H(u64 seed, u64 stream, u64 j) {
    return mix64(seed + 0x9e3779b97f4a7c15ull * ((stream << 40) + j + 1));
}

// ------------------------------------------------------------------ work descriptors
struct Bucket {   // a contiguous range of items, in buffer `buf`, still to be sorted
    u32 beg, len, buf, level;
    u64 lo, hi;   // ordered-key bounds of the items (from the splitters around it)
};

struct Seg {      // a range being partitioned by one splitter set (one classifier)
    u64 lo, hi;   // ordered-key bounds of the segment
    u64 base;     // classifier LUT base key
    u32 beg, len, P, shift, L, chunk0, nchunk, src, loose, pad;
};

struct Chunk { u32 beg, end, seg, pad; };

// the two ping-pong buffers of a sort: buffer 0 is the caller's array (raw keys on entry,
// raw sorted keys on exit), buffer 1 is workspace.  Key-value sorts also carry the values
// and the original index (the stability tie-break).
template <class U> struct Bufs {
    U* k[2];
    u32* v[2];
    u32* i[2];
};

// Multi-GPU: every rank's receive window as addressable from this GPU (NVLink peer mappings of
// the NCCL symmetric window: peers[d] = window base of rank d), and an offset into it
struct PeerOut {
    char* const* peers;  // device array [world]
    size_t off;          // byte offset of the region inside every window
    u32 world;
};

// DIST sample records: record rk of the global sample goes to slot rk of every rank's window
// (32-bit keys: one word ord key << 32 | global index; 64-bit keys: key word, index word)
template <bool WIDE>
__device__ __forceinline__ void put_rec(const PeerOut& po, u32 rk, u64 kw, u64 c) {
    for (u32 d = 0; d < po.world; ++d) {
        u64* r = (u64*)(po.peers[d] + po.off);
        if (!WIDE) r[rk] = (kw << 32) | c;
        else { r[2 * (u64)rk] = kw; r[2 * (u64)rk + 1] = c; }
    }
}

// Bucket.level flags: lo/hi are not tight bounds; the items are the caller's raw keys (codec
// not applied yet, value/index arrays not built yet: index = position)
enum : u32 { BK_LOOSE = 0x80000000u, BK_RAW = 0x40000000u, BK_FORCE = 0x20000000u /* re-split it */ };

// ------------------------------------------------------------------ the classifier
// bucket(k, tag) = #{q : S[q] <lex (k, tag)}: a lower_bound over the p-1 splitters with the
// (key, tag) tie-break.  The binary search is narrowed by a lookup
// table over the ordered-key space: entry e covers keys [base + e<<shift, base + (e+1)<<shift)
// and stores (32 bits) lo_e = #{q : S[q].key < base + e<<shift} (bits 0-12, p <= 8192), cnt_e =
// #splitter keys inside the entry (bits 13-15, 7 = "see entry e+1") and frac_e = the position of
// the first of them inside the entry at 16-bit resolution (bits 16-31).  cnt 0: the bucket is
// lo; cnt 1: comparing the key's own 16-bit position with frac decides unless they are equal
// (then one exact (key, tag) comparison); cnt >= 2: binary search of those cnt splitters.  The
// result is exactly the lower_bound (tests/test_gpu_parity.py compares bucket counts with the
// oracle).
template <class U> struct ClsView {
    const U* sk; const u32* st; const u32* lut;
    U base; u32 shift, L, P;
    u32 fr, fl;  // 16-bit position of x = key - base inside its entry: ((x >> fr) << fl) & 0xffff
};

// 16-bit position of an offset inside a table entry of 2^shift keys
template <class U> __device__ __host__ __forceinline__ u32 cls_frac(U off, u32 shift) {
    return shift >= 16 ? (u32)(off >> (shift - 16)) : (u32)(off << (16 - shift));
}
template <class U> __device__ __forceinline__ u32 cls_kfrac(const ClsView<U>& c, U x) {
    return (u32)((x >> c.fr) << c.fl) & 0xffffu;
}

template <class U>
__device__ __forceinline__ u32 classify(const ClsView<U>& c, U k, u32 tag) {
    if (c.P <= 1) return 0;
    if (k < c.base) return 0;
    const U x = (U)(k - c.base);
    const U d = x >> c.shift;
    if (d >= (U)c.L) return c.P - 1;
    const u32 e = c.lut[(u32)d];
    u32 lo = e & 0x1fffu, cnt = (e >> 13) & 7u;
    if (cnt == 1) {
        const u32 kf = cls_kfrac<U>(c, x), sf = e >> 16;
        if (kf != sf) return lo + (kf > sf ? 1u : 0u);
    }
    if (cnt == 7) cnt = (c.lut[(u32)d + 1] & 0x1fffu) - lo;  // saturated: the next entry's lo bounds it
    while (cnt > 0) {
        u32 half = cnt >> 1, mid = lo + half;
        U s = c.sk[mid];
        bool less = (s < k) || (s == k && c.st[mid] < tag);
        if (less) { lo = mid + 1; cnt -= half + 1; } else { cnt = half; }
    }
    return lo;
}

#ifdef OVS_CLS_OLD  // round-1 form (A/B experiments): lookups first, then the position test per key
template <class U, int N, class TagF>
__device__ __forceinline__ void classify_n(const ClsView<U>& c, const U (&k)[N], TagF&& tag, u32 (&b)[N]) {
    if (c.P <= 1) {
#pragma unroll
        for (int j = 0; j < N; ++j) b[j] = 0;
        return;
    }
    u32 e[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
        const U x = (U)(k[j] - c.base);
        const U d = x >> c.shift;
        const bool below = k[j] < c.base, above = !below && d >= (U)c.L;
        e[j] = (below || above) ? 0u : c.lut[(u32)d];
        b[j] = below ? 0u : above ? c.P - 1 : (e[j] & 0x1fffu);
    }
    u32 left = 0;
#pragma unroll
    for (int j = 0; j < N; ++j) {
        const u32 cnt = (e[j] >> 13) & 7u;
        if (cnt == 1) {
            const U x = (U)(k[j] - c.base);
            const u32 kf = cls_kfrac<U>(c, x), sf = e[j] >> 16;
            if (kf != sf) b[j] += kf > sf ? 1u : 0u;
            else left |= 1u << j;
        } else if (cnt > 1) {
            left |= 1u << j;
        }
    }
    if (__any_sync(0xffffffffu, left != 0)) {
#pragma unroll
        for (int j = 0; j < N; ++j) {
            if (!((left >> j) & 1u)) continue;
            u32 cnt = (e[j] >> 13) & 7u;
            if (cnt == 7) cnt = (c.lut[(u32)((U)(k[j] - c.base) >> c.shift) + 1] & 0x1fffu) - b[j];
            while (cnt > 0) {
                const u32 half = cnt >> 1, mid = b[j] + half;
                const U s = c.sk[mid];
                const bool less = (s < k[j]) || (s == k[j] && c.st[mid] < tag(j));
                if (less) { b[j] = mid + 1; cnt -= half + 1; } else { cnt = half; }
            }
        }
    }
}
#else
// Batched form for N keys held in registers, branch-free on the common path: entry d of the table
// (d clamped to L; lut[L] is the sentinel entry "bucket P-1, no splitter") gives b = lo + (kf > sf),
// exact whenever the entry holds no splitter (sf = 0xffff there, so kf > sf never holds) or one
// splitter whose 16-bit position differs from the key's.  The keys left (two or more splitters in
// the entry, or kf == sf) take the binary search among the entry's splitters, from lo.
template <class U, int N, class TagF>
__device__ __forceinline__ void classify_n(const ClsView<U>& c, const U (&k)[N], TagF&& tag, u32 (&b)[N]) {
    if (c.P <= 1) {
#pragma unroll
        for (int j = 0; j < N; ++j) b[j] = 0;
        return;
    }
    u32 e[N], left = 0;
#pragma unroll
    for (int j = 0; j < N; ++j) {
        const U x = (U)(k[j] - c.base);
        const bool below = k[j] < c.base;
        const U d = min((U)(x >> c.shift), (U)c.L);
        e[j] = c.lut[(u32)d];
        const u32 kf = cls_kfrac<U>(c, x), sf = e[j] >> 16;
        b[j] = below ? 0u : (e[j] & 0x1fffu) + (kf > sf ? 1u : 0u);
        const bool ex = !below && (((e[j] >> 13) & 7u) >= 2u || kf == sf);
        left |= (ex ? 1u : 0u) << j;
    }
    if (__any_sync(0xffffffffu, left != 0)) {
#pragma unroll
        for (int j = 0; j < N; ++j) {
            if (!((left >> j) & 1u)) continue;
            b[j] = e[j] & 0x1fffu;
            u32 cnt = (e[j] >> 13) & 7u;
            if (cnt == 7) cnt = (c.lut[(u32)((U)(k[j] - c.base) >> c.shift) + 1] & 0x1fffu) - b[j];
            while (cnt > 0) {
                const u32 half = cnt >> 1, mid = b[j] + half;
                const U s = c.sk[mid];
                const bool less = (s < k[j]) || (s == k[j] && c.st[mid] < tag(j));
                if (less) { b[j] = mid + 1; cnt -= half + 1; } else { cnt = half; }
            }
        }
    }
}

#endif

// ------------------------------------------------------------------ block helpers
template <int NT>
__device__ __forceinline__ u32 block_exclusive_scan(u32 v, u32* red /*[NT/32+1]*/, u32* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    u32 x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        u32 y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) red[wid] = x;
    __syncthreads();
    if (wid == 0) {
        u32 w = (lane < NT / 32) ? red[lane] : 0u;
        u32 t = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            u32 y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        if (lane < NT / 32) red[lane] = t - w;
        if (lane == NT / 32 - 1) red[NT / 32] = t;
    }
    __syncthreads();
    u32 r = red[wid] + x - v;
    if (total) *total = red[NT / 32];
    __syncthreads();
    return r;
}

// exclusive scan of 4 words per thread at once (each word may pack independent 16-bit fields
// whose sums stay below 2^16); total[] receives the CTA totals
template <int NT>
__device__ __forceinline__ void block_exclusive_scan4(u32 (&v)[4], u32 (*red)[4] /*[NT/32 + 1]*/, u32 (&total)[4]) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    u32 x[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) x[q] = v[q];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const u32 y = __shfl_up_sync(0xffffffffu, x[q], o);
            if (lane >= o) x[q] += y;
        }
    }
    if (lane == 31)
#pragma unroll
        for (int q = 0; q < 4; ++q) red[wid][q] = x[q];
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const u32 w = lane < NT / 32 ? red[lane][q] : 0u;
            u32 t = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const u32 y = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += y;
            }
            if (lane < NT / 32) red[lane][q] = t - w;
            if (lane == NT / 32 - 1) red[NT / 32][q] = t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        total[q] = red[NT / 32][q];
        v[q] = red[wid][q] + x[q] - v[q];
    }
    __syncthreads();
}

// exclusive scan in place of a[0..cnt) (cnt arbitrary) by a CTA of NT threads; a[cnt] = total
template <int NT>
__device__ void block_scan_array(u32* a, u32 cnt, u32* red) {
    u32 carry = 0;
    for (u32 b0 = 0; b0 < cnt; b0 += NT * 4) {
        u32 i0 = b0 + threadIdx.x * 4;
        u32 v[4], s = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) { v[j] = (i0 + j < cnt) ? a[i0 + j] : 0u; s += v[j]; }
        u32 tot;
        u32 ex = block_exclusive_scan<NT>(s, red, &tot);
        ex += carry;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (i0 + j < cnt) a[i0 + j] = ex;
            ex += v[j];
        }
        carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) a[cnt] = carry;
    __syncthreads();
}

// exclusive scan in place of a[0..cnt), cnt <= NT*16, one round (16 consecutive per thread)
// Thread t owns a[16t .. 16t+16) but visits them rotated by r = (t/2) mod 16 (element
// (j + r) mod 16 at step j), so the 32 lanes of a warp hit 32 distinct banks at every step.
template <int NT>
__device__ void block_scan_small(u32* a, u32 cnt, u32* red) {
    const u32 i0 = threadIdx.x * 16, r = (threadIdx.x >> 1) & 15;
    u32 v[16], s = 0, head = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const u32 e = (j + r) & 15;
        v[j] = (i0 + e < cnt) ? a[i0 + e] : 0u;
        s += v[j];
        if (e < r) head += v[j];
    }
    const u32 base = block_exclusive_scan<NT>(s, red, nullptr);
    u32 run = base + head;  // prefix of element r
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const u32 e = (j + r) & 15;
        if (e == 0) run = base;
        if (i0 + e < cnt) a[i0 + e] = run;
        run += v[j];
    }
    __syncthreads();
}

// block_scan_small that also lists every index whose count is >= T in list[] (ascending; *nlist =
// their number, *over set when it exceeds cap).  Each thread marks its big elements in a 16-bit mask
// and their number rides in the high half of the value the CTA scans (the counts sum to < 2^16:
// cnt <= NT*16 elements of a bucket that fits on chip), so the list needs no shared atomics
// (a shared counter bumped by every warp serialised this scan: 5.5K cycles per bucket).  The
// 32-bit keys-only bucket sorter lists its large groups here.
template <int NT>
__device__ void block_scan_small_list(u32* a, u32 cnt, u32* red, u32 T, u32* list, u32* nlist, u32 cap, u32* over) {
    const u32 i0 = threadIdx.x * 16, r = (threadIdx.x >> 1) & 15;
    u32 v[16], s = 0, head = 0, bm = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const u32 e = (j + r) & 15;
        v[j] = (i0 + e < cnt) ? a[i0 + e] : 0u;
        s += v[j];
        if (e < r) head += v[j];
        bm |= (v[j] >= T ? 1u : 0u) << e;
    }
    u32 tot;
    const u32 packed = block_exclusive_scan<NT>(s | ((u32)__popc(bm) << 16), red, &tot);
    const u32 base = packed & 0xffffu;
    u32 lb = packed >> 16;  // list slot of this thread's first big element
    u32 run = base + head;  // prefix of element r
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const u32 e = (j + r) & 15;
        if (e == 0) run = base;
        if (i0 + e < cnt) a[i0 + e] = run;
        run += v[j];
    }
    while (bm) {
        const u32 e = __ffs(bm) - 1;
        bm &= bm - 1;
        if (lb < cap) list[lb] = i0 + e;
        ++lb;
    }
    if (threadIdx.x == 0) {
        *nlist = tot >> 16;
        if ((tot >> 16) > cap) *over = 1u;
    }
    __syncthreads();
}

// ------------------------------------------------------------------ CTA bitonic sort of (key, tag)
// N a power of two, records in shared memory; ascending by (key, tag).  Every thread step is one
// comparator (x, x + j): t's bits below j stay, the bits above move up one place.
template <class U>
__device__ void cta_bitonic_kt(U* tk, u32* tt, u32 N) {
    for (u32 kk = 2; kk <= N; kk <<= 1) {
        for (u32 j = kk >> 1; j > 0; j >>= 1) {
            for (u32 t = threadIdx.x; t < N / 2; t += blockDim.x) {
                const u32 x = ((t & ~(j - 1)) << 1) | (t & (j - 1)), y = x | j;
                const bool asc = (x & kk) == 0;
                const U a = tk[x], b = tk[y];
                const u32 ta = tt[x], tb = tt[y];
                const bool gt = a > b || (a == b && ta > tb);
                if (gt == asc) { tk[x] = b; tk[y] = a; tt[x] = tb; tt[y] = ta; }
            }
            __syncthreads();
        }
    }
}

// ------------------------------------------------------------------ a1+a2: hash-set form
// I = the first m distinct values of c_j = floor(H(seed,1,j) n / 2^64), j = 0, 1, ... (reading
// Q1).  Draw j is "first" iff no j' < j has c_j' = c_j.  An open-addressing hash set keyed by c
// keeps the smallest j of every c; an entry holds ~((c << 32) | j) so that the empty slot is 0
// (one memset) and "smallest j" is an atomicMax.  The first draws ranked by j are the members of
// I; the records T[rank] = (x[c], c) are written in draw order, a uniformly random order that
// the coarse level of the sample sort relies on (T's order is not part of any result).
__device__ __forceinline__ u32 ht_slot(u64 c, u32 lg) { return (u32)((c * 0x9e3779b97f4a7c15ull) >> (64 - lg)); }
__device__ __forceinline__ u64 ros_draw_c(u64 seed, u64 j, u64 n) { return __umul64hi(rng_H(seed, 1, j), n); }

__global__ void k_ros_draw(u64* tab, u32 lg, u32 M, u64 n, u64 seed) {
    PDL_PROLOGUE();
    const u32 j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= M) return;
    const u64 c = ros_draw_c(seed, j, n);
    const u64 e = ~((c << 32) | j);
    const u32 mask = (1u << lg) - 1;
    for (u32 s = ht_slot(c, lg);; s = (s + 1) & mask) {
        u64 v = __ldcg(tab + s);
        if (v == 0) {
            v = atomicCAS((unsigned long long*)(tab + s), 0ull, (unsigned long long)e);
            if (v == 0) return;
        }
        if ((~v >> 32) == c) {
            atomicMax((unsigned long long*)(tab + s), (unsigned long long)e);
            return;
        }
    }
}

__device__ __forceinline__ u32 ht_min_j(const u64* tab, u32 lg, u64 c) {
    const u32 mask = (1u << lg) - 1;
    for (u32 s = ht_slot(c, lg);; s = (s + 1) & mask) {
        const u64 v = ~__ldcg(tab + s);
        if ((v >> 32) == c) return (u32)v;
    }
}

constexpr int TK_NT = 1024;
// per block of TK_NT draws: the warps' masks of first draws, and the block's count
__global__ void __launch_bounds__(TK_NT) k_ros_first(const u64* tab, u32 lg, u32 M, u64 n, u64 seed, u32* bits, u32* bcnt) {
    PDL_PROLOGUE();
    __shared__ u32 wcnt[TK_NT / 32];
    const u32 j = blockIdx.x * TK_NT + threadIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    bool first = false;
    if (j < M) first = ht_min_j(tab, lg, ros_draw_c(seed, j, n)) == j;
    const u32 mask = __ballot_sync(0xffffffffu, first);
    if (lane == 0) { bits[j >> 5] = mask; wcnt[wid] = __popc(mask); }
    __syncthreads();
    if (wid == 0) {
        u32 v = wcnt[lane];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) bcnt[blockIdx.x] = v;
    }
}

// rank(j) among the first draws = the blocks before + the warps before + the lanes before; a
// first draw of rank < m is a member of I.  Record layout: 32-bit keys one word
// (ord key << 32 | c), 64-bit keys a key word and a tag (c).  DIST: only indices inside the
// shard [offset, offset + nl) contribute (rec slots of other ranks stay zero; the all-reduce SUM
// over ranks assembles T, 2 words per record for 64-bit keys).
template <int DT, bool DIST>
__global__ void __launch_bounds__(TK_NT) k_ros_take(const u32* bits, const u32* bcnt, u32 M, u64 n, u64 seed, u32 m,
                                                     const typename Codec<DT>::U* x, u64 offset, u32 nl, u64* tk, u32* tt,
                                                     u32* status, PeerOut po) {
    PDL_PROLOGUE();
    typedef typename Codec<DT>::U U;
    __shared__ u32 red[TK_NT / 32], wpre[TK_NT / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    u32 s = 0;
    for (u32 b = threadIdx.x; b < blockIdx.x; b += TK_NT) s += bcnt[b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const u32 j = blockIdx.x * TK_NT + threadIdx.x;
    const u32 mask = bits[j >> 5];
    if (lane == 0) { red[wid] = s; wpre[wid] = __popc(mask); }
    __syncthreads();
    if (wid == 0) {
        u32 b = red[lane], w = wpre[lane], x2 = w;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 y = __shfl_up_sync(0xffffffffu, x2, o);
            if (lane >= o) x2 += y;
        }
        wpre[lane] = b + x2 - w;  // exclusive prefix of warp `lane` in the whole draw order
        if (blockIdx.x + 1 == gridDim.x && lane == 31 && b + x2 < m) st_set(status, ST_SAMPLE_SHORT);
    }
    __syncthreads();
    if (!((mask >> lane) & 1u)) return;
    const u32 rank = wpre[wid] + __popc(mask & ((1u << lane) - 1));
    if (rank >= m) return;
    const u64 c = ros_draw_c(seed, j, n);
    if (DIST && (c < offset || c >= offset + nl)) return;
    const U k = load_key<DT>(x, c - offset);
    if (DIST) {
        put_rec<sizeof(U) == 8>(po, rank, (u64)k, c);
    } else if (sizeof(U) == 4) {
        tk[rank] = ((u64)k << 32) | c;
    } else {
        tk[rank] = (u64)k;
        tt[rank] = (u32)c;
    }
}

// ------------------------------------------------------------------ a1+a2: direct-address form
// For samples that are a large fraction of n (ps-1 up to n; the draws then number up to
// n(ln n + 1)), the set of draws is a direct-address table over the n indices: minj[c] = the
// smallest draw number j with c_j = c (atomicMin; empty = ~0).  I = the m indices with the m
// smallest minj, i.e. {c : minj[c] <= j*} where j* is the m-th smallest minj (radix select over
// the table); the records are written in index order (the sample sort then draws its coarse
// splitters at random positions, Selector::stride = 0).  Same set as the hash-set form.
__global__ void k_ros_draw_direct(u64* minj, u64 M, u64 n, u64 seed) {
    PDL_PROLOGUE();
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 j = (u64)blockIdx.x * blockDim.x + threadIdx.x; j < M; j += stride)
        atomicMin((unsigned long long*)(minj + ros_draw_c(seed, j, n)), (unsigned long long)j);
}

// radix select of j*: sel = {prefix, rank remaining, shift}; pass k histograms digit
// (minj >> sh) & (RS_BINS-1) of the entries whose bits above sh+RS_BITS equal the prefix
constexpr u32 RS_BITS = 13, RS_BINS = 1u << RS_BITS;
struct RSel { u64 prefix; u64 rank; u32 hibits; u32 found; };  // hibits: bits fixed so far (from the top)
__global__ void __launch_bounds__(1024) k_rsel_hist(const u64* minj, u64 n, const RSel* sel, u32 sh, u32* ghist) {
    PDL_PROLOGUE();
    __shared__ u32 h[RS_BINS];
    for (u32 i = threadIdx.x; i < RS_BINS; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const RSel sv = *sel;
    const u32 top = sh + RS_BITS;  // entries must match the prefix in bits [top, 64)
    for (u64 c = (u64)blockIdx.x * blockDim.x + threadIdx.x; c < n; c += (u64)gridDim.x * blockDim.x) {
        const u64 v = minj[c];
        if (v == ~0ull) continue;
        if (top < 64 && (v >> top) != (sv.prefix >> top)) continue;
        atomicAdd(&h[(u32)(v >> sh) & (RS_BINS - 1)], 1u);
    }
    __syncthreads();
    for (u32 i = threadIdx.x; i < RS_BINS; i += blockDim.x)
        if (h[i]) atomicAdd(&ghist[i], h[i]);
}
__global__ void k_rsel_init(RSel* sel, u64 rank, u32* ghist) {
    PDL_PROLOGUE();
    if (threadIdx.x == 0) {
        RSel v;
        v.prefix = 0; v.rank = rank; v.hibits = 0; v.found = 0;
        *sel = v;
    }
    for (u32 i = threadIdx.x; i < RS_BINS; i += blockDim.x) ghist[i] = 0;
}
// one CTA: the digit holding rank sel.rank (0-based) -> prefix; zeroes ghist for the next pass
__global__ void __launch_bounds__(1024) k_rsel_pick(RSel* sel, u32 sh, u32* ghist, u32* status, u32 last) {
    PDL_PROLOGUE();
    __shared__ u32 red[33];
    __shared__ u32 s_d;
    __shared__ u64 s_before;
    // per thread 16 consecutive bins; exclusive scan of the thread sums
    const u32 per = RS_BINS / 1024;
    u32 loc[RS_BINS / 1024], sum = 0;
#pragma unroll
    for (u32 q = 0; q < per; ++q) { loc[q] = ghist[threadIdx.x * per + q]; sum += loc[q]; }
    u32 tot = 0;
    const u32 ex = block_exclusive_scan<1024>(sum, red, &tot);
    if (threadIdx.x == 0) { s_d = 0xffffffffu; s_before = 0; }
    __syncthreads();
    const u64 r = sel->rank;
    if ((u64)ex <= r && r < (u64)ex + sum) {
        u32 run = ex;
        for (u32 q = 0; q < per; ++q) {
            if (r < (u64)run + loc[q]) { s_d = threadIdx.x * per + q; s_before = run; break; }
            run += loc[q];
        }
    }
    __syncthreads();
#pragma unroll
    for (u32 q = 0; q < per; ++q) ghist[threadIdx.x * per + q] = 0;
    if (threadIdx.x == 0) {
        RSel sv = *sel;
        if (s_d == 0xffffffffu) {  // fewer than rank+1 entries: not enough distinct draws
            st_set(status, ST_SAMPLE_SHORT);
            sv.found = 0;
            sv.prefix = 0;
        } else {
            const u64 mask = (sh + RS_BITS >= 64) ? ~0ull : ((1ull << (sh + RS_BITS)) - 1);
            sv.prefix = (sv.prefix & ~mask) | ((u64)s_d << sh);
            sv.rank = r - s_before;
            sv.found = last;
        }
        *sel = sv;
    }
}

constexpr u32 DT_NT = 1024, DT_PER = 8;  // compaction: 8192 table entries per block
// per block of DT_NT*DT_PER entries: the number of members (minj <= j*)
__global__ void __launch_bounds__(DT_NT) k_direct_count(const u64* minj, u64 n, const RSel* sel, u32* bcnt) {
    PDL_PROLOGUE();
    __shared__ u32 red[33];
    const u64 js = sel->found ? sel->prefix : 0ull;
    const bool any = sel->found != 0;
    u32 cnt = 0;
    const u64 b0 = (u64)blockIdx.x * DT_NT * DT_PER;
#pragma unroll
    for (u32 q = 0; q < DT_PER; ++q) {
        const u64 c = b0 + q * DT_NT + threadIdx.x;
        if (any && c < n && minj[c] <= js) ++cnt;
    }
    u32 tot = 0;
    block_exclusive_scan<DT_NT>(cnt, red, &tot);
    if (threadIdx.x == 0) bcnt[blockIdx.x] = tot;
}
// records of the members in index order; DIST: only the shard [offset, offset + nl) writes
template <int DT, bool DIST>
__global__ void __launch_bounds__(DT_NT) k_direct_take(const u64* minj, u64 n, const RSel* sel, const u32* bscan,
                                                        const typename Codec<DT>::U* x, u64 offset, u32 nl, u64* tk,
                                                        u32* tt, PeerOut po) {
    PDL_PROLOGUE();
    typedef typename Codec<DT>::U U;
    __shared__ u32 red[33];
    const u64 js = sel->found ? sel->prefix : 0ull;
    const bool any = sel->found != 0;
    const u64 b0 = (u64)blockIdx.x * DT_NT * DT_PER;
    bool mem[DT_PER];
    u32 cnt = 0;
#pragma unroll
    for (u32 q = 0; q < DT_PER; ++q) {
        // thread t owns the consecutive entries b0 + t*DT_PER + q (index order inside the block)
        const u64 c = b0 + (u64)threadIdx.x * DT_PER + q;
        mem[q] = any && c < n && minj[c] <= js;
        cnt += mem[q] ? 1u : 0u;
    }
    u32 rank = bscan[blockIdx.x] + block_exclusive_scan<DT_NT>(cnt, red, nullptr);
#pragma unroll
    for (u32 q = 0; q < DT_PER; ++q) {
        if (!mem[q]) continue;
        const u64 c = b0 + (u64)threadIdx.x * DT_PER + q;
        const u32 rk = rank++;
        if (DIST && (c < offset || c >= offset + nl)) continue;
        const U k = load_key<DT>(x, c - offset);
        if (DIST) {
            put_rec<sizeof(U) == 8>(po, rk, (u64)k, c);
        } else if (sizeof(U) == 4) {
            tk[rk] = ((u64)k << 32) | c;
        } else {
            tk[rk] = (u64)k;
            tt[rk] = (u32)c;
        }
    }
}
// exclusive scan of the block counts (one CTA); a shortfall of members sets ST_SAMPLE_SHORT
__global__ void __launch_bounds__(1024) k_direct_scan(u32* bcnt, u32 nb, u32 m, u32* status) {
    PDL_PROLOGUE();
    __shared__ u32 red[33];
    block_scan_array<1024>(bcnt, nb, red);
    if (threadIdx.x == 0 && bcnt[nb] != m) st_set(status, ST_SAMPLE_SHORT);
}

// ------------------------------------------------------------------ register sorting networks
template <class U> __device__ __forceinline__ U shfl_xor_any(U x, int o) {
    if (sizeof(U) == 8) return (U)__shfl_xor_sync(0xffffffffu, (unsigned long long)x, o);
    return (U)__shfl_xor_sync(0xffffffffu, (u32)x, o);
}
template <class U, bool KV> struct Elem;
template <class U> struct Elem<U, false> {
    U k;
    __device__ __forceinline__ bool lt(const Elem& o) const { return k < o.k; }
    __device__ __forceinline__ static Elem inf() { Elem e; e.k = umax_of<U>(); return e; }
    __device__ __forceinline__ Elem shfl_xor(int m) const { Elem e; e.k = shfl_xor_any(k, m); return e; }
};
template <class U> struct Elem<U, true> {
    U k; u32 i, v;
    __device__ __forceinline__ bool lt(const Elem& o) const { return k < o.k || (k == o.k && i < o.i); }
    __device__ __forceinline__ static Elem inf() { Elem e; e.k = umax_of<U>(); e.i = 0xffffffffu; e.v = 0; return e; }
    __device__ __forceinline__ Elem shfl_xor(int m) const {
        Elem e;
        e.k = shfl_xor_any(k, m);
        e.i = __shfl_xor_sync(0xffffffffu, i, m);
        e.v = __shfl_xor_sync(0xffffffffu, v, m);
        return e;
    }
};

template <class E> __device__ __forceinline__ void cex(E& a, E& b) {
    if (b.lt(a)) { E t = a; a = b; b = t; }
}

// Batcher's odd-even merge network for 8 inputs (19 comparators)
template <class E> __device__ __forceinline__ void network8(E (&a)[8]) {
    cex(a[0], a[1]); cex(a[2], a[3]); cex(a[4], a[5]); cex(a[6], a[7]);
    cex(a[0], a[2]); cex(a[1], a[3]); cex(a[4], a[6]); cex(a[5], a[7]);
    cex(a[1], a[2]); cex(a[5], a[6]);
    cex(a[0], a[4]); cex(a[1], a[5]); cex(a[2], a[6]); cex(a[3], a[7]);
    cex(a[2], a[4]); cex(a[3], a[5]);
    cex(a[1], a[2]); cex(a[3], a[4]); cex(a[5], a[6]);
}

// Batcher's odd-even merge sort for 16 inputs: two 8-sorts (19 + 19 comparators) and the
// odd-even merge of the halves (25 comparators), 63 in all
template <class E> __device__ __forceinline__ void network16(E (&a)[16]) {
    E* lo = a;
    E* hi = a + 8;
    E (&l8)[8] = *reinterpret_cast<E(*)[8]>(lo);
    E (&h8)[8] = *reinterpret_cast<E(*)[8]>(hi);
    network8(l8);
    network8(h8);
    // odd-even merge of a[0..8) and a[8..16)
#pragma unroll
    for (int i = 0; i < 8; ++i) cex(a[i], a[i + 8]);
    cex(a[4], a[8]); cex(a[5], a[9]); cex(a[6], a[10]); cex(a[7], a[11]);
    cex(a[2], a[4]); cex(a[3], a[5]); cex(a[6], a[8]); cex(a[7], a[9]); cex(a[10], a[12]); cex(a[11], a[13]);
    cex(a[1], a[2]); cex(a[3], a[4]); cex(a[5], a[6]); cex(a[7], a[8]); cex(a[9], a[10]); cex(a[11], a[12]);
    cex(a[13], a[14]);
}

// bitonic sort of 32*R elements held as a[r] at lane: element index e = r*32 + lane
template <class E, int R>
__device__ __forceinline__ void warp_bitonic(E (&a)[R]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 2; k <= 32 * R; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
                const int jr = j >> 5;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if ((r & jr) == 0) {
                        const int e = r * 32 + lane;
                        const bool asc = (e & k) == 0;
                        E x = a[r], y = a[r | jr];
                        const bool sw = asc ? y.lt(x) : x.lt(y);
                        if (sw) { a[r] = y; a[r | jr] = x; }
                    }
                }
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int e = r * 32 + lane;
                    const bool asc = (e & k) == 0;
                    const bool lower = (lane & j) == 0;
                    E o = a[r].shfl_xor(j);
                    const bool keep_min = (lower == asc);
                    const bool take = keep_min ? o.lt(a[r]) : a[r].lt(o);
                    if (take) a[r] = o;
                }
            }
        }
    }
}

// One element per thread (N == blockDim.x, a power of two >= 32): the comparators of distance
// j < 32 exchange through warp shuffles (no block barrier); only j >= 32 goes through shared
// memory.  55 barrier-separated steps of the plain network become 15 for N = 1024.
template <class U>
__device__ void cta_bitonic_1pt(U* tk, u32* tt, u32 N) {
    const u32 e = threadIdx.x;
    U k = tk[e];
    u32 t = tt[e];
    for (u32 kk = 2; kk <= N; kk <<= 1) {
        for (u32 j = kk >> 1; j > 0; j >>= 1) {
            U ok;
            u32 ot;
            if (j >= 32) {
                __syncthreads();
                tk[e] = k; tt[e] = t;
                __syncthreads();
                ok = tk[e ^ j]; ot = tt[e ^ j];
            } else {
                ok = shfl_xor_any(k, (int)j);
                ot = __shfl_xor_sync(0xffffffffu, t, (int)j);
            }
            const bool asc = (e & kk) == 0, lower = (e & j) == 0;
            const bool o_less = ok < k || (ok == k && ot < t);
            // the lower slot of an ascending pair keeps the minimum, etc.
            const bool take = (lower == asc) ? o_less : (!o_less && !(ok == k && ot == t));
            if (take) { k = ok; t = ot; }
        }
    }
    __syncthreads();
    tk[e] = k; tt[e] = t;
    __syncthreads();
}

// ------------------------------------------------------------------ a3: sample sort (coarse level)
// The m sample records (key word, tag) are sorted by (key, tag) in two steps: G coarse buckets,
// then every coarse bucket by the bucket sorter.  Coarse splitter i = CS[(i+1)Q/G - 1], CS =
// the first Q = min(m, 1024) records of T sorted (a uniform random subset, T being in draw
// order).  Every CTA of k_sel_count sorts CS itself (a 1024-record bitonic network, ~1 us) so
// no separate launch is needed; CTA 0 stores the coarse splitters for k_sel_scatter.
constexpr u32 SEL_Q = 1024, SEL_PER = 4096, SEL_GMAX = 128;

__device__ __forceinline__ bool rec_lt(u64 ak, u32 at, u64 bk, u32 bt) { return ak < bk || (ak == bk && at < bt); }

__device__ __forceinline__ u32 coarse_of(const u64* ck, const u32* ct, u32 nc, u64 k, u32 t) {
    u32 lo = 0, cnt = nc;
    while (cnt > 0) {
        const u32 half = cnt >> 1, mid = lo + half;
        if (rec_lt(ck[mid], ct[mid], k, t)) { lo = mid + 1; cnt -= half + 1; } else cnt = half;
    }
    return lo;
}

template <bool TAG>
__global__ void __launch_bounds__(1024) k_sel_count(const u64* tk, const u32* tt, u32 m, u32 G, u32 stride, u64* csk, u32* cst,
                                                    uint8_t* cb, u32* gcnt) {
    PDL_PROLOGUE();
    __shared__ u64 qk[SEL_Q];
    __shared__ u32 qt[SEL_Q];
    __shared__ u32 h[SEL_GMAX];
    const u32 Q = min(m, SEL_Q);
    if (G > 1) {
        u32 N = 1;
        while (N < Q) N <<= 1;
        for (u32 i = threadIdx.x; i < N; i += blockDim.x) {
            // records i (stride 1: T in random order, ROS) or at random positions (stride 0: T made
            // of sorted runs, DRO's regular samples, where fixed offsets would be biased)
            const u64 r = stride ? (u64)i * stride : __umul64hi(rng_H(0x5e1ec7ull, 90, i), (u64)m);
            qk[i] = i < Q ? tk[r] : ~0ull;
            qt[i] = i < Q ? (TAG ? tt[r] : 0u) : 0xffffffffu;
        }
        __syncthreads();
        if (N == blockDim.x) cta_bitonic_1pt<u64>(qk, qt, N);
        else cta_bitonic_kt<u64>(qk, qt, N);
        // coarse splitters in place at the front (reads before writes: ranks are increasing)
        u64 ck = 0;
        u32 ct = 0;
        if (threadIdx.x + 1 < G) {
            const u32 r = (u32)(((u64)(threadIdx.x + 1) * Q) / G) - 1;
            ck = qk[r];
            ct = qt[r];
        }
        __syncthreads();
        if (threadIdx.x + 1 < G) {
            qk[threadIdx.x] = ck;
            qt[threadIdx.x] = ct;
            if (blockIdx.x == 0) { csk[threadIdx.x] = ck; cst[threadIdx.x] = ct; }
        }
    }
    for (u32 g = threadIdx.x; g < G; g += blockDim.x) h[g] = 0;
    __syncthreads();
    const u32 b0 = blockIdx.x * SEL_PER, b1 = min(m, b0 + SEL_PER);
    for (u32 i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
        const u32 g = coarse_of(qk, qt, G - 1, tk[i], TAG ? tt[i] : 0u);
        cb[i] = (uint8_t)g;
        atomicAdd(&h[g], 1u);
    }
    __syncthreads();
    for (u32 g = threadIdx.x; g < G; g += blockDim.x)
        if (h[g]) atomicAdd(&gcnt[g], h[g]);
}

// coarse buckets -> T2 (bucket-contiguous, order inside a bucket irrelevant: every bucket is
// sorted next); CTA 0 writes the bucket sorter's work list (bounds = the coarse splitters' keys)
template <bool TAG>
__global__ void __launch_bounds__(1024) k_sel_scatter(const u64* tk, const u32* tt, u32 m, u32 G, const uint8_t* cb,
                                                      const u32* gcnt, u32* gcur, const u64* csk, u64* ok, u32* ot,
                                                      u32* oi, Bucket* list, u32* nlist) {
    PDL_PROLOGUE();
    __shared__ u32 st[SEL_GMAX + 1], h[SEL_GMAX], base[SEL_GMAX];
    if (threadIdx.x == 0) {
        u32 run = 0;
        for (u32 g = 0; g < G; ++g) { st[g] = run; run += gcnt[g]; }
        st[G] = run;
    }
    for (u32 g = threadIdx.x; g < G; g += blockDim.x) h[g] = 0;
    __syncthreads();
    const u32 b0 = blockIdx.x * SEL_PER, b1 = min(m, b0 + SEL_PER);
    constexpr u32 IT = SEL_PER / 1024;
    u32 gg[IT], rr[IT];
#pragma unroll
    for (u32 q = 0; q < IT; ++q) {
        const u32 i = b0 + q * 1024 + threadIdx.x;
        if (i < b1) { gg[q] = cb[i]; rr[q] = atomicAdd(&h[gg[q]], 1u); }
    }
    __syncthreads();
    for (u32 g = threadIdx.x; g < G; g += blockDim.x) base[g] = h[g] ? atomicAdd(&gcur[g], h[g]) : 0u;
    __syncthreads();
#pragma unroll
    for (u32 q = 0; q < IT; ++q) {
        const u32 i = b0 + q * 1024 + threadIdx.x;
        if (i < b1) {
            const u32 d = st[gg[q]] + base[gg[q]] + rr[q];
            ok[d] = tk[i];
            if (TAG) { ot[d] = tt[i]; oi[d] = tt[i]; }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        u32 nb = 0;
        for (u32 g = 0; g < G; ++g) {
            const u32 len = st[g + 1] - st[g];
            if (len == 0) continue;
            Bucket b;
            b.beg = st[g]; b.len = len; b.buf = 1;  // sorted into buffer 0 (not in place: windows allowed)
            b.level = (g == 0 || g + 1 == G) ? BK_LOOSE : 0u;
            b.lo = g ? csk[g - 1] : 0ull;
            b.hi = g + 1 < G ? csk[g] : ~0ull;
            list[nb++] = b;
        }
        nlist[0] = nb;
        nlist[1] = 0;
    }
}

// a3+a4 in one launch (32-bit keys, packed records ord(key) << 32 | index, all distinct): the
// same coarse buckets as k_sel_count / k_sel_scatter, then every coarse bucket sorted by one CTA
// and S[q] = T[(q+1)s/f - 1] read off at once.  The steps are separated by grid-wide barriers
// (cooperative launch: every CTA is resident) instead of four launches and the bucket sorter's
// list machinery (sample phase 0.128 ms, most of it launch ramps and one-bucket-per-CTA tails).
constexpr u32 SF_NT = 1024, SF_MAXB = 8192, SF_NG = 4096, SF_IT = 2, SF_BIG = 256;

// grid-wide barrier number k (1, 2, ...) on a counter zeroed before the launch
// (bounded wait: a CTA that is never scheduled cannot hang the device; status ST_LIST_OVER)
__device__ __forceinline__ void grid_sync(u32* ctr, u32 k, u32* status) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        for (u32 it = 0; *(volatile u32*)ctr < k * gridDim.x; ++it) {
            if (it > (1u << 24)) { st_set(status, ST_LIST_OVER); break; }
            __nanosleep(64);
        }
        __threadfence();
    }
    __syncthreads();
}

// ascending sort of a[0..len) of distinct u64 (shared or global memory) by a bitonic network
// whose comparators all point up (the first step of every merge compares i with its mirror), so
// the virtual +inf padding beyond len never moves and len need not be a power of two
template <int NT>
__device__ void cta_sort_u64(u64* a, u32 len) {
    u32 N = 1;
    while (N < len) N <<= 1;
    for (u32 kk = 2; kk <= N; kk <<= 1) {
        const u32 hk = kk >> 1;
        for (u32 t = threadIdx.x; t < N / 2; t += NT) {
            const u32 x = (t / hk) * kk + (t % hk), y = (t / hk) * kk + kk - 1 - (t % hk);
            if (y < len) { const u64 u = a[x], v = a[y]; if (v < u) { a[x] = v; a[y] = u; } }
        }
        __syncthreads();
        for (u32 j = kk >> 2; j > 0; j >>= 1) {
            for (u32 t = threadIdx.x; t < N / 2; t += NT) {
                const u32 x = ((t & ~(j - 1)) << 1) | (t & (j - 1)), y = x + j;
                if (y < len) { const u64 u = a[x], v = a[y]; if (v < u) { a[x] = v; a[y] = u; } }
            }
            __syncthreads();
        }
    }
}

// cta_bitonic_1pt for distinct u64 keys without tags (N == blockDim.x)
__device__ void cta_bitonic_1pt_u64(u64* a, u32 N) {
    const u32 e = threadIdx.x;
    u64 k = a[e];
    for (u32 kk = 2; kk <= N; kk <<= 1) {
        for (u32 j = kk >> 1; j > 0; j >>= 1) {
            u64 o;
            if (j >= 32) {
                __syncthreads();
                a[e] = k;
                __syncthreads();
                o = a[e ^ j];
            } else {
                o = shfl_xor_any(k, (int)j);
            }
            k = (((e & kk) == 0) == ((e & j) == 0)) ? min(k, o) : max(k, o);
        }
    }
    __syncthreads();
    a[e] = k;
    __syncthreads();
}

// grid = G CTAs (<= SEL_GMAX, m <= G * SF_NT * SF_IT); gcnt[G] and *gbar zeroed before the launch;
// t2 = coarse-bucket order (workspace), ts = T sorted; S[q] = ts[(q+1)s/f - 1] for q < P-1
#ifdef OVS_SF_PROF
__device__ unsigned long long g_sfprof[8];
#define SF_PROBE(i) if (threadIdx.x == 0) { const long long n_ = clock64(); atomicAdd(&g_sfprof[i], (unsigned long long)(n_ - sf_t_)); sf_t_ = n_; }
#else
#define SF_PROBE(i)
#endif
template <int DT>
__global__ void __launch_bounds__(SF_NT, 1) k_sel_fused(const u64* tk, u32 m, u32* gcnt, u32* gbar, u64* t2, u64* ts,
                                                        u32 P, u32 s, u32 f, typename Codec<DT>::U* sk, u32* st,
                                                        u32* status) {
    typedef typename Codec<DT>::U U;
    extern __shared__ __align__(16) u64 sbuf[];  // 2 x SF_MAXB records, SF_NG group counters
    __shared__ u64 qk[SEL_Q];
    __shared__ u32 qt[SEL_Q];
    __shared__ u32 h[SEL_GMAX], base[SEL_GMAX], start[SEL_GMAX + 1];
    __shared__ u32 red[SF_NT / 32 + 1], big[SF_BIG], nbig, over;
    __shared__ u64 rmn[SF_NT / 32], rmx[SF_NT / 32];
#ifdef OVS_SF_PROF
    long long sf_t_ = clock64();
#endif
    const u32 G = gridDim.x;
    constexpr u32 RC = SF_IT;
    u64 rc[RC];
    u32 rv = 0;  // valid records of this thread (bit q)
    u32 nbar = 0;
    // 1. coarse splitters from the first Q records (T in draw order: a uniform random subset)
    const u32 Q = min(m, SEL_Q);
    if (G > 1) {
        for (u32 i = threadIdx.x; i < SF_NT; i += SF_NT) qk[i] = i < Q ? tk[i] : ~0ull;  // padding sorts last
        __syncthreads();
        cta_bitonic_1pt_u64(qk, SF_NT);
        u64 ck = 0;
        if (threadIdx.x + 1 < G) ck = qk[(u32)(((u64)(threadIdx.x + 1) * Q) / G) - 1];
        __syncthreads();
        if (threadIdx.x + 1 < G) { qk[threadIdx.x] = ck; qt[threadIdx.x] = 0u; }
    }
    SF_PROBE(0)
    for (u32 g = threadIdx.x; g < G; g += SF_NT) h[g] = 0;
    __syncthreads();
    // 2. this CTA's slice of T per coarse bucket; the CTA's run inside each bucket claimed
    {
        const u32 b0 = (u32)(((u64)m * blockIdx.x) / G), b1 = (u32)(((u64)m * (blockIdx.x + 1)) / G);
#pragma unroll
        for (u32 q = 0; q < RC; ++q) {
            const u32 i = b0 + q * SF_NT + threadIdx.x;
            if (i < b1) { rc[q] = tk[i]; rv |= 1u << q; }
        }
    }
    u32 gg[RC], rr[RC];
#pragma unroll
    for (u32 q = 0; q < RC; ++q) {
        if ((rv >> q) & 1u) {
            gg[q] = coarse_of(qk, qt, G - 1, rc[q], 0u);
            rr[q] = atomicAdd(&h[gg[q]], 1u);
        }
    }
    __syncthreads();
    for (u32 g = threadIdx.x; g < G; g += SF_NT) base[g] = h[g] ? atomicAdd(&gcnt[g], h[g]) : 0u;
    SF_PROBE(1)
    grid_sync(gbar, ++nbar, status);
    SF_PROBE(2)
    // 3. bucket starts (every CTA scans the G totals) and the scatter into coarse-bucket order
    if (threadIdx.x < 32) {
        u32 v[SEL_GMAX / 32], sum = 0;
#pragma unroll
        for (u32 j = 0; j < SEL_GMAX / 32; ++j) {
            const u32 g = threadIdx.x * (SEL_GMAX / 32) + j;
            v[j] = g < G ? __ldcg(&gcnt[g]) : 0u;
            sum += v[j];
        }
        u32 x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 y = __shfl_up_sync(0xffffffffu, x, o);
            if ((int)threadIdx.x >= o) x += y;
        }
        u32 run = x - sum;
#pragma unroll
        for (u32 j = 0; j < SEL_GMAX / 32; ++j) {
            const u32 g = threadIdx.x * (SEL_GMAX / 32) + j;
            if (g < G) start[g] = run;
            run += v[j];
        }
        if (threadIdx.x == 31) start[G] = x;  // = m
    }
    __syncthreads();
#pragma unroll
    for (u32 q = 0; q < RC; ++q)
        if ((rv >> q) & 1u) t2[start[gg[q]] + base[gg[q]] + rr[q]] = rc[q];
    SF_PROBE(3)
    grid_sync(gbar, ++nbar, status);
    SF_PROBE(4)
    // 4. CTA b sorts coarse bucket b: a counting sort by a fine digit of (record - min) spreads it
    // over ~len/2 groups (the records are a random sample: mostly 0-4 per group), then groups of
    // <= 8 by one thread (Batcher network), larger ones (listed by the scan) by a warp or the CTA.
    // A bucket over SF_MAXB records (the 8-records-per-splitter coarse sample makes that
    // vanishingly rare) is sorted in place in global memory by the bitonic network instead.
    const u32 bs = start[blockIdx.x], len = start[blockIdx.x + 1] - bs;
    u64* a = t2 + bs;
    if (len <= SF_MAXB) {
        u64* A = sbuf;
        u64* Bv = sbuf + SF_MAXB;
        u32* cnt = (u32*)(sbuf + 2 * SF_MAXB);
        u64 mn = ~0ull, mx = 0;
        for (u32 i = threadIdx.x; i < len; i += SF_NT) {
            const u64 v = __ldcg(t2 + bs + i);
            A[i] = v;
            mn = min(mn, v);
            mx = max(mx, v);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) { mn = min(mn, shfl_xor_any(mn, o)); mx = max(mx, shfl_xor_any(mx, o)); }
        if ((threadIdx.x & 31) == 0) { rmn[threadIdx.x >> 5] = mn; rmx[threadIdx.x >> 5] = mx; }
        u32 ng = 32;
        while (ng < SF_NG && ng * 2 < len) ng <<= 1;
        for (u32 g = threadIdx.x; g < ng; g += SF_NT) cnt[g] = 0;
        if (threadIdx.x == 0) over = 0;
        __syncthreads();
        mn = rmn[0]; mx = rmx[0];
        for (u32 w = 1; w < SF_NT / 32; ++w) { mn = min(mn, rmn[w]); mx = max(mx, rmx[w]); }
        // digit = floor((x - mn) * ng / (mx - mn + 1)), a fixed-point multiply-high: monotone
        const double mq = (double)ng * 18446744073709551616.0 / ((double)(mx - mn) + 1.0);
        const u64 mult = mq >= 18446744073709549568.0 ? 0xffffffffffffffffull : (u64)mq;
        auto digit = [&](u64 x) -> u32 { return min((u32)__umul64hi(x - mn, mult), ng - 1); };
        for (u32 i = threadIdx.x; i < len; i += SF_NT) atomicAdd(&cnt[digit(A[i])], 1u);
        __syncthreads();
        block_scan_small_list<SF_NT>(cnt, ng, red, 9u, big, &nbig, SF_BIG, &over);  // cnt[g] = start
        for (u32 i = threadIdx.x; i < len; i += SF_NT) {
            const u64 v = A[i];
            Bv[atomicAdd(&cnt[digit(v)], 1u)] = v;  // afterwards cnt[g] = end of group g
        }
        __syncthreads();
        typedef Elem<u64, false> E;
        for (u32 g = threadIdx.x; g < ng; g += SF_NT) {
            const u32 gs = g ? cnt[g - 1] : 0u, gl = cnt[g] - gs;
            if (gl < 2 || gl > 8) continue;
            E e[8];
#pragma unroll
            for (u32 q = 0; q < 8; ++q) e[q].k = q < gl ? Bv[gs + q] : ~0ull;
            network8(e);
#pragma unroll
            for (u32 q = 0; q < 8; ++q)
                if (q < gl) Bv[gs + q] = e[q].k;
        }
        const u32 nl = over ? ng : min(nbig, SF_BIG);  // list overflow: scan every group
        const int lane = threadIdx.x & 31;
        for (u32 q = threadIdx.x >> 5; q < nl; q += SF_NT / 32) {
            const u32 g = over ? q : big[q];
            const u32 gs = g ? cnt[g - 1] : 0u, gl = cnt[g] - gs;
            if (gl <= 8 || gl > 256) continue;
            E e[8];
#pragma unroll
            for (u32 r = 0; r < 8; ++r) { const u32 x = r * 32 + lane; e[r].k = x < gl ? Bv[gs + x] : ~0ull; }
            warp_bitonic<E, 8>(e);
#pragma unroll
            for (u32 r = 0; r < 8; ++r) { const u32 x = r * 32 + lane; if (x < gl) Bv[gs + x] = e[r].k; }
        }
        __syncthreads();
        for (u32 q = 0; q < nl; ++q) {  // groups over 256 records (heavy key repeats): the CTA
            const u32 g = over ? q : big[q];
            const u32 gs = g ? cnt[g - 1] : 0u, gl = cnt[g] - gs;
            if (gl > 256) cta_sort_u64<SF_NT>(Bv + gs, gl);
        }
        __syncthreads();
        a = Bv;
    } else {
        cta_sort_u64<SF_NT>(a, len);
        __syncthreads();
    }
    SF_PROBE(5)
    for (u32 i = threadIdx.x; i < len; i += SF_NT) ts[bs + i] = a[i];
    // 5. the splitters whose rank falls in this bucket: r = (q+1)s/f - 1 in [bs, bs + len)
    const u64 q0 = ((u64)bs * f + f) / s;  // first q+1 with (q+1)s/f - 1 >= bs, up to rounding
    for (u64 q1 = (q0 > 0 ? q0 - 1 : 0) + threadIdx.x; q1 < P; q1 += SF_NT) {
        const u64 r = q1 * s / f;  // (q+1) = q1 >= 1
        if (q1 == 0 || r == 0) continue;
        if (r - 1 < bs) continue;
        if (r - 1 >= (u64)bs + len) break;
        const u64 v = a[r - 1 - bs];
        sk[q1 - 1] = (U)(v >> 32);
        st[q1 - 1] = (u32)v;
    }
    SF_PROBE(6)
}

// a4: S[q] = T[(q+1)s - 1] (reading Q4); also the p-1 report arrays
template <class U>
// (f > 1: the refined splitters floor((q+1)s/f) - 1 of RosSort, a superset of the contract's)
__global__ void k_pick_splitters(const u64* t_pack, const u64* t_key, const u32* t_tag, u32 P, u32 s, u32 f,
                                 U* sk, u32* st) {
    PDL_PROLOGUE();
    u32 q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q + 1 >= P) return;
    u64 r = (u64)(q + 1) * s / f - 1;
    if (sizeof(U) == 4) {
        u64 v = t_pack[r];
        sk[q] = (U)(v >> 32);
        st[q] = (u32)v;
    } else {
        sk[q] = (U)t_key[r];
        st[q] = t_tag[r];
    }
}

// contract bucket q = refined level-0 buckets qf .. qf+f-1 (RosSort refinement)
__global__ void k_fold_counts(const u64* in, u32 f, u32 p, u64* out) {
    PDL_PROLOGUE();
    const u32 q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= p) return;
    u64 s = 0;
    for (u32 j = 0; j < f; ++j) s += in[(u64)q * f + j];
    out[q] = s;
}

// ------------------------------------------------------------------ classifier LUT build
// lo(e) = #{q : S[q].key < base + e<<shift}, cnt(e) = lo(e+1) - lo(e), frac(e) (see the classifier).
template <class U>
__device__ u32 count_less_key(const U* sk, u32 nsp, U thr) {
    u32 lo = 0, cnt = nsp;
    while (cnt > 0) {
        u32 half = cnt >> 1, mid = lo + half;
        if (sk[mid] < thr) { lo = mid + 1; cnt -= half + 1; } else cnt = half;
    }
    return lo;
}

// Classifier of a single segment covering [0, n) of buffer 0 (the contract level, or an
// internal sort of a whole array): LUT entries in parallel over CTAs, splitter keys staged in
// shared memory; CTA 0 writes the segment header.
template <class U>
// Also the rest of level 0's setup (one launch instead of five): the chunk list, the device
// counts (chunks, segments), the zeroed bucket-list counters and the zeroed histogram rows.
__global__ void __launch_bounds__(1024) k_build_cls0(const U* sk, u32 P, u32 L, u32 log2L, u32* lut, Seg* seg, u32 n,
                                                     u32 nchunk, u32 chunk, Chunk* chunks, u32* ncounts, u32* nfit,
                                                     u32* hist, u32 hist_words) {
    PDL_PROLOGUE();
    {
        const u32 gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
        for (u32 c = gt; c < nchunk; c += gs) {
            Chunk x;
            x.beg = c * chunk;
            x.end = min(n, (c + 1) * chunk);
            x.seg = 0; x.pad = 0;
            chunks[c] = x;
        }
        uint4* h4 = (uint4*)hist;  // hist_words is a multiple of 4 (carved 256-byte aligned)
        for (u32 i = gt; i < hist_words / 4; i += gs) h4[i] = make_uint4(0, 0, 0, 0);
        for (u32 i = (hist_words / 4) * 4 + gt; i < hist_words; i += gs) hist[i] = 0;
        if (gt == 0) { ncounts[0] = nchunk; ncounts[1] = 1; nfit[0] = 0; nfit[1] = 0; }
    }
    extern __shared__ __align__(16) char smem[];
    U* s = (U*)smem;
    for (u32 i = threadIdx.x; i + 1 < P; i += blockDim.x) s[i] = sk[i];
    __syncthreads();
    U base = 0;
    u32 shift = 0;
    if (P > 1) {
        base = s[0];
        U span = s[P - 2] - base;
        u32 bl = bitlen<U>(span);
        shift = bl > log2L ? bl - log2L : 0u;
        U lim = span >> shift;
        for (u32 e = blockIdx.x * blockDim.x + threadIdx.x; e < L; e += gridDim.x * blockDim.x) {
            u32 a = ((U)e > lim) ? (P - 1) : count_less_key<U>(s, P - 1, (U)(base + ((U)e << shift)));
            u32 b = ((U)(e + 1) > lim) ? (P - 1) : count_less_key<U>(s, P - 1, (U)(base + ((U)(e + 1) << shift)));
            // position of the first splitter key inside the entry (16-bit resolution)
            const u32 fr = b > a ? cls_frac<U>((U)(s[a] - base) & (((U)1 << shift) - 1), shift) : 0xffffu;
            lut[e] = a | (min(b - a, 7u) << 13) | (fr << 16);
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) lut[L] = (P - 1) | (0xffffu << 16);  // keys past the table
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        Seg g;
        g.lo = 0;  // loose: the edge buckets' key bounds are found by the bucket sorter
        g.hi = (u64)umax_of<U>();
        g.base = (u64)base;
        g.beg = 0; g.len = n; g.P = P; g.shift = shift; g.L = L; g.chunk0 = 0; g.nchunk = nchunk; g.src = 0;
        g.loose = 1; g.pad = 0;
        *seg = g;
    }
}


// ------------------------------------------------------------------ partition: classifier loader
__host__ __device__ constexpr size_t a16(size_t x) { return (x + 15) & ~(size_t)15; }

template <class U>
__device__ __forceinline__ ClsView<U> load_cls(char* sp, const Seg& sg, u32 segi, const U* sk_pool, const u32* st_pool,
                                               const u32* lut_pool, u32 PS, u32 LS, bool load) {
    U* sk = (U*)sp; sp += a16(sizeof(U) * (size_t)PS);
    u32* st = (u32*)sp; sp += a16(4 * (size_t)PS);
    u32* lut = (u32*)sp;
    if (load) {
        const U* gsk = sk_pool + (size_t)segi * PS;
        const u32* gst = st_pool + (size_t)segi * PS;
        const u32* glut = lut_pool + (size_t)segi * (LS + 1);
        for (u32 i = threadIdx.x; i + 1 < sg.P; i += blockDim.x) { sk[i] = gsk[i]; st[i] = gst[i]; }
        for (u32 i = threadIdx.x; i <= sg.L; i += blockDim.x) lut[i] = glut[i];
    }
    ClsView<U> c;
    c.sk = sk; c.st = st; c.lut = lut; c.base = (U)sg.base; c.shift = sg.shift; c.L = sg.L; c.P = sg.P;
    c.fr = sg.shift >= 16 ? sg.shift - 16 : 0u;
    c.fl = sg.shift >= 16 ? 0u : 16 - sg.shift;
    return c;
}
template <class U> __host__ __device__ constexpr size_t cls_smem_bytes(u32 PS, u32 LS) {
    return a16(sizeof(U) * (size_t)PS) + a16(4 * (size_t)PS) + a16(4 * ((size_t)LS + 1));
}


// ------------------------------------------------------------------ vectorised item loops
// for_items(src, beg, m, f): calls f(key, o) for every o in [0, m) (any order) with 16-byte
// vector loads, UNR vectors in flight per thread (the bucket and partition passes are
// latency bound without this: v1 kept one 4-byte load in flight per thread).
template <class U, int NT, int UNR, class F, bool STREAM = false>
__device__ __forceinline__ void for_items(const U* __restrict__ src, u32 beg, u32 m, F&& f) {
    constexpr u32 V = 16 / sizeof(U);
    const u32 mis = (u32)(((uintptr_t)(src + beg)) & 15u) / (u32)sizeof(U);
    const u32 head = mis ? min(m, V - mis) : 0u;
    if (threadIdx.x < head) f(src[beg + threadIdx.x], threadIdx.x);
    const uint4* a = (const uint4*)(src + beg + head);
    const u32 nv = (m - head) / V;
    u32 v0 = 0;
    for (; v0 + NT * UNR <= nv; v0 += NT * UNR) {  // full batches: no bound tests
        uint4 r[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) r[u] = STREAM ? __ldcs(a + v0 + u * NT + threadIdx.x) : a[v0 + u * NT + threadIdx.x];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const u32 idx = v0 + u * NT + threadIdx.x;
            const U* e = (const U*)&r[u];
#pragma unroll
            for (u32 q = 0; q < V; ++q) f(e[q], head + idx * V + q);
        }
    }
    if (v0 < nv) {
        uint4 r[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const u32 idx = v0 + u * NT + threadIdx.x;
            if (idx < nv) r[u] = STREAM ? __ldcs(a + idx) : a[idx];
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const u32 idx = v0 + u * NT + threadIdx.x;
            if (idx < nv) {
                const U* e = (const U*)&r[u];
#pragma unroll
                for (u32 q = 0; q < V; ++q) f(e[q], head + idx * V + q);
            }
        }
    }
    for (u32 o = head + nv * V + threadIdx.x; o < m; o += NT) f(src[beg + o], o);
}

// ------------------------------------------------------------------ a5+a6: classify + histogram
// Persistent CTAs over chunks; per-chunk histogram row hist[c*PS + b].  LEVEL0 reads buffer 0
// through the codec (the caller's raw keys) with tag = index (ROS: the original index,
// P:524-532); later levels read ordered keys with tag = position (keys only) or the carried
// original index (key-value).
#ifndef OVS_HIST_UNR
#define OVS_HIST_UNR 2
#endif
#ifndef OVS_HIST_MINB
#define OVS_HIST_MINB 1
#endif
template <int DT, bool KV, bool LEVEL0, int NT>
__global__ void __launch_bounds__(NT, OVS_HIST_MINB) k_hist(Bufs<typename Codec<DT>::U> B, const Chunk* chunks, const u32* nchunks,
                                             Seg* segs, const typename Codec<DT>::U* sk_pool, const u32* st_pool,
                                             const u32* lut_pool, u32 PS, u32 LS, u32* hist, u32 split,
                                             u32 tag_base, u16* bid) {
    PDL_PROLOGUE();
    // `split` CTAs share a chunk (each a contiguous part) and add into its (zeroed) row;
    // bid != NULL: every key's bucket is also stored (bid[i]: the scatter then skips classify)
    typedef typename Codec<DT>::U U;
    extern __shared__ __align__(16) char smem[];
    const u32 nc = *nchunks;
    u32 loaded = 0xffffffffu;
    for (u32 w = blockIdx.x; w < nc * split; w += gridDim.x) {
        const u32 c = w / split, part = w % split;
        const Chunk ch = chunks[c];
        const Seg sg = segs[ch.seg];
        ClsView<U> cls = load_cls<U>(smem, sg, ch.seg, sk_pool, st_pool, lut_pool, PS, LS, loaded != ch.seg);
        loaded = ch.seg;
        u32* h = (u32*)(smem + cls_smem_bytes<U>(PS, LS));
        for (u32 i = threadIdx.x; i < sg.P; i += NT) h[i] = 0;
        __syncthreads();
        const u32 len = ch.end - ch.beg;
        const u32 pbeg = ch.beg + (u32)(((u64)len * part / split) & ~15ull);
        const u32 pend = (part + 1 == split) ? ch.end : ch.beg + (u32)(((u64)len * (part + 1) / split) & ~15ull);
        const U* src = B.k[LEVEL0 ? 0 : sg.src];
        const u32* isrc = (KV && !LEVEL0) ? B.i[sg.src] : nullptr;
        auto tag_at = [&](u32 o) -> u32 { return (KV && !LEVEL0) ? isrc[pbeg + o] : (LEVEL0 ? tag_base : 0u) + pbeg + o; };
        auto body = [&](U kr, u32 o) {
            const U k = LEVEL0 ? Codec<DT>::ord(kr) : kr;
            const u32 b = classify<U>(cls, k, tag_at(o));
            atomicAdd(&h[b], 1u);
            if (bid) bid[pbeg + o] = (u16)b;
        };
        // misaligned head and the tail one key at a time, the body in batches of UNR vectors
        constexpr u32 V = 16 / sizeof(U);
        constexpr int UNR = OVS_HIST_UNR, NB = UNR * (int)V;
        const u32 m = pend - pbeg;
        const u32 mis = (u32)(((uintptr_t)(src + pbeg)) & 15u) / (u32)sizeof(U);
        const u32 head = mis ? min(m, V - mis) : 0u;
        if (threadIdx.x < head) body(src[pbeg + threadIdx.x], threadIdx.x);
        const uint4* a4 = (const uint4*)(src + pbeg + head);
        const u32 nv = (m - head) / V;
        // software pipelined: the next batch's vectors are loaded before this batch is classified
        uint4 nr[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const u32 idx = u * NT + threadIdx.x;
            nr[u] = idx < nv ? __ldcs(a4 + idx) : make_uint4(0, 0, 0, 0);
        }
        u16* const bo = bid ? bid + pbeg + head : nullptr;
        const bool bo_al = V == 4 && (((uintptr_t)bo) & 7u) == 0;  // the V ids of a vector as one 8-byte store
        for (u32 v0 = 0; v0 < nv; v0 += NT * UNR) {
            // (full batches, all but the last, take the variant without per-vector bound tests)
            auto batch = [&](auto full_t) {
                constexpr bool FULL = decltype(full_t)::value;
                U kk[NB];
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    const uint4 r = nr[u];
                    const U* e = (const U*)&r;
#pragma unroll
                    for (u32 x = 0; x < V; ++x) kk[u * V + x] = LEVEL0 ? Codec<DT>::ord(e[x]) : e[x];
                }
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    const u32 idx = v0 + NT * UNR + u * NT + threadIdx.x;
                    nr[u] = idx < nv ? __ldcs(a4 + idx) : make_uint4(0, 0, 0, 0);
                }
                u32 bb[NB];
                classify_n<U, NB>(cls, kk, [&](int j) -> u32 {
                    return tag_at(head + (v0 + (j / V) * NT + threadIdx.x) * V + (j % V));
                }, bb);
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    const u32 idx = v0 + u * NT + threadIdx.x;
                    if (!FULL && idx >= nv) continue;
#pragma unroll
                    for (u32 x = 0; x < V; ++x) atomicAdd(&h[bb[u * V + x]], 1u);
                    if (bo) {
                        if (bo_al) {
                            uint2 w;
                            w.x = bb[u * V] | (bb[u * V + 1] << 16);
                            w.y = bb[u * V + 2 % V] | (bb[u * V + 3 % V] << 16);
                            *(uint2*)(bo + idx * V) = w;
                        } else {
#pragma unroll
                            for (u32 x = 0; x < V; ++x) bo[idx * V + x] = (u16)bb[u * V + x];
                        }
                    }
                }
            };
            if (v0 + NT * UNR <= nv) batch(std::true_type{});
            else batch(std::false_type{});
        }
        for (u32 o = head + nv * V + threadIdx.x; o < m; o += NT) body(src[pbeg + o], o);
        __syncthreads();
        u32* row = hist + (size_t)c * PS;
        if (split == 1) {
            for (u32 b = threadIdx.x; b < sg.P; b += NT) row[b] = h[b];
        } else {
            for (u32 b = threadIdx.x; b < sg.P; b += NT)
                if (h[b]) atomicAdd(&row[b], h[b]);
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ a6: column scan
// Work item = (segment s, 32 buckets): exclusive prefix over the segment's chunks of
// hist[c][b], in place; totals -> tot[s*(PS+1) + b].  Warp w owns a contiguous slice of
// chunks, lane = bucket.
__global__ void __launch_bounds__(1024) k_colscan(u32* hist, const Seg* segs, const u32* nsegs, u32 PS, u32* tot) {
    PDL_PROLOGUE();
    __shared__ u32 part[32][33];
    const u32 bgroups = (PS + 31) / 32;
    const u32 nitems = *nsegs * bgroups;
    const u32 lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (u32 it = blockIdx.x; it < nitems; it += gridDim.x) {
        const u32 s = it / bgroups, bg = it % bgroups;
        const Seg sg = segs[s];
        if (bg * 32 >= sg.P) continue;  // uniform across the CTA
        const u32 b = bg * 32 + lane;
        const u32 per = (sg.nchunk + 31) / 32;
        const u32 c0 = sg.chunk0 + min(sg.nchunk, w * per), c1 = sg.chunk0 + min(sg.nchunk, (w + 1) * per);
        u32 sum = 0;
        if (b < sg.P)
            for (u32 c = c0; c < c1; ++c) sum += hist[(size_t)c * PS + b];
        part[w][lane] = sum;
        __syncthreads();
        if (w == 0) {
            u32 run = 0;
            for (int k = 0; k < 32; ++k) { u32 v = part[k][lane]; part[k][lane] = run; run += v; }
            if (b < sg.P) tot[(size_t)s * (PS + 1) + b] = run;
        }
        __syncthreads();
        if (b < sg.P) {
            u32 run = part[w][lane];
            for (u32 c = c0; c < c1; ++c) {
                u32 v = hist[(size_t)c * PS + b];
                hist[(size_t)c * PS + b] = run;
                run += v;
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ a6: segment scan + lists
// Per segment: bucket starts = exclusive scan of the totals (in place in tot[]); every
// non-empty bucket becomes a Bucket on `big` (len > cap and big != NULL) or `fit`.
// counts_out (level 0 of the contract) receives the bucket counts.
template <class U>
__global__ void __launch_bounds__(1024) k_segscan(const Seg* segs, const u32* nsegs, u32 PS, u32* tot_pool,
                                                  const U* sk_pool, u32 level, u32 cap, Bucket* fit, u32* nfit,
                                                  u32 fit_cap, Bucket* big, u32* nbig, u32 big_cap, u64* counts_out,
                                                  u32* status) {
    PDL_PROLOGUE();
    __shared__ u32 red[33];
    const u32 ns = *nsegs;
    const u32 lane = threadIdx.x & 31;
    for (u32 s = blockIdx.x; s < ns; s += gridDim.x) {
        const Seg sg = segs[s];
        u32* tot = tot_pool + (size_t)s * (PS + 1);
        if (counts_out)
            for (u32 b = threadIdx.x; b < sg.P; b += 1024) counts_out[b] = tot[b];
        __syncthreads();
        block_scan_array<1024>(tot, sg.P, red);
        const U* sk = sk_pool + (size_t)s * PS;
        for (u32 b0 = 0; b0 < sg.P; b0 += 1024) {
            const u32 b = b0 + threadIdx.x;
            u32 st = 0, len = 0;
            if (b < sg.P) { st = tot[b]; len = tot[b + 1] - st; }
            const bool isbig = big != nullptr && len > cap, isfit = len > 0 && !isbig;
            const u32 mf = __ballot_sync(0xffffffffu, isfit), mb = __ballot_sync(0xffffffffu, isbig);
            u32 of = 0, ob = 0;
            if (lane == 0) {
                if (mf) of = atomicAdd(nfit, __popc(mf));
                if (mb) ob = atomicAdd(nbig, __popc(mb));
            }
            of = __shfl_sync(0xffffffffu, of, 0) + __popc(mf & ((1u << lane) - 1));
            ob = __shfl_sync(0xffffffffu, ob, 0) + __popc(mb & ((1u << lane) - 1));
            if (isfit || isbig) {
                Bucket bk;
                bk.beg = sg.beg + st; bk.len = len; bk.buf = 1 - sg.src;
                bk.level = level | (((b == 0 || b + 1 == sg.P) && sg.loose) ? BK_LOOSE : 0u);
                bk.lo = (b == 0) ? sg.lo : (u64)sk[b - 1];
                bk.hi = (b + 1 == sg.P) ? sg.hi : (u64)sk[b];
                if (isfit) { if (of < fit_cap) fit[of] = bk; else st_set(status, ST_LIST_OVER); }
                else { if (ob < big_cap) big[ob] = bk; else st_set(status, ST_LIST_OVER); }
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ a7: scatter
// Persistent CTAs over chunks, sub-tiles of NT*ITEMS items: classify, rank inside the sub-tile
// with shared atomics, stage the sub-tile in bucket order in shared memory, then write every
// bucket run contiguously at its cursor.  Cursors start at segment base + bucket start +
// the chunk's column-scan offset, so chunks write disjoint, deterministic ranges.
template <class U, bool KV, int ITEMS, int NT>
__host__ __device__ constexpr size_t scatter_smem_bytes(u32 PS, u32 LS) {
    return cls_smem_bytes<U>(PS, LS) + (sizeof(U) + (KV ? 8 : 0) + 2) * (size_t)NT * ITEMS +
           3 * a16(4 * ((size_t)PS + 1));
}

// DIST (multi-GPU f1, key-value sorts): bucket b's items go to its owner's window (keys at
// po.off, values at off_v, original indices at off_i) at dst_off[b] + the chunk's offset.
template <int DT, bool KV, bool LEVEL0, int NT, int ITEMS, bool DIST = false>
__global__ void __launch_bounds__(NT) k_scatter(Bufs<typename Codec<DT>::U> B, const Chunk* chunks, const u32* nchunks,
                                                const Seg* segs, const typename Codec<DT>::U* sk_pool,
                                                const u32* st_pool, const u32* lut_pool, u32 PS, u32 LS,
                                                const u32* hist, const u32* tot_pool, u32 tag_base,
                                                const u32* dst_off = nullptr, PeerOut po = PeerOut{nullptr, 0, 1},
                                                size_t off_v = 0, size_t off_i = 0) {
    PDL_PROLOGUE();
    typedef typename Codec<DT>::U U;
    constexpr int TS = NT * ITEMS;
    extern __shared__ __align__(16) char smem[];
    __shared__ u32 red[NT / 32 + 1];
    const u32 nc = *nchunks;
    u32 loaded = 0xffffffffu;
    char* sp0 = smem + cls_smem_bytes<U>(PS, LS);
    U* stk = (U*)sp0; sp0 += sizeof(U) * TS;
    u32* stv = nullptr;
    u32* sti = nullptr;
    if (KV) { stv = (u32*)sp0; sp0 += 4 * TS; sti = (u32*)sp0; sp0 += 4 * TS; }
    u32* cur = (u32*)sp0; sp0 += a16(4 * ((size_t)PS + 1));
    u32* work = (u32*)sp0; sp0 += a16(4 * ((size_t)PS + 1));
    u32* dbase = (u32*)sp0; sp0 += a16(4 * ((size_t)PS + 1));
    unsigned short* stb = (unsigned short*)sp0;
    for (u32 c = blockIdx.x; c < nc; c += gridDim.x) {
        const Chunk ch = chunks[c];
        const Seg sg = segs[ch.seg];
        ClsView<U> cls = load_cls<U>(smem, sg, ch.seg, sk_pool, st_pool, lut_pool, PS, LS, loaded != ch.seg);
        loaded = ch.seg;
        const u32 P = sg.P;
        const u32* hrow = hist + (size_t)c * PS;
        const u32* bst = tot_pool + (size_t)ch.seg * (PS + 1);
        for (u32 b = threadIdx.x; b < P; b += NT) cur[b] = DIST ? dst_off[b] + hrow[b] : sg.beg + bst[b] + hrow[b];
        const u32 srcb = LEVEL0 ? 0 : sg.src, dstb = 1 - srcb;
        const U* src = B.k[srcb];
        const u32* vsrc = KV ? B.v[srcb] : nullptr;
        const u32* isrc = (KV && !LEVEL0) ? B.i[srcb] : nullptr;
        U* dst = B.k[dstb];
        u32* vdst = KV ? B.v[dstb] : nullptr;
        u32* idst = KV ? B.i[dstb] : nullptr;
        for (u32 t0 = ch.beg; t0 < ch.end; t0 += TS) {
            const u32 nt = min((u32)TS, ch.end - t0);
            for (u32 b = threadIdx.x; b < P; b += NT) work[b] = 0;
            __syncthreads();
            U k[ITEMS];
            u32 v[ITEMS], ix[ITEMS], bk[ITEMS], rk[ITEMS];
            // item slot j of this thread is sub-tile offset off(j): 16-byte vectors when the
            // sub-tile is full and aligned, otherwise a strided scalar loop
            constexpr u32 V = 16 / sizeof(U);
            const bool vec = nt == (u32)TS && ((((uintptr_t)(src + t0)) & 15u) == 0) &&
                             (!KV || ((((uintptr_t)(vsrc + t0)) & 15u) == 0));
            auto off = [&](int j) -> u32 {
                return vec ? ((j / V) * NT + threadIdx.x) * V + (j % V) : j * NT + threadIdx.x;
            };
            if (vec) {
#pragma unroll
                for (int jv = 0; jv < ITEMS / (int)V; ++jv) {
                    const u32 vi = jv * NT + threadIdx.x;
                    uint4 r = __ldcs((const uint4*)(src + t0) + vi);
                    const U* e = (const U*)&r;
#pragma unroll
                    for (u32 q = 0; q < V; ++q) k[jv * V + q] = LEVEL0 ? Codec<DT>::ord(e[q]) : e[q];
                    if (KV) {
#pragma unroll
                        for (u32 q = 0; q < V; ++q) {
                            const u32 i = t0 + vi * V + q;
                            v[jv * V + q] = vsrc[i];
                            ix[jv * V + q] = LEVEL0 ? tag_base + i : isrc[i];
                        }
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < ITEMS; ++j) {
                    const u32 o = off(j);
                    if (o < nt) {
                        const u32 i = t0 + o;
                        k[j] = LEVEL0 ? Codec<DT>::ord(src[i]) : src[i];
                        if (KV) { v[j] = vsrc[i]; ix[j] = LEVEL0 ? tag_base + i : isrc[i]; }
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < ITEMS; ++j) {
                const u32 o = off(j);
                if (o < nt) {
                    const u32 tag = KV ? ix[j] : (LEVEL0 ? tag_base : 0u) + t0 + o;
                    bk[j] = classify<U>(cls, k[j], tag);
                    rk[j] = atomicAdd(&work[bk[j]], 1u);
                }
            }
            __syncthreads();
            block_scan_array<NT>(work, P, red);
#pragma unroll
            for (int j = 0; j < ITEMS; ++j) {
                const u32 o = off(j);
                if (o < nt) {
                    const u32 pos = work[bk[j]] + rk[j];
                    stk[pos] = k[j];
                    stb[pos] = (unsigned short)bk[j];
                    if (KV) { stv[pos] = v[j]; sti[pos] = ix[j]; }
                }
            }
            for (u32 b = threadIdx.x; b < P; b += NT) {
                const u32 st = work[b], cnt = work[b + 1] - st;
                dbase[b] = cur[b] - st;
                cur[b] += cnt;
            }
            __syncthreads();
            for (u32 o = threadIdx.x; o < nt; o += NT) {
                const u32 bb = stb[o];
                const u32 d = dbase[bb] + o;
                if constexpr (DIST) {
                    char* const w = po.peers[(bb * po.world) / P];
                    ((U*)(w + po.off))[d] = stk[o];
                    if (KV) { ((u32*)(w + off_v))[d] = stv[o]; ((u32*)(w + off_i))[d] = sti[o]; }
                } else {
                    dst[d] = stk[o];
                    if (KV) { vdst[d] = stv[o]; idst[d] = sti[o]; }
                }
            }
            __syncthreads();
        }
    }
    if (DIST) __threadfence_system();
}

// ------------------------------------------------------------------ a7: write-combining scatter
// Keys-only level-0 scatter, driven by the bucket ids the histogram pass stored (bid[i]).  Per
// chunk and bucket b the chunk's keys of b go to the global positions [r_b, r_b + n_b) (r_b
// from the histogram scans, so chunks write disjoint, deterministic ranges).  q[b] = the next
// position to hand out (a shared atomic gives every key its absolute output position); sb[b] =
// the 32-byte global sector whose keys are gathered in b's shared sector wc[b] (low 3 bits: the
// first valid slot, non-zero only for the chunk's first sector of b, whose front belongs to the
// previous chunk).  (Packing q and sb into one 64-bit word for a single atomic measured 1.7x
// slower: 64-bit shared atomics are not native-speed.)  A sector goes to global memory only when complete, as one 32-byte store, so
// DRAM never sees a partially written sector (measured on B200: partial-sector stores cost a
// DRAM read-modify-write even when the rest of the sector follows microseconds later) except the
// (at most two) boundary sectors of every (chunk, bucket) run.
// Per sub-tile (keys in registers; the next sub-tile's loads are in flight meanwhile):
//   P1: pos = atomicAdd(q[b], 1); pos inside the current sector -> wc[b][pos - sector]
//   P2: the key at the sector's last slot flushes wc[b] and moves sb[b] to the sector of the
//       final q[b]; keys of complete sectors beyond it -> global directly (whole sectors)
//   P3: keys of the new, incomplete sector -> wc[b]
// Ranks come from shared atomics: positions inside a (chunk, bucket) run are not in input
// order, which the bucket sorter makes irrelevant (module notes).
#ifndef OVS_WC_SB  // bytes of a write-combining sector (the DRAM sector is 32)
#define OVS_WC_SB 32
#endif
#ifndef OVS_WC_MINB  // resident CTAs per SM of the write-combining scatter
#define OVS_WC_MINB 1
#endif
template <class U> __host__ __device__ constexpr size_t wc_smem_bytes(u32 PS) {
    return OVS_WC_SB * (size_t)PS + 8 * (size_t)PS;  // wc, q, sb
}

// LEVEL0: the caller's raw keys in buffer 0 -> buffer 1; otherwise ordered keys of every chunk's
// segment source buffer -> the other buffer (level 1)
// DIST (multi-GPU): bucket b's keys go straight to its owner rank
// floor(b*world/P)'s receive window over NVLink (po.peers[owner] + po.off), at dst_off[b] (this
// rank's run of b inside the owner's region, ovs_dist.cu) + the chunk's offset in the run.
template <int DT, int NT, int ITEMS, bool LEVEL0, bool DIST = false>
__global__ void __launch_bounds__(NT, OVS_WC_MINB) k_scatter_wc(Bufs<typename Codec<DT>::U> B, const Chunk* chunks,
                                                       const u32* nchunks, const Seg* segs, u32 PS, const u32* hist,
                                                       const u32* tot_pool, const u16* bid, const u32* dst_off = nullptr,
                                                       PeerOut po = PeerOut{nullptr, 0, 1}) {
    PDL_PROLOGUE();
    typedef typename Codec<DT>::U U;
    constexpr u32 SV = OVS_WC_SB / sizeof(U);  // keys per write-combining sector
    constexpr u32 V = 16 / sizeof(U);   // keys per 16-byte vector
    constexpr u32 TS = NT * ITEMS;
    constexpr u32 NI = (ITEMS + 1) / 2;  // two u16 bucket ids per word
    static_assert(ITEMS % V == 0 && ITEMS <= 32, "whole vectors per thread, one mask bit per item");
    extern __shared__ __align__(16) char smem[];
    U* wc = (U*)smem;
    u32* q = (u32*)(smem + OVS_WC_SB * (size_t)PS);
    u32* sb = q + PS;
    const u32 nc = *nchunks;
    for (u32 c = blockIdx.x; c < nc; c += gridDim.x) {
        const Chunk ch = chunks[c];
        const Seg sg = segs[ch.seg];
        const u32 P = sg.P;
        const U* src = B.k[LEVEL0 ? 0 : sg.src];
        // positions are counted from an aligned base (the output array may be the caller's, not
        // 32-byte aligned): position x is dst[x] with dst = the array - al
        U* const dst0 = DIST ? nullptr : B.k[LEVEL0 ? 1 : 1 - sg.src];
        const u32 al = DIST ? 0u : (u32)(((uintptr_t)dst0 / sizeof(U)) & (SV - 1));
        U* dst = dst0 - al;
        // destination array of bucket b (DIST: the owner's window, 256-byte aligned)
        auto dst_of = [&](u32 b) -> U* {
            if constexpr (DIST) return (U*)(po.peers[(b * po.world) / P] + po.off);
            else return dst;
        };
        const u32* hrow = hist + (size_t)c * PS;
        const u32* bst = tot_pool + (size_t)ch.seg * (PS + 1);
        for (u32 b = threadIdx.x; b < P; b += NT) {
            const u32 r = DIST ? dst_off[b] + hrow[b] : sg.beg + bst[b] + hrow[b] + al;
            q[b] = r;
            sb[b] = r;  // sector r & ~(SV-1), first valid slot r & (SV-1)
        }
        __syncthreads();
        const bool vec_ok = ((((uintptr_t)(src + ch.beg)) & 15u) == 0) && ((((uintptr_t)(bid + ch.beg)) & 7u) == 0);
        U nk[ITEMS];
        u32 nid[NI];
        auto load = [&](u32 t0, U (&k)[ITEMS], u32 (&id)[NI]) {
            const u32 nt = min(TS, ch.end - t0);
            if (vec_ok && nt == TS) {
#pragma unroll
                for (u32 jv = 0; jv < ITEMS / V; ++jv) {
                    const uint4 r = __ldcs((const uint4*)(src + t0) + jv * NT + threadIdx.x);
                    const U* e = (const U*)&r;
#pragma unroll
                    for (u32 x = 0; x < V; ++x) k[jv * V + x] = e[x];
                    if (V == 4) {
                        const uint2 w = __ldcs((const uint2*)(bid + t0) + jv * NT + threadIdx.x);
                        id[jv * 2] = w.x;
                        id[(jv * 2 + 1) % NI] = w.y;
                    } else {
                        id[jv] = __ldcs((const unsigned int*)(bid + t0) + jv * NT + threadIdx.x);
                    }
                }
            } else {
#pragma unroll
                for (u32 j = 0; j < ITEMS; ++j) {
                    const u32 o = ((j / V) * NT + threadIdx.x) * V + (j % V);
                    k[j] = o < nt ? src[t0 + o] : (U)0;
                    const u32 v = o < nt ? (u32)bid[t0 + o] : 0u;
                    if (j & 1) id[j / 2] |= v << 16; else id[j / 2] = v;
                }
            }
        };
        if (ch.beg < ch.end) load(ch.beg, nk, nid);
        for (u32 t0 = ch.beg; t0 < ch.end; t0 += TS) {
            const u32 nt = min(TS, ch.end - t0);
            U k[ITEMS];
            u32 id[NI];
#pragma unroll
            for (u32 j = 0; j < ITEMS; ++j) k[j] = nk[j];
#pragma unroll
            for (u32 j = 0; j < NI; ++j) id[j] = nid[j];
            if (t0 + TS < ch.end) load(t0 + TS, nk, nid);  // in flight while this sub-tile is processed
            u32 vmask = 0xffffffffu;
            if (nt < TS) {
                vmask = 0;
#pragma unroll
                for (u32 j = 0; j < ITEMS; ++j)
                    if (((j / V) * NT + threadIdx.x) * V + (j % V) < nt) vmask |= 1u << j;
            }
#if OVS_WC_BFLUSH
            // P1: a position per key; keys inside their bucket's current sector are parked in it,
            // the others (rare: a bucket whose sector fills up within this sub-tile) are marked
            u32 pos[ITEMS], sv[ITEMS], out = 0;
            // (full sub-tiles, all but a chunk's last, take the variant without per-item validity tests)
            auto p1 = [&](auto full_t) {
                constexpr bool FULL = decltype(full_t)::value;
#pragma unroll
                for (u32 j = 0; j < ITEMS; ++j) {
                    const u32 b = (id[j / 2] >> (16 * (j & 1))) & 0xffffu;
                    if (LEVEL0) k[j] = Codec<DT>::ord(k[j]);
                    if (FULL || (vmask & (1u << j))) pos[j] = atomicAdd(&q[b], 1u);
                }
#pragma unroll
                for (u32 j = 0; j < ITEMS; ++j) sv[j] = sb[(id[j / 2] >> (16 * (j & 1))) & 0xffffu];
#pragma unroll
                for (u32 j = 0; j < ITEMS; ++j) {
                    const u32 b = (id[j / 2] >> (16 * (j & 1))) & 0xffffu;
                    const u32 d = pos[j] - (sv[j] & ~(SV - 1));
                    if (FULL || (vmask & (1u << j))) {
                        if (d < SV) wc[(size_t)b * SV + d] = k[j];
                        else out |= 1u << j;
                    }
                }
            };
            if (nt == TS) p1(std::true_type{});
            else p1(std::false_type{});
            __syncthreads();
            // P2: every bucket whose current sector is complete is flushed by the thread that owns
            // the bucket (one check per bucket instead of per key); keys of complete sectors past it
            // go straight out, keys of the new incomplete sector wait for P3
            for (u32 b = threadIdx.x; b < P; b += NT) {
                const u32 qe = q[b], sv0 = sb[b], s0 = sv0 & ~(SV - 1);
                if (qe >= s0 + SV) {
                    const u32 front = sv0 & (SV - 1);
                    const U* wb = wc + (size_t)b * SV;
                    U* const db = dst_of(b);
                    if (front == 0) {
                        const uint4* w4 = (const uint4*)wb;
                        uint4* g4 = (uint4*)(db + s0);
#pragma unroll
                        for (u32 x = 0; x < OVS_WC_SB / 16; ++x) g4[x] = w4[x];
                    } else {
                        for (u32 x = front; x < SV; ++x) db[s0 + x] = wb[x];
                    }
                    sb[b] = qe & ~(SV - 1);
                }
            }
            u32 tail = 0;
            if (__any_sync(0xffffffffu, out != 0)) {
#pragma unroll
                for (u32 j = 0; j < ITEMS; ++j) {
                    if (out & (1u << j)) {
                        const u32 b = (id[j / 2] >> (16 * (j & 1))) & 0xffffu;
                        const u32 qf = q[b];
                        if (pos[j] < (qf & ~(SV - 1))) dst_of(b)[pos[j]] = k[j];
                        else tail |= 1u << j;
                    }
                }
            }
            __syncthreads();
            // P3: keys of the new incomplete sector
            if (__any_sync(0xffffffffu, tail != 0)) {
#pragma unroll
                for (u32 j = 0; j < ITEMS; ++j) {
                    if (tail & (1u << j)) {
                        const u32 b = (id[j / 2] >> (16 * (j & 1))) & 0xffffu;
                        wc[(size_t)b * SV + (pos[j] & (SV - 1))] = k[j];
                    }
                }
            }
        }
#else
            // P1: a position and the current sector per key; park it there if it is inside
            // (separate passes over the ITEMS keys: all atomics, then all sector loads, then the
            // stores, so ITEMS independent shared accesses are in flight instead of one chain)
            u32 pos[ITEMS], sv[ITEMS], inmask = 0, lead = 0;
#pragma unroll
            for (u32 j = 0; j < ITEMS; ++j) {
                const u32 b = (id[j / 2] >> (16 * (j & 1))) & 0xffffu;
                if (LEVEL0) k[j] = Codec<DT>::ord(k[j]);
                if (vmask & (1u << j)) pos[j] = atomicAdd(&q[b], 1u);
            }
#pragma unroll
            for (u32 j = 0; j < ITEMS; ++j) sv[j] = sb[(id[j / 2] >> (16 * (j & 1))) & 0xffffu];
#pragma unroll
            for (u32 j = 0; j < ITEMS; ++j) {
                const u32 b = (id[j / 2] >> (16 * (j & 1))) & 0xffffu;
                const u32 d = pos[j] - (sv[j] & ~(SV - 1));
                if ((vmask & (1u << j)) && d < SV) {
                    wc[(size_t)b * SV + d] = k[j];
                    inmask |= 1u << j;
                    if (d == SV - 1) lead |= 1u << j;
                }
            }
            __syncthreads();
            // P2: flush completed sectors; keys of complete sectors past them go straight out
            u32 tail = 0, qf[ITEMS];
#pragma unroll
            for (u32 j = 0; j < ITEMS; ++j)
                if (((vmask & ~inmask) | lead) & (1u << j)) qf[j] = q[(id[j / 2] >> (16 * (j & 1))) & 0xffffu];
#pragma unroll
            for (u32 j = 0; j < ITEMS; ++j) {
                const u32 b = (id[j / 2] >> (16 * (j & 1))) & 0xffffu;
                if (lead & (1u << j)) {
                    const u32 sv = sb[b], s0 = sv & ~(SV - 1), front = sv & (SV - 1);
                    const U* wb = wc + (size_t)b * SV;
                    U* const db = dst_of(b);
                    if (front == 0) {
                        const uint4* w4 = (const uint4*)wb;
                        uint4* g4 = (uint4*)(db + s0);
#pragma unroll
                        for (u32 x = 0; x < OVS_WC_SB / 16; ++x) g4[x] = w4[x];
                    } else {
                        for (u32 x = front; x < SV; ++x) db[s0 + x] = wb[x];
                    }
                    sb[b] = qf[j] & ~(SV - 1);
                } else if ((vmask & ~inmask) & (1u << j)) {
                    if (pos[j] < (qf[j] & ~(SV - 1))) dst_of(b)[pos[j]] = k[j];
                    else tail |= 1u << j;
                }
            }
            __syncthreads();
            // P3: keys of the new incomplete sector
#pragma unroll
            for (u32 j = 0; j < ITEMS; ++j) {
                if (tail & (1u << j)) {
                    const u32 b = (id[j / 2] >> (16 * (j & 1))) & 0xffffu;
                    wc[(size_t)b * SV + (pos[j] & (SV - 1))] = k[j];
                }
            }
        }
#endif
        __syncthreads();
        // the chunk's last, incomplete sectors (and runs inside one sector)
        for (u32 b = threadIdx.x; b < P; b += NT) {
            const u32 qe = q[b], sv = sb[b], s0 = sv & ~(SV - 1), front = sv & (SV - 1);
            U* const db = dst_of(b);
            for (u32 x = front; s0 + x < qe; ++x) db[s0 + x] = wc[(size_t)b * SV + x];
        }
        __syncthreads();
    }
    // the peers read these stores after the next barrier (ovs_dist.cu): make them visible system-wide
    if (DIST) __threadfence_system();
}

// ------------------------------------------------------------------ level 1: buckets far over capacity
// A list of buckets much larger than one SM's shared memory is re-split by the whole GPU ("the
// split keys are to be sorted ... recursively by this same extended method"): every
// bucket becomes a segment with its own sub-splitters (a sorted random sample of it, 8 records per
// sub-splitter, tie-broken by position / original index), classifier table and chunks; then the
// segment-aware histogram, column scan, segment scan and staged scatter kernels partition all of
// them at once (all SMs instead of one CTA per bucket), and the sub-buckets join a bucket list.
// Sub-splitter choice only affects sub-bucket sizes: the sorted result is unique either way.
constexpr u32 L1_SI = 8;

template <int DT, bool KV>
__global__ void __launch_bounds__(1024) k_l1_setup(Bufs<typename Codec<DT>::U> B, const Bucket* list, const u32* nlist,
                                                   u32 part, u32 PS, u32 LS, u32 log2LS, typename Codec<DT>::U* sk_pool,
                                                   u32* st_pool, u32* lut_pool, Seg* segs, u32* nsegs, u64 seed,
                                                   u32 chunk) {
    PDL_PROLOGUE();
    typedef typename Codec<DT>::U U;
    extern __shared__ __align__(16) char smem[];
    const u32 nl = *nlist;
    const u32 g = blockIdx.x;
    if (g == 0 && threadIdx.x == 0) *nsegs = nl;
    if (g >= nl) return;
    const Bucket bk = list[g];
    const u32 len = bk.len;
    const U* src = B.k[bk.buf];
    const u32* isrc = KV ? B.i[bk.buf] : nullptr;
    u32 P = (len + part - 1) / part;
    P = max(2u, min(PS, P));
    const u32 ns = P * L1_SI - 1;
    u32 N = 32;
    while (N < ns) N <<= 1;
    U* tk = (U*)smem;
    u32* tt = (u32*)(smem + sizeof(U) * (size_t)PS * L1_SI);
    for (u32 j = threadIdx.x; j < N; j += blockDim.x) {
        if (j < ns) {
            const u32 o = bk.beg + (u32)__umul64hi(rng_H(seed ^ ((u64)bk.beg * 0x9e3779b97f4a7c15ull), 80, j), (u64)len);
            tk[j] = src[o];
            tt[j] = KV ? isrc[o] : o;
        } else {
            tk[j] = umax_of<U>();
            tt[j] = 0xffffffffu;
        }
    }
    __syncthreads();
    cta_bitonic_kt<U>(tk, tt, N);
    // sub-splitters (rank (i+1) L1_SI - 1 of the sample) to the pool and to the front of tk
    U ck = 0;
    u32 ct = 0;
    const bool mine = threadIdx.x + 1 < P;
    if (mine) { ck = tk[(threadIdx.x + 1) * L1_SI - 1]; ct = tt[(threadIdx.x + 1) * L1_SI - 1]; }
    __syncthreads();
    if (mine) {
        tk[threadIdx.x] = ck;
        sk_pool[(size_t)g * PS + threadIdx.x] = ck;
        st_pool[(size_t)g * PS + threadIdx.x] = ct;
    }
    __syncthreads();
    // classifier table of the segment (same format as k_build_cls0)
    u32 L = 64;
    while (L < 4 * P && L < LS) L <<= 1;
    u32 log2L = 6;
    while ((1u << log2L) < L) ++log2L;
    const U base = tk[0];
    const U span = tk[P - 2] - base;
    const u32 bl = bitlen<U>(span);
    const u32 shift = bl > log2L ? bl - log2L : 0u;
    const U lim = span >> shift;
    u32* lut = lut_pool + (size_t)g * (LS + 1);
    for (u32 e = threadIdx.x; e < L; e += blockDim.x) {
        const u32 a = ((U)e > lim) ? (P - 1) : count_less_key<U>(tk, P - 1, (U)(base + ((U)e << shift)));
        const u32 b = ((U)(e + 1) > lim) ? (P - 1) : count_less_key<U>(tk, P - 1, (U)(base + ((U)(e + 1) << shift)));
        const u32 fr = b > a ? cls_frac<U>((U)(tk[a] - base) & (((U)1 << shift) - 1), shift) : 0xffffu;
        lut[e] = a | (min(b - a, 7u) << 13) | (fr << 16);
    }
    if (threadIdx.x == 0) {
        lut[L] = (P - 1) | (0xffffu << 16);
        Seg sg;
        sg.lo = bk.lo; sg.hi = bk.hi; sg.base = (u64)base;
        sg.beg = bk.beg; sg.len = len; sg.P = P; sg.shift = shift; sg.L = L;
        sg.chunk0 = 0; sg.nchunk = (len + chunk - 1) / chunk; sg.src = bk.buf;
        sg.loose = (bk.level & BK_LOOSE) ? 1u : 0u; sg.pad = (bk.level & 0xffffu) + 1;
        segs[g] = sg;
    }
}

// chunk list of all segments (one CTA): chunk0 = exclusive scan of the segments' chunk counts
__global__ void __launch_bounds__(1024) k_l1_chunks(Seg* segs, const u32* nsegs, u32 chunk, Chunk* chunks, u32* nchunks) {
    PDL_PROLOGUE();
    __shared__ u32 red[33];
    const u32 ns = *nsegs;
    u32 carry = 0;
    for (u32 s0 = 0; s0 < ns; s0 += 1024) {
        const u32 s = s0 + threadIdx.x;
        const u32 c = s < ns ? segs[s].nchunk : 0u;
        u32 tot;
        const u32 ex = block_exclusive_scan<1024>(c, red, &tot) + carry;
        if (s < ns) {
            segs[s].chunk0 = ex;
            const Seg sg = segs[s];
            for (u32 q = 0; q < c; ++q) {
                Chunk ch;
                ch.beg = sg.beg + q * chunk;
                ch.end = min(sg.beg + sg.len, sg.beg + (q + 1) * chunk);
                ch.seg = s; ch.pad = 0;
                chunks[ex + q] = ch;
            }
        }
        carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) *nchunks = carry;
}

// raw keys of buffer 0 -> ordered keys in buffer 1 (+ values and original indices): the DRO
// sequences become ordinary (non-raw) buckets for level 1
template <int DT, bool KV>
__global__ void k_to_ordered(Bufs<typename Codec<DT>::U> B, u32 n) {
    PDL_PROLOGUE();
    for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        B.k[1][i] = Codec<DT>::ord(B.k[0][i]);
        if (KV) { B.v[1][i] = B.v[0][i]; B.i[1][i] = i; }
    }
}

// every bucket of a list moved to buffer 1 - buf (the DRO sequences after k_to_ordered)
__global__ void k_list_flip(Bucket* list, const u32* nlist) {
    PDL_PROLOGUE();
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= *nlist) return;
    Bucket b = list[i];
    b.buf = 1 - b.buf;
    b.level &= ~BK_RAW;
    list[i] = b;
}

// ------------------------------------------------------------------ internal splitters
// Splitters of an internal sort of a whole array of n items (not part of the contract; used
// for p == 1 and for sorting the sample / candidate arrays): a random sample with
// replacement of P*si-1 (key, index) records, sorted in one CTA, S[q] = T[(q+1)si - 1].
template <int DT, bool KV>
__global__ void __launch_bounds__(1024) k_internal_sample(Bufs<typename Codec<DT>::U> B, u32 n, u32 P, u32 si, u32 N,
                                                          u64 seed, typename Codec<DT>::U* sk, u32* st) {
    PDL_PROLOGUE();
    typedef typename Codec<DT>::U U;
    extern __shared__ __align__(16) char smem[];
    U* tk = (U*)smem;
    u32* tt = (u32*)(smem + sizeof(U) * N);
    const u32 m = P * si - 1;
    for (u32 j = threadIdx.x; j < N; j += blockDim.x) {
        if (j < m) {
            const u32 pos = (u32)__umul64hi(rng_H(seed, 63, j), (u64)n);
            tk[j] = Codec<DT>::ord(B.k[0][pos]);
            tt[j] = pos;
        } else {
            tk[j] = umax_of<U>();
            tt[j] = 0xffffffffu;
        }
    }
    __syncthreads();
    cta_bitonic_kt<U>(tk, tt, N);
    for (u32 q = threadIdx.x; q + 1 < P; q += blockDim.x) {
        sk[q] = tk[(q + 1) * si - 1];
        st[q] = tt[(q + 1) * si - 1];
    }
}

// ------------------------------------------------------------------ a8: bucket sort
// Persistent CTAs pull buckets from the list.  A bucket of len <= cap is sorted on chip:
//  1. histogram of the top lg bits of (key - lo) [key-value: of the composite (key, index)]
//     over ng ~ len/3 fine groups (the bounds come from the splitters around the bucket),
//  2. scatter from global (L2-resident after pass 1) into shared memory grouped by digit,
//  3. every group (mostly <= 8 items) sorted by one thread with Batcher's 19-comparator
//     network; larger groups by a warp (bitonic, <= 512) or the CTA (bitonic in place),
//  4. the sorted bucket copied to the output at its final position (raw codec).
// All global reads of a bucket finish before any write, so the source may alias the output.
// A bucket over the capacity is re-split by the CTA itself ("sorted ... recursively by this
// same extended method"): a random sample of it gives <= 64 sub-splitters, the
// bucket is partitioned into the other buffer and the sub-buckets go on a per-CTA stack.
#ifndef OVS_BS_NT
#define OVS_BS_NT 512
#endif
constexpr int BS_NT = OVS_BS_NT;
#ifndef OVS_BS_PF2  // prefetch two buckets ahead into L2
#define OVS_BS_PF2 0
#endif
#ifndef OVS_BS_STCS  // streaming (evict-first) stores of the sorted output
#define OVS_BS_STCS 0
#endif
#ifndef OVS_BS_WIN16  // 32-bit keys only: swizzled items + 16-key window networks (0: round-1 path)
#define OVS_BS_WIN16 1
#endif
constexpr u32 BS_WARPMAX = BS_NT >= 1024 ? 256 : 512;  // largest group a warp sorts in registers
#ifdef OVS_BS_PROF  // phase profile of the bucket sorter (experiments only): CTA-0-thread cycles per phase
__device__ unsigned long long g_bsprof[16];
#define BS_T0 long long bs_t_ = clock64();
#define BS_PROBE(i) if (threadIdx.x == 0) { const long long n_ = clock64(); atomicAdd(&g_bsprof[i], (unsigned long long)(n_ - bs_t_)); bs_t_ = n_; }
#else
#define BS_T0
#define BS_PROBE(i)
#endif
constexpr int BS_NGMAX = 8192;
constexpr u32 BS_WMAX = 4;  // buckets up to BS_WMAX * cap are sorted on chip in windows
#ifndef OVS_BS_UNR
#define OVS_BS_UNR 4
#endif
#ifndef OVS_NET8_X
#define OVS_NET8_X 2
#endif
constexpr int BS_BIGMAX = 768;
constexpr int BS_HUGEMAX = 256;  // groups > BS_WARPMAX items: at most cap/BS_WARPMAX exist
constexpr int BS_STACK = 256;
constexpr u32 BS_SPMAX = 64;
constexpr u32 BS_SI = 32;
constexpr u32 BS_SSMAX = BS_SPMAX * BS_SI;

template <class U, bool KV> struct BucketSmem {
    U* k; u32* i; u32* v; u32* cnt;
};

template <class U, bool KV>
__device__ __forceinline__ Elem<U, KV> sm_get(const BucketSmem<U, KV>& S, u32 x) {
    Elem<U, KV> e;
    e.k = S.k[x];
    if constexpr (KV) { e.i = S.i[x]; e.v = S.v[x]; }
    return e;
}
template <class U, bool KV>
__device__ __forceinline__ void sm_put(const BucketSmem<U, KV>& S, u32 x, const Elem<U, KV>& e) {
    S.k[x] = e.k;
    if constexpr (KV) { S.i[x] = e.i; S.v[x] = e.v; }
}

// a group of len <= 32*R items in shared memory, sorted in place by one warp
template <class U, bool KV, int R>
__device__ __forceinline__ void warp_sort_group(const BucketSmem<U, KV>& S, u32 gs, u32 len) {
    typedef Elem<U, KV> E;
    const int lane = threadIdx.x & 31;
    E a[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const u32 e = r * 32 + lane;
        a[r] = e < len ? sm_get<U, KV>(S, gs + e) : E::inf();
    }
    warp_bitonic<E, R>(a);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const u32 e = r * 32 + lane;
        if (e < len) sm_put<U, KV>(S, gs + e, a[r]);
    }
}

template <class U, bool KV>
__device__ __forceinline__ void smem_cex(const BucketSmem<U, KV>& S, u32 x, u32 y) {
    bool gt;
    if constexpr (KV) gt = S.k[y] < S.k[x] || (S.k[y] == S.k[x] && S.i[y] < S.i[x]);
    else gt = S.k[y] < S.k[x];
    if (gt) {
        U t = S.k[x]; S.k[x] = S.k[y]; S.k[y] = t;
        if constexpr (KV) {
            u32 a = S.i[x]; S.i[x] = S.i[y]; S.i[y] = a;
            u32 b = S.v[x]; S.v[x] = S.v[y]; S.v[y] = b;
        }
    }
}

template <class U> __device__ __forceinline__ u32 lower_bound_kt(const U* sk, const u32* st, u32 nsp, U k, u32 tag) {
    u32 lo = 0, cnt = nsp;
    while (cnt > 0) {
        const u32 half = cnt >> 1, mid = lo + half;
        const bool less = sk[mid] < k || (sk[mid] == k && st[mid] < tag);
        if (less) { lo = mid + 1; cnt -= half + 1; } else cnt = half;
    }
    return lo;
}

// ---- 32-bit keys-only buckets: the item array is swizzled at 16-byte
// granularity (chunk c of 4 keys lives at chunk c ^ ((c >> 2) & 7)), so that the 16-key windows
// below (4 chunks per thread, consecutive threads on consecutive windows) and the sequential
// write-out both touch 8 distinct 16-byte bank groups per quarter warp (no bank conflicts).
__device__ __forceinline__ u32 sw16(u32 P) { return P ^ (((P >> 4) & 7u) << 2); }
__device__ __forceinline__ void cexu(u32& a, u32& b) {
    const u32 lo = min(a, b);
    b = max(a, b);
    a = lo;
}
// Batcher odd-even merge sort of 16 (63 comparators) and the merge of two sorted 8s (25)
__device__ __forceinline__ void sort8u(u32* a) {
    cexu(a[0], a[1]); cexu(a[2], a[3]); cexu(a[4], a[5]); cexu(a[6], a[7]);
    cexu(a[0], a[2]); cexu(a[1], a[3]); cexu(a[4], a[6]); cexu(a[5], a[7]);
    cexu(a[1], a[2]); cexu(a[5], a[6]);
    cexu(a[0], a[4]); cexu(a[1], a[5]); cexu(a[2], a[6]); cexu(a[3], a[7]);
    cexu(a[2], a[4]); cexu(a[3], a[5]);
    cexu(a[1], a[2]); cexu(a[3], a[4]); cexu(a[5], a[6]);
}
__device__ __forceinline__ void merge16u(u32 (&a)[16]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) cexu(a[i], a[i + 8]);
    cexu(a[4], a[8]); cexu(a[5], a[9]); cexu(a[6], a[10]); cexu(a[7], a[11]);
    cexu(a[2], a[4]); cexu(a[3], a[5]); cexu(a[6], a[8]); cexu(a[7], a[9]); cexu(a[10], a[12]); cexu(a[11], a[13]);
    cexu(a[1], a[2]); cexu(a[3], a[4]); cexu(a[5], a[6]); cexu(a[7], a[8]); cexu(a[9], a[10]); cexu(a[11], a[12]);
    cexu(a[13], a[14]);
}
__device__ __forceinline__ void sort16u(u32 (&a)[16]) {
    sort8u(a);
    sort8u(a + 8);
    merge16u(a);
}
// load / store the 16 keys of a window that starts at physical chunk c0 (4 chunks)
__device__ __forceinline__ void win_ld(const u32* kb, u32 c0, u32 (&e)[16]) {
    const uint4* k4 = (const uint4*)kb;
#pragma unroll
    for (u32 j = 0; j < 4; ++j) {
        const u32 c = c0 + j;
        const uint4 v = k4[c ^ ((c >> 2) & 7u)];
        e[4 * j] = v.x; e[4 * j + 1] = v.y; e[4 * j + 2] = v.z; e[4 * j + 3] = v.w;
    }
}
__device__ __forceinline__ void win_st(u32* kb, u32 c0, const u32 (&e)[16]) {
    uint4* k4 = (uint4*)kb;
#pragma unroll
    for (u32 j = 0; j < 4; ++j) {
        const u32 c = c0 + j;
        k4[c ^ ((c >> 2) & 7u)] = make_uint4(e[4 * j], e[4 * j + 1], e[4 * j + 2], e[4 * j + 3]);
    }
}
// a group of len <= 32*R swizzled keys (logical start gs, alignment offset al) sorted by one warp
template <int R>
__device__ __forceinline__ void warp_sort_sw(u32* kb, u32 al, u32 gs, u32 len) {
    typedef Elem<u32, false> E;
    const int lane = threadIdx.x & 31;
    E a[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const u32 e = r * 32 + lane;
        a[r].k = e < len ? kb[sw16(gs + e + al)] : 0xffffffffu;
    }
    warp_bitonic<E, R>(a);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const u32 e = r * 32 + lane;
        if (e < len) kb[sw16(gs + e + al)] = a[r].k;
    }
}

template <class U, bool KV> __host__ __device__ constexpr size_t bucket_smem_fixed() {
    return 4 * ((size_t)BS_NGMAX + 4) + 96;  // group counters + slack of the items (alignment, window tails)
}
template <class U, bool KV> __host__ __device__ constexpr size_t bucket_item_bytes() {
    return sizeof(U) + (KV ? 8 : 0);
}

// WIN = false: buckets that fit on chip, oversized ones re-split or (up to BS_WMAX * cap, not in
// the output array) appended to wlist; WIN = true: the wlist buckets, sorted on chip in windows
// of consecutive digit groups (kept out of the first kernel: its register allocation, and so the
// common path's speed, must not pay for the window loop)
template <int DT, bool KV, bool WIN>
__global__ void __launch_bounds__(BS_NT, 1) k_bucket_sort(const Bucket* list, const u32* nlist, u32* ticket,
                                                           Bufs<typename Codec<DT>::U> B, typename Codec<DT>::U* okeys,
                                                           u32* ovals, u32* oidx, bool out_raw, u32 cap,
                                                           Bucket* stack_pool, u64 seed, u32* status, u32 ixbits,
                                                           Bucket* wlist, u32* nwlist, u32 wcap) {
    // ixbits: key-value sorts' indices are < 2^ixbits
    PDL_PROLOGUE();
    typedef typename Codec<DT>::U U;
    typedef Elem<U, KV> E;
    extern __shared__ __align__(16) char smem[];
    __shared__ u32 red[BS_NT / 32 + 1];
    __shared__ u32 s_work, s_next, s_nbig, s_nhuge, s_over, s_sp;
    __shared__ u32 s_big[BS_BIGMAX];
    __shared__ u32 s_huge[BS_HUGEMAX];
    __shared__ U s_mn[BS_NT / 32], s_mx[BS_NT / 32];
    __shared__ u32 s_hl[4][BS_NT / 32];  // DT_U64 records: key-word and tag-word ranges
    __shared__ U sp_k[BS_SPMAX];
    __shared__ u32 sp_t[BS_SPMAX], sp_cnt[BS_SPMAX + 1], sp_cur[BS_SPMAX];
    __shared__ u32 rs_cnt[BS_SPMAX], rs_off[BS_SPMAX], s_w[4];
    __shared__ u32 rs_red[BS_NT / 32 + 1][4];
    __shared__ int rs_base[BS_SPMAX];
    BucketSmem<U, KV> S;
    {
        char* sp = smem;
        S.cnt = (u32*)sp; sp += 4 * ((size_t)BS_NGMAX + 4);
        S.k = (U*)sp; sp += sizeof(U) * (size_t)cap + 96;
        if (KV) { S.i = (u32*)sp; sp += 4 * (size_t)cap; S.v = (u32*)sp; sp += 4 * (size_t)cap; }
    }
    Bucket* stk = stack_pool + (size_t)blockIdx.x * BS_STACK;
    const u32 nl = *nlist;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#ifdef OVS_BS_PROF
    const long long bs_start_ = clock64();
#endif
    // Work distribution: the next bucket is claimed (ticket) and its descriptor loaded one bucket
    // ahead, and the claim after that is issued at the start of a bucket and consumed at its end,
    // so no global round trip sits between two buckets.  The claimed bucket is kept in shared
    // memory; only resplit children go through the CTA's stack in global memory.
    __shared__ Bucket s_cur, s_nxt;
    __shared__ u32 s_base, s_first;
    if (threadIdx.x == 0) {
        s_first = 1;
        s_work = atomicAdd(ticket, 1u);
        if (s_work < nl) s_cur = list[s_work];
        s_next = atomicAdd(ticket, 1u);
        if (s_next < nl) s_nxt = list[s_next];
    }
    __syncthreads();
    for (;;) {
        if (s_work >= nl) break;
        u32 t3 = 0xffffffffu;  // thread 0: the claim after the next one (consumed at the end)
        if (threadIdx.x == 0) {
            // bucket keys into L2 with one bulk prefetch (16-byte aligned cover)
            auto prefetch = [&](const Bucket& nx) {
                const uintptr_t a0 = (uintptr_t)(B.k[nx.buf] + nx.beg) & ~(uintptr_t)15;
                const uintptr_t a1 = ((uintptr_t)(B.k[nx.buf] + nx.beg + nx.len) + 15) & ~(uintptr_t)15;
                if (a1 > a0)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((u32)(a1 - a0)) : "memory");
            };
            // the next bucket (OVS_BS_PF2: already prefetched one bucket earlier, except the first)
            if (s_next < nl && (!OVS_BS_PF2 || s_first)) prefetch(s_nxt);
            t3 = atomicAdd(ticket, 1u);
            if (OVS_BS_PF2 && t3 < nl) prefetch(list[t3]);  // the bucket after it
            s_first = 0;
            s_sp = 0;
            s_base = 1;
        }
        __syncthreads();
        while (s_base || s_sp > 0) {
            const Bucket bk = s_base ? s_cur : stk[s_sp - 1];
            __syncthreads();
            if (threadIdx.x == 0) {
                if (s_base) s_base = 0; else s_sp -= 1;
                s_nbig = 0; s_nhuge = 0; s_over = 0;
            }
            const u32 m = bk.len;
            const U* src = B.k[bk.buf];
            const u32* vsrc = KV ? B.v[bk.buf] : nullptr;
            const u32* isrc = KV ? B.i[bk.buf] : nullptr;
            const bool rawin = (bk.level & BK_RAW) != 0;
            auto K = [&](U x) -> U { return rawin ? Codec<DT>::ord(x) : x; };
            auto IX = [&](u32 pos) -> u32 { return (KV && !rawin) ? isrc[pos] : pos; };
            BS_T0
            // windows re-read the bucket after writing earlier windows' output: only when the
            // bucket does not live in the output array
            const bool can_window = (const void*)B.k[bk.buf] != (const void*)okeys;
            // (slightly oversized buckets, m <= 1.1 cap, are re-split right here: they are rare
            // outliers of a bucket-size distribution that fits, and the window launch only starts
            // after this one, so a few of them would sit alone in its tail)
            if (!WIN && m > cap + cap / 10 && m <= BS_WMAX * cap && can_window && !(bk.level & BK_FORCE)) {
                // sorted on chip in windows by the second launch (k_bucket_sort<..., true>)
                if (threadIdx.x == 0) {
                    const u32 w = atomicAdd(nwlist, 1u);
                    if (w < wcap) wlist[w] = bk; else st_set(status, ST_LIST_OVER);
                }
                __syncthreads();
                continue;
            }
            if (m > cap && (m > BS_WMAX * cap || (bk.level & BK_FORCE) || !can_window || !WIN)) {
                // ---------------- CTA-local re-split of an oversized bucket
                const u32 part = (u32)((cap * 60ull) / 100);
                u32 P = (m + part - 1) / part;
                P = max(2u, min(BS_SPMAX, P));
                const u32 ms = P * BS_SI - 1;
                u32 NS = 32;  // the sample, padded to a power of two for the bitonic network
                while (NS < ms) NS <<= 1;
                U* tk = S.k;
                u32* tt = (u32*)(smem + bucket_smem_fixed<U, KV>() + sizeof(U) * BS_SSMAX);
                for (u32 j = threadIdx.x; j < NS; j += BS_NT) {
                    if (j < ms) {
                        const u64 u = rng_H(seed ^ ((u64)bk.beg * 0x9e3779b97f4a7c15ull), 64 + (bk.level & 0xffffu), j);
                        const u32 o = (u32)__umul64hi(u, (u64)m);
                        tk[j] = K(src[bk.beg + o]);
                        tt[j] = IX(bk.beg + o);
                    } else {
                        tk[j] = umax_of<U>();
                        tt[j] = 0xffffffffu;
                    }
                }
                __syncthreads();
                cta_bitonic_kt<U>(tk, tt, NS);
                if (threadIdx.x + 1 < P) {
                    sp_k[threadIdx.x] = tk[(threadIdx.x + 1) * BS_SI - 1];
                    sp_t[threadIdx.x] = tt[(threadIdx.x + 1) * BS_SI - 1];
                }
                if (threadIdx.x <= P) sp_cnt[threadIdx.x] = 0;
                if (threadIdx.x < BS_SPMAX) rs_cnt[threadIdx.x] = 0;
                __syncthreads();
                BS_PROBE(10)
                // P <= 8: per-thread counters in registers, two 16-bit fields per word (a thread sees
                // < 2^16 keys: m <= 64 * cap), one CTA reduction; otherwise shared atomics (a fan-out
                // this small makes them collide on the same counters)
                const bool small = P <= 8;
                u32 pc[4] = {0u, 0u, 0u, 0u};
                for_items<U, BS_NT, OVS_BS_UNR>(src, bk.beg, m, [&](U kr, u32 o) {
                    const U k = K(kr);
                    const u32 tg = IX(bk.beg + o);
                    const u32 b = lower_bound_kt<U>(sp_k, sp_t, P - 1, k, tg);
                    if (small) {
#pragma unroll
                        for (u32 q = 0; q < 4; ++q) pc[q] += (b >> 1) == q ? (1u << (16 * (b & 1))) : 0u;
                    } else {
                        atomicAdd(&sp_cnt[b], 1u);
                    }
                });
                if (small) {
                    u32 tot[4];
                    block_exclusive_scan4<BS_NT>(pc, rs_red, tot);
                    if (threadIdx.x < P) sp_cnt[threadIdx.x] = (tot[threadIdx.x >> 1] >> (16 * (threadIdx.x & 1))) & 0xffffu;
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    u32 run = 0;
                    for (u32 b = 0; b < P; ++b) { const u32 c = sp_cnt[b]; sp_cnt[b] = run; sp_cur[b] = run; run += c; }
                    sp_cnt[P] = run;
                }
                __syncthreads();
                BS_PROBE(11)
                // scatter in tiles of RS_IT * BS_NT items staged in shared memory by sub-bucket, so
                // every sub-bucket's items of a tile leave as one coalesced run (whole sectors)
                const u32 db = 1 - bk.buf;
                constexpr u32 RS_IT = 8, RT = RS_IT * BS_NT;
                uint8_t* sbk = (uint8_t*)S.cnt;  // sub-bucket of each staged item
                for (u32 t0 = 0; t0 < m; t0 += RT) {
                    const u32 nt = min(RT, m - t0);
                    U kk[RS_IT];
                    u32 tg[RS_IT], vv[RS_IT], bb[RS_IT], rr[RS_IT];
#pragma unroll
                    for (u32 j = 0; j < RS_IT; ++j) {
                        const u32 o = j * BS_NT + threadIdx.x;
                        if (o < nt) {
                            kk[j] = K(src[bk.beg + t0 + o]);
                            tg[j] = IX(bk.beg + t0 + o);
                            if (KV) vv[j] = vsrc[bk.beg + t0 + o];
                        }
                    }
#pragma unroll
                    for (u32 j = 0; j < RS_IT; ++j)
                        if (j * BS_NT + threadIdx.x < nt) bb[j] = lower_bound_kt<U>(sp_k, sp_t, P - 1, kk[j], tg[j]);
                    if (small) {
                        // rank = the thread's earlier items of the bucket + the earlier threads' (one
                        // scan of packed 16-bit counters); tile totals -> rs_cnt
                        u32 w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
                        for (u32 j = 0; j < RS_IT; ++j) {
                            if (j * BS_NT + threadIdx.x < nt) {
                                const u32 q = bb[j] >> 1, sh = 16 * (bb[j] & 1);
                                u32 cur = 0;
#pragma unroll
                                for (u32 x = 0; x < 4; ++x) cur = x == q ? w[x] : cur;
                                rr[j] = (cur >> sh) & 0xffffu;
#pragma unroll
                                for (u32 x = 0; x < 4; ++x) w[x] += x == q ? (1u << sh) : 0u;
                            }
                        }
                        u32 ex[4] = {w[0], w[1], w[2], w[3]}, tot[4];
                        block_exclusive_scan4<BS_NT>(ex, rs_red, tot);
#pragma unroll
                        for (u32 j = 0; j < RS_IT; ++j) {
                            if (j * BS_NT + threadIdx.x < nt) {
                                const u32 q = bb[j] >> 1, sh = 16 * (bb[j] & 1);
                                u32 e0 = 0;
#pragma unroll
                                for (u32 x = 0; x < 4; ++x) e0 = x == q ? ex[x] : e0;
                                rr[j] += (e0 >> sh) & 0xffffu;
                            }
                        }
                        if (threadIdx.x < P) rs_cnt[threadIdx.x] = (tot[threadIdx.x >> 1] >> (16 * (threadIdx.x & 1))) & 0xffffu;
                    } else {
#pragma unroll
                        for (u32 j = 0; j < RS_IT; ++j)
                            if (j * BS_NT + threadIdx.x < nt) rr[j] = atomicAdd(&rs_cnt[bb[j]], 1u);
                    }
                    __syncthreads();
                    if (threadIdx.x < 32) {  // tile offsets (P <= 64: two per lane) and run bases
                        const u32 b0 = 2 * threadIdx.x, b1 = b0 + 1;
                        const u32 c0 = b0 < P ? rs_cnt[b0] : 0u, c1 = b1 < P ? rs_cnt[b1] : 0u;
                        u32 x = c0 + c1;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const u32 y = __shfl_up_sync(0xffffffffu, x, o);
                            if (threadIdx.x >= (u32)o) x += y;
                        }
                        const u32 ex = x - c0 - c1;
                        if (b0 < P) { rs_off[b0] = ex; rs_base[b0] = (int)sp_cur[b0] - (int)ex; sp_cur[b0] += c0; rs_cnt[b0] = 0; }
                        if (b1 < P) { rs_off[b1] = ex + c0; rs_base[b1] = (int)sp_cur[b1] - (int)(ex + c0); sp_cur[b1] += c1; rs_cnt[b1] = 0; }
                    }
                    __syncthreads();
#pragma unroll
                    for (u32 j = 0; j < RS_IT; ++j) {
                        if (j * BS_NT + threadIdx.x < nt) {
                            const u32 s = rs_off[bb[j]] + rr[j];
                            S.k[s] = kk[j];
                            sbk[s] = (uint8_t)bb[j];
                            if (KV) { S.i[s] = tg[j]; S.v[s] = vv[j]; }
                        }
                    }
                    __syncthreads();
                    for (u32 s = threadIdx.x; s < nt; s += BS_NT) {
                        const u32 d = bk.beg + (u32)(rs_base[sbk[s]] + (int)s);
                        B.k[db][d] = S.k[s];
                        if (KV) { B.v[db][d] = S.v[s]; B.i[db][d] = S.i[s]; }
                    }
                    __syncthreads();
                }
                BS_PROBE(12)
                if (threadIdx.x == 0) {
                    u32 sp = s_sp;
                    for (int b = (int)P - 1; b >= 0; --b) {
                        const u32 len = sp_cnt[b + 1] - sp_cnt[b];
                        if (len == 0) continue;
                        if (sp >= BS_STACK) { st_set(status, ST_LIST_OVER); break; }
                        Bucket nb;
                        nb.beg = bk.beg + sp_cnt[b]; nb.len = len; nb.buf = db;
                        const bool edge = (b == 0 || b + 1 == (int)P);
                        nb.level = ((bk.level & 0xffffu) + 1) | ((edge && (bk.level & BK_LOOSE)) ? BK_LOOSE : 0u);
                        nb.lo = (b == 0) ? bk.lo : (u64)sp_k[b - 1];
                        nb.hi = (b + 1 == (int)P) ? bk.hi : (u64)sp_k[b];
                        stk[sp++] = nb;
                    }
                    s_sp = sp;
                }
                __syncthreads();
                BS_PROBE(0)
                continue;
            }
            if constexpr (!WIN) {
                // ---------------- on-chip sort of a bucket that fits
                // items sit at shared index = output address mod 16 bytes, so the write-out is aligned
                // 16-byte shared loads and global stores
                BucketSmem<U, KV> Sa = S;
                Sa.k = S.k + ((((uintptr_t)(okeys + bk.beg)) / sizeof(U)) & (16 / sizeof(U) - 1));
                BS_PROBE(1)
                U lo = (U)bk.lo, hi = (U)bk.hi;
                // internal records (DT_U64: key word << 32 | tag) whose key words take few values
                // (few distinct keys) sit in a few narrow clusters of the record range, so a digit
                // over [lo, hi] puts each cluster in one or two huge groups: such buckets take a
                // two-level digit instead, (key word - its min) * per + the tag's digit inside
                // [min tag, max tag] over per groups (monotone in the record)
                bool two = false;
                u32 hmn = 0, per = 1, lmn = 0, multl = 0;
                if constexpr (DT == DT_U64 && !KV) {
                    u32 a = 0xffffffffu, b = 0, c2 = 0xffffffffu, d = 0;
                    for_items<U, BS_NT, OVS_BS_UNR>(src, bk.beg, m, [&](U k, u32) {
                        const u32 h = (u32)((u64)k >> 32), l = (u32)k;
                        a = min(a, h); b = max(b, h); c2 = min(c2, l); d = max(d, l);
                    });
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        a = min(a, __shfl_xor_sync(0xffffffffu, a, o)); b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
                        c2 = min(c2, __shfl_xor_sync(0xffffffffu, c2, o)); d = max(d, __shfl_xor_sync(0xffffffffu, d, o));
                    }
                    if (lane == 0) { s_hl[0][wid] = a; s_hl[1][wid] = b; s_hl[2][wid] = c2; s_hl[3][wid] = d; }
                    __syncthreads();
                    a = s_hl[0][0]; b = s_hl[1][0]; c2 = s_hl[2][0]; d = s_hl[3][0];
                    for (int q = 1; q < BS_NT / 32; ++q) {
                        a = min(a, s_hl[0][q]); b = max(b, s_hl[1][q]); c2 = min(c2, s_hl[2][q]); d = max(d, s_hl[3][q]);
                    }
                    __syncthreads();
                    lo = ((u64)a << 32) | c2;  // every record lies in [lo, hi] (tighter than the bounds)
                    hi = ((u64)b << 32) | d;
                    u32 ngt = 32;
                    while (ngt < (u32)BS_NGMAX && ngt * 3 < m) ngt <<= 1;
                    const u64 H = (u64)b - a + 1;
                    if (H >= 2 && H * 4 <= ngt) {
                        two = true;
                        hmn = a;
                        per = ngt / (u32)H;
                        lmn = c2;
                        const double mqt = (double)per * 4294967296.0 / ((double)(d - c2) + 1.0);
                        multl = mqt >= 4294967295.0 ? 0xffffffffu : (u32)mqt;
                    }
                }
                if ((bk.level & BK_LOOSE) && !(DT == DT_U64 && !KV)) {
                    U mn = umax_of<U>(), mx = 0;
                    for_items<U, BS_NT, OVS_BS_UNR>(src, bk.beg, m, [&](U kr, u32) { const U k = K(kr); mn = min(mn, k); mx = max(mx, k); });
    #pragma unroll
                    for (int o = 16; o > 0; o >>= 1) { mn = min(mn, shfl_xor_any(mn, o)); mx = max(mx, shfl_xor_any(mx, o)); }
                    if (lane == 0) { s_mn[wid] = mn; s_mx[wid] = mx; }
                    __syncthreads();
                    mn = s_mn[0]; mx = s_mx[0];
                    for (int q = 1; q < BS_NT / 32; ++q) { mn = min(mn, s_mn[q]); mx = max(mx, s_mx[q]); }
                    lo = mn; hi = mx;
                    __syncthreads();
                }
                u32 ng = 32;
                while (ng < (u32)BS_NGMAX && ng * 3 < m) ng <<= 1;
                // digit = floor(x * ng / R) for x = (sort key - lo) in [0, R): monotone in the key
                // and spreads [lo, hi] over all ng groups (computed as a 64-bit fixed-point
                // multiply-high).  Key-value sorts of 32-bit keys use the composite (key, index) with
                // the index in its ixbits low bits (indices < 2^ixbits, so the groups spread over the
                // indices that occur); 64-bit keys use the key (equal keys share a group, ordered by
                // index).  R <= ng: digit = x, every group holds one key value (keys only: the groups
                // need no sorting, e.g. few distinct keys).
                const bool comp = KV && sizeof(U) == 4;
                const u64 xmax = comp ? ((((u64)(hi - lo)) << ixbits) | ((1ull << ixbits) - 1)) : (u64)(U)(hi - lo);
                const bool direct = xmax < (u64)ng;
                // multiplier ~ ng * 2^64 / R in double precision: any multiplier keeps the digit monotone
                // (and the clamp keeps it < ng), so rounding only perturbs the group sizes slightly
                const double mq = (double)ng * 18446744073709551616.0 / ((double)xmax + 1.0);
                const u64 mult = mq >= 18446744073709549568.0 ? 0xffffffffffffffffull : (u64)mq;
                const double mq32 = mq * (1.0 / 4294967296.0);
                const u32 mult32 = mq32 >= 4294967295.0 ? 0xffffffffu : (u32)mq32;
                auto digit = [&](U k, u32 ix) -> u32 {
                    if constexpr (!KV && sizeof(U) == 4) {
                        const u32 x = (u32)(k - lo);
                        return direct ? x : min(__umulhi(x, mult32), ng - 1);  // min: memory safety only
                    } else {
                        if (DT == DT_U64 && !KV && two) {
                            const u32 h = (u32)((u64)k >> 32) - hmn, l = (u32)k - lmn;
                            return min(h * per + min(__umulhi(l, multl), per - 1), ng - 1);
                        }
                        const u64 x = comp ? ((((u64)(k - lo)) << ixbits) | ix) : (u64)(U)(k - lo);
                        return direct ? (u32)x : min((u32)__umul64hi(x, mult), ng - 1);
                    }
                };
                const bool need_sort = KV || !direct || two;
                constexpr bool FAST32 = !KV && sizeof(U) == 4 && OVS_BS_WIN16;
                for (u32 g = threadIdx.x; g < ng; g += BS_NT) Sa.cnt[g] = 0;
                __syncthreads();
                BS_PROBE(2)
                // 1. digit histogram
                for_items<U, BS_NT, OVS_BS_UNR>(src, bk.beg, m, [&](U kr, u32 o) {
                    const u32 ix = KV ? IX(bk.beg + o) : 0u;
                    atomicAdd(&Sa.cnt[digit(K(kr), ix)], 1u);
                });
                __syncthreads();
                BS_PROBE(3)
                if constexpr (FAST32) {
                    // (groups of >= 10 keys are listed here for the window networks below)
                    block_scan_small_list<BS_NT>(Sa.cnt, ng, red, need_sort ? 10u : 0xffffffffu, s_big, &s_nbig,
                                                 (u32)BS_BIGMAX, &s_over);
                } else {
                    block_scan_small<BS_NT>(Sa.cnt, ng, red);  // cnt[g] = start of group g
                }
                BS_PROBE(4)
                if constexpr (FAST32) {
                    // ---- 32-bit keys only: swizzled item array, windowed networks
                    u32* const kb = (u32*)S.k;  // 16-byte aligned; logical item x at kb[sw16(x + al)]
                    const u32 al = (u32)(((uintptr_t)(okeys + bk.beg)) / sizeof(U)) & 3u;
                    // 2. scatter into shared memory by digit; afterwards cnt[g] = end of group g
                    for_items<U, BS_NT, OVS_BS_UNR>(src, bk.beg, m, [&](U kr, u32) {
                        const u32 k = (u32)K(kr);
                        const u32 pos = atomicAdd(&S.cnt[digit((U)k, 0u)], 1u);
                        kb[sw16(pos + al)] = k;
                    });
                    __syncthreads();
                    BS_PROBE(5)
                    if (need_sort) {
                        // groups of >= 10 keys were listed by the scan; every shorter group lies inside
                        // one window of 16 consecutive keys starting at a multiple of 8 (pass A: starts
                        // 16w, pass B: 16w + 8), and sorting a window by key never breaks the digit order
                        // pass A: physical windows [16w, 16w + 16); slots outside [al, al + m) get the
                        // minimum / maximum key, so they stay in place
                        const u32 nw = (al + m + 15) >> 4;
                        for (u32 w = threadIdx.x; w < nw; w += BS_NT) {
                            u32 e[16];
                            win_ld(kb, 4 * w, e);
                            if (16 * w < al || 16 * w + 16 > al + m) {  // the two edge windows only
#pragma unroll
                                for (u32 i = 0; i < 16; ++i) {
                                    const u32 P = 16 * w + i;
                                    if (P < al) e[i] = 0u;
                                    else if (P >= al + m) e[i] = 0xffffffffu;
                                }
                            }
                            sort16u(e);
                            win_st(kb, 4 * w, e);
                        }
                        __syncthreads();
                        // pass B: windows [16w + 8, 16w + 24) = two sorted halves: one merge
                        for (u32 w = threadIdx.x; w + 1 < nw; w += BS_NT) {
                            u32 e[16];
                            win_ld(kb, 4 * w + 2, e);
                            merge16u(e);
                            win_st(kb, 4 * w + 2, e);
                        }
                        __syncthreads();
                        BS_PROBE(6)
                        const u32 nlisted = min(s_nbig, (u32)BS_BIGMAX);
                        const bool rescan = s_over != 0;  // list overflow (pathological skew): scan all groups
                        const u32 nwork = rescan ? ng : nlisted;
                        // listed groups of 10..16: one thread each
                        for (u32 q = threadIdx.x; q < nwork; q += BS_NT) {
                            const u32 g = rescan ? q : s_big[q];
                            const u32 gs = g ? S.cnt[g - 1] : 0u, len = S.cnt[g] - gs;
                            if (len < 10 || len > 16) continue;
                            u32 e[16];
#pragma unroll
                            for (u32 t = 0; t < 16; ++t) e[t] = t < len ? kb[sw16(gs + t + al)] : 0xffffffffu;
                            sort16u(e);
#pragma unroll
                            for (u32 t = 0; t < 16; ++t)
                                if (t < len) kb[sw16(gs + t + al)] = e[t];
                        }
                        // 17..512: one warp each (register bitonic); larger: the CTA
                        for (u32 q = wid; q < nwork; q += BS_NT / 32) {
                            const u32 g = rescan ? q : s_big[q];
                            const u32 gs = g ? S.cnt[g - 1] : 0u, len = S.cnt[g] - gs;
                            if (len <= 16) continue;
                            if (len <= 32) warp_sort_sw<1>(kb, al, gs, len);
                            else if (len <= 64) warp_sort_sw<2>(kb, al, gs, len);
                            else if (len <= 128) warp_sort_sw<4>(kb, al, gs, len);
                            else if (len <= 256) warp_sort_sw<8>(kb, al, gs, len);
                            else if (len <= 512 && BS_WARPMAX >= 512) warp_sort_sw<BS_WARPMAX / 32>(kb, al, gs, len);
                            else if (lane == 0) {
                                const u32 h = atomicAdd(&s_nhuge, 1u);
                                if (h < BS_HUGEMAX) s_huge[h] = g;
                                else st_set(status, ST_LIST_OVER);
                            }
                        }
                        __syncthreads();
                        BS_PROBE(7)
                        const u32 nhuge = min(s_nhuge, (u32)BS_HUGEMAX);
                        for (u32 q = 0; q < nhuge; ++q) {
                            const u32 g = s_huge[q];
                            const u32 gs = g ? S.cnt[g - 1] : 0u, len = S.cnt[g] - gs;
                            u32 N = 1;
                            while (N < len) N <<= 1;
                            auto cx = [&](u32 x, u32 y) {
                                const u32 px = sw16(gs + x + al), py = sw16(gs + y + al);
                                const u32 u = kb[px], v = kb[py];
                                if (v < u) { kb[px] = v; kb[py] = u; }
                            };
                            for (u32 kk = 2; kk <= N; kk <<= 1) {
                                const u32 hk = kk >> 1;
                                for (u32 t = threadIdx.x; t < N / 2; t += BS_NT) {
                                    const u32 blk = t / hk, off = t % hk;
                                    const u32 x = blk * kk + off, y = blk * kk + kk - 1 - off;
                                    if (y < len) cx(x, y);
                                }
                                __syncthreads();
                                for (u32 j = kk >> 2; j > 0; j >>= 1) {
                                    for (u32 t = threadIdx.x; t < N / 2; t += BS_NT) {
                                        const u32 x = (t / j) * 2 * j + (t % j), y = x + j;
                                        if (y < len) cx(x, y);
                                    }
                                    __syncthreads();
                                }
                            }
                        }
                    }
                    __syncthreads();
                    BS_PROBE(8)
                    // 4. write the sorted bucket: swizzled 16-byte shared loads, 16-byte global stores
                    {
                        U* out = okeys + bk.beg;
                        const u32 head = al ? min(m, 4u - al) : 0u;
                        auto R = [&](u32 x) -> u32 { return out_raw ? (u32)Codec<DT>::raw((U)x) : x; };
                        if (threadIdx.x < head) out[threadIdx.x] = (U)R(kb[sw16(threadIdx.x + al)]);
                        const u32 nv = (m - head) / 4;
                        uint4* o4 = (uint4*)(out + head);
                        const uint4* k4 = (const uint4*)kb;
                        const u32 c0 = (head + al) >> 2;
                        for (u32 v = threadIdx.x; v < nv; v += BS_NT) {
                            const u32 c = c0 + v;
                            uint4 r = k4[c ^ ((c >> 2) & 7u)];
                            r.x = R(r.x); r.y = R(r.y); r.z = R(r.z); r.w = R(r.w);
                            if (OVS_BS_STCS) __stcs(o4 + v, r);  // evict-first: keep the prefetched buckets in L2
                            else o4[v] = r;
                        }
                        for (u32 o = head + nv * 4 + threadIdx.x; o < m; o += BS_NT) out[o] = (U)R(kb[sw16(o + al)]);
                    }
                } else {
                    // 2. scatter into shared memory by digit; afterwards cnt[g] = end of group g
                    for_items<U, BS_NT, OVS_BS_UNR>(src, bk.beg, m, [&](U kr, u32 o) {
                        const U k = K(kr);
                        u32 ix = 0, vv = 0;
                        if (KV) { ix = IX(bk.beg + o); vv = vsrc[bk.beg + o]; }
                        const u32 pos = atomicAdd(&Sa.cnt[digit(k, ix)], 1u);
                        Sa.k[pos] = k;
                        if (KV) { Sa.i[pos] = ix; Sa.v[pos] = vv; }
                    });
                    __syncthreads();
                    BS_PROBE(5)
                    // 3. one thread per group of <= 8: Batcher network in registers; larger groups are
                    // appended (warp-aggregated) to a list for 3b
                    // (OVS_NET8_X: groups per thread per iteration, their loads and networks interleaved)
                    for (u32 g0 = 0; need_sort && g0 < ng; g0 += BS_NT * OVS_NET8_X) {
                        u32 gs[OVS_NET8_X], len[OVS_NET8_X];
                        E a[OVS_NET8_X][8];
        #pragma unroll
                        for (int x = 0; x < OVS_NET8_X; ++x) {
                            const u32 g = g0 + x * BS_NT + threadIdx.x;
                            gs[x] = 0; len[x] = 0;
                            if (g < ng) { gs[x] = g ? Sa.cnt[g - 1] : 0u; len[x] = Sa.cnt[g] - gs[x]; }
                        }
        #pragma unroll
                        for (int x = 0; x < OVS_NET8_X; ++x) {
                            const u32 lx = (len[x] > 1 && len[x] <= 8) ? len[x] : 0u;
        #pragma unroll
                            for (u32 q = 0; q < 8; ++q) a[x][q] = q < lx ? sm_get<U, KV>(Sa, gs[x] + q) : E::inf();
                        }
        #pragma unroll
                        for (int x = 0; x < OVS_NET8_X; ++x) network8(a[x]);
        #pragma unroll
                        for (int x = 0; x < OVS_NET8_X; ++x) {
                            const u32 lx = (len[x] > 1 && len[x] <= 8) ? len[x] : 0u;
        #pragma unroll
                            for (u32 q = 0; q < 8; ++q)
                                if (q < lx) sm_put<U, KV>(Sa, gs[x] + q, a[x][q]);
                        }
        #pragma unroll
                        for (int x = 0; x < OVS_NET8_X; ++x) {
                            const u32 g = g0 + x * BS_NT + threadIdx.x;
                            const u32 mb = __ballot_sync(0xffffffffu, len[x] > 8);
                            if (mb) {
                                u32 base = 0;
                                if (lane == 0) base = atomicAdd(&s_nbig, __popc(mb));
                                base = __shfl_sync(0xffffffffu, base, 0) + __popc(mb & ((1u << lane) - 1));
                                if (len[x] > 8) {
                                    if (base < BS_BIGMAX) s_big[base] = g;
                                    else atomicOr(&s_over, 1u);
                                }
                            }
                        }
                    }
                    __syncthreads();
                    BS_PROBE(6)
                    // 3b. listed groups of 9..16: one thread each (63-comparator network)
                    const u32 nlisted = min(s_nbig, (u32)BS_BIGMAX);
                    const bool rescan = s_over != 0;  // list overflow (pathological skew): scan all groups
                    const u32 nwork = rescan ? ng : nlisted;
                    for (u32 q = threadIdx.x; q < nwork; q += BS_NT) {
                        const u32 g = rescan ? q : s_big[q];
                        const u32 gs = g ? Sa.cnt[g - 1] : 0u, len = Sa.cnt[g] - gs;
                        if (len <= 8 || len > 16) continue;
                        E a[16];
        #pragma unroll
                        for (u32 t = 0; t < 16; ++t) a[t] = t < len ? sm_get<U, KV>(Sa, gs + t) : E::inf();
                        network16(a);
        #pragma unroll
                        for (u32 t = 0; t < 16; ++t)
                            if (t < len) sm_put<U, KV>(Sa, gs + t, a[t]);
                    }
                    // 3c'. groups of 17..512: one warp each (register bitonic); over 512: the CTA
                    for (u32 q = wid; q < nwork; q += BS_NT / 32) {
                        const u32 g = rescan ? q : s_big[q];
                        const u32 gs = g ? Sa.cnt[g - 1] : 0u, len = Sa.cnt[g] - gs;
                        if (len <= 16) continue;
                        if (len <= 32) warp_sort_group<U, KV, 1>(Sa, gs, len);
                        else if (len <= 64) warp_sort_group<U, KV, 2>(Sa, gs, len);
                        else if (len <= 128) warp_sort_group<U, KV, 4>(Sa, gs, len);
                        else if (len <= 256) warp_sort_group<U, KV, 8>(Sa, gs, len);
                        else if (len <= 512 && BS_WARPMAX >= 512) warp_sort_group<U, KV, BS_WARPMAX / 32>(Sa, gs, len);
                        else if (lane == 0) {
                            const u32 h = atomicAdd(&s_nhuge, 1u);
                            if (h < BS_HUGEMAX) s_huge[h] = g;
                            else st_set(status, ST_LIST_OVER);
                        }
                    }
                    __syncthreads();
                    BS_PROBE(7)
                    // 3c. groups over BS_WARPMAX: in-place bitonic network in shared memory, all comparators
                    // ascending (the first step of each merge compares i with its mirror), so virtual
                    // +inf padding beyond len never moves and len need not be a power of two
                    const u32 nhuge = min(s_nhuge, (u32)BS_HUGEMAX);
                    for (u32 q = 0; q < nhuge; ++q) {
                        const u32 g = s_huge[q];
                        const u32 gs = g ? Sa.cnt[g - 1] : 0u, len = Sa.cnt[g] - gs;
                        u32 N = 1;
                        while (N < len) N <<= 1;
                        for (u32 kk = 2; kk <= N; kk <<= 1) {
                            const u32 hk = kk >> 1;
                            for (u32 t = threadIdx.x; t < N / 2; t += BS_NT) {
                                const u32 blk = t / hk, off = t % hk;
                                const u32 x = blk * kk + off, y = blk * kk + kk - 1 - off;
                                if (y < len) smem_cex<U, KV>(Sa, gs + x, gs + y);
                            }
                            __syncthreads();
                            for (u32 j = kk >> 2; j > 0; j >>= 1) {
                                for (u32 t = threadIdx.x; t < N / 2; t += BS_NT) {
                                    const u32 x = (t / j) * 2 * j + (t % j), y = x + j;
                                    if (y < len) smem_cex<U, KV>(Sa, gs + x, gs + y);
                                }
                                __syncthreads();
                            }
                        }
                    }
                    __syncthreads();
                    BS_PROBE(8)
                    // 4. write the sorted bucket (16-byte stores where the output is aligned)
                    {
                        constexpr u32 V = 16 / sizeof(U);
                        U* out = okeys + bk.beg;
                        const u32 mis = (u32)(((uintptr_t)out) & 15u) / (u32)sizeof(U);
                        const u32 head = mis ? min(m, V - mis) : 0u;
                        auto R = [&](U x) -> U { return out_raw ? Codec<DT>::raw(x) : x; };
                        if (threadIdx.x < head) out[threadIdx.x] = R(Sa.k[threadIdx.x]);
                        const u32 nv = (m - head) / V;
                        uint4* o4 = (uint4*)(out + head);
                        const uint4* s4 = (const uint4*)(Sa.k + head);
                        for (u32 v = threadIdx.x; v < nv; v += BS_NT) {
                            uint4 r = s4[v];
                            U* e = (U*)&r;
        #pragma unroll
                            for (u32 q = 0; q < V; ++q) e[q] = R(e[q]);
                            o4[v] = r;
                        }
                        for (u32 o = head + nv * V + threadIdx.x; o < m; o += BS_NT) out[o] = R(Sa.k[o]);
                        if (KV) {
                            for (u32 o = threadIdx.x; o < m; o += BS_NT) ovals[bk.beg + o] = Sa.v[o];
                            if (oidx)
                                for (u32 o = threadIdx.x; o < m; o += BS_NT) oidx[bk.beg + o] = Sa.i[o];
                        }
                    }
                }
                __syncthreads();
            } else {
                // ---------------- on-chip sort of a bucket that fits
                // items sit at shared index = output address mod 16 bytes, so the write-out is aligned
                // 16-byte shared loads and global stores
                BucketSmem<U, KV> Sa = S;
                Sa.k = S.k + ((((uintptr_t)(okeys + bk.beg)) / sizeof(U)) & (16 / sizeof(U) - 1));
                BS_PROBE(1)
                U lo = (U)bk.lo, hi = (U)bk.hi;
                if (bk.level & BK_LOOSE) {
                    U mn = umax_of<U>(), mx = 0;
                    for_items<U, BS_NT, OVS_BS_UNR>(src, bk.beg, m, [&](U kr, u32) { const U k = K(kr); mn = min(mn, k); mx = max(mx, k); });
    #pragma unroll
                    for (int o = 16; o > 0; o >>= 1) { mn = min(mn, shfl_xor_any(mn, o)); mx = max(mx, shfl_xor_any(mx, o)); }
                    if (lane == 0) { s_mn[wid] = mn; s_mx[wid] = mx; }
                    __syncthreads();
                    mn = s_mn[0]; mx = s_mx[0];
                    for (int q = 1; q < BS_NT / 32; ++q) { mn = min(mn, s_mn[q]); mx = max(mx, s_mx[q]); }
                    lo = mn; hi = mx;
                    __syncthreads();
                }
                u32 ng = 32;
                while (ng < (u32)BS_NGMAX && ng * 3 < m) ng <<= 1;
                // digit = floor(x * ng / R) for x = (sort key - lo) in [0, R): monotone in the key
                // and spreads [lo, hi] over all ng groups (computed as a 64-bit fixed-point
                // multiply-high).  Key-value sorts of 32-bit keys use the composite (key, index) with
                // the index in its ixbits low bits (indices < 2^ixbits, so the groups spread over the
                // indices that occur); 64-bit keys use the key (equal keys share a group, ordered by
                // index).  R <= ng: digit = x, every group holds one key value (keys only: the groups
                // need no sorting, e.g. few distinct keys).
                const bool comp = KV && sizeof(U) == 4;
                const u64 xmax = comp ? ((((u64)(hi - lo)) << ixbits) | ((1ull << ixbits) - 1)) : (u64)(U)(hi - lo);
                const bool direct = xmax < (u64)ng;
                // multiplier ~ ng * 2^64 / R in double precision: any multiplier keeps the digit monotone
                // (and the clamp keeps it < ng), so rounding only perturbs the group sizes slightly
                const double mq = (double)ng * 18446744073709551616.0 / ((double)xmax + 1.0);
                const u64 mult = mq >= 18446744073709549568.0 ? 0xffffffffffffffffull : (u64)mq;
                const double mq32 = mq * (1.0 / 4294967296.0);
                const u32 mult32 = mq32 >= 4294967295.0 ? 0xffffffffu : (u32)mq32;
                auto digit = [&](U k, u32 ix) -> u32 {
                    if constexpr (!KV && sizeof(U) == 4) {
                        const u32 x = (u32)(k - lo);
                        return direct ? x : min(__umulhi(x, mult32), ng - 1);  // min: memory safety only
                    } else {
                        const u64 x = comp ? ((((u64)(k - lo)) << ixbits) | ix) : (u64)(U)(k - lo);
                        return direct ? (u32)x : min((u32)__umul64hi(x, mult), ng - 1);
                    }
                };
                const bool need_sort = KV || !direct;
                for (u32 g = threadIdx.x; g < ng; g += BS_NT) Sa.cnt[g] = 0;
                __syncthreads();
                BS_PROBE(2)
                // 1. digit histogram
                for_items<U, BS_NT, OVS_BS_UNR>(src, bk.beg, m, [&](U kr, u32 o) {
                    const u32 ix = KV ? IX(bk.beg + o) : 0u;
                    atomicAdd(&Sa.cnt[digit(K(kr), ix)], 1u);
                });
                __syncthreads();
                BS_PROBE(3)
                block_scan_small<BS_NT>(Sa.cnt, ng, red);  // cnt[g] = start of group g
                BS_PROBE(4)
                if (m > cap) {
                    // windows need every group to fit: otherwise re-split the bucket instead
                    u32 mg = 0;
                    for (u32 g = threadIdx.x; g < ng; g += BS_NT) mg = max(mg, (g + 1 < ng ? Sa.cnt[g + 1] : m) - Sa.cnt[g]);
    #pragma unroll
                    for (int o = 16; o > 0; o >>= 1) mg = max(mg, __shfl_xor_sync(0xffffffffu, mg, o));
                    if (lane == 0) red[wid] = mg;
                    __syncthreads();
                    if (threadIdx.x == 0) {
                        u32 x = 0;
                        for (int w = 0; w < BS_NT / 32; ++w) x = max(x, red[w]);
                        s_w[3] = x;
                    }
                    __syncthreads();
                    if (s_w[3] > cap) {
                        if (threadIdx.x == 0) {
                            Bucket fb = bk;
                            fb.level |= BK_FORCE;
                            if (s_sp < BS_STACK) stk[s_sp++] = fb; else st_set(status, ST_LIST_OVER);
                        }
                        __syncthreads();
                        continue;
                    }
                }
                // 2-4 per window: consecutive groups [wg0, wg1) whose items fit on chip (one window
                // covering every group when m <= cap; a bucket of up to BS_WMAX * cap items is sorted in
                // several windows, each reading the bucket again (from L2) instead of re-splitting it)
                for (u32 wg0 = 0; wg0 < ng;) {
                    if (threadIdx.x == 0) {
                        u32 lo_g = wg0 + 1, hi_g = ng;  // largest wg1 with start(wg1) - start(wg0) <= cap
                        const u32 s0 = Sa.cnt[wg0];
                        while (lo_g < hi_g) {
                            const u32 mid = (lo_g + hi_g + 1) >> 1;
                            const u32 sm = mid < ng ? Sa.cnt[mid] : m;
                            if (sm - s0 <= cap) lo_g = mid; else hi_g = mid - 1;
                        }
                        s_w[0] = lo_g;
                        s_w[1] = s0;
                        s_w[2] = (lo_g < ng ? Sa.cnt[lo_g] : m) - s0;
                    }
                    __syncthreads();
                    const u32 wg1 = s_w[0], wbase = s_w[1], wm = s_w[2];
                    __syncthreads();
    #ifdef OVS_DEBUG_CHECKS
                    if (threadIdx.x == 0 && (wm > cap || wg1 <= wg0 || wg1 > ng)) { printf("BS window wm %u cap %u wg0 %u wg1 %u ng %u m %u\n", wm, cap, wg0, wg1, ng, m); __trap(); }
    #endif
                    if (threadIdx.x == 0) { s_nbig = 0; s_nhuge = 0; s_over = 0; }
                    BucketSmem<U, KV> Sw = S;
                    Sw.k = S.k + ((((uintptr_t)(okeys + bk.beg + wbase)) / sizeof(U)) & (16 / sizeof(U) - 1));
                    {
                        BucketSmem<U, KV>& Sa = Sw;
                    // 2. scatter into shared memory by digit; afterwards cnt[g] = end of group g
                    for_items<U, BS_NT, OVS_BS_UNR>(src, bk.beg, m, [&](U kr, u32 o) {
                        const U k = K(kr);
                        u32 ix = 0, vv = 0;
                        if (KV) ix = IX(bk.beg + o);
                        const u32 dg = digit(k, ix);
                        if (dg >= wg0 && dg < wg1) {
                            if (KV) vv = vsrc[bk.beg + o];
                            const u32 pos = atomicAdd(&Sa.cnt[dg], 1u) - wbase;
    #ifdef OVS_DEBUG_CHECKS
                            if (pos >= wm) { printf("BS pos %u wm %u dg %u wg0 %u wg1 %u wbase %u m %u\n", pos, wm, dg, wg0, wg1, wbase, m); __trap(); }
    #endif
                            Sa.k[pos] = k;
                            if (KV) { Sa.i[pos] = ix; Sa.v[pos] = vv; }
                        }
                    });
                    __syncthreads();
                    BS_PROBE(5)
                    // 3. one thread per group of <= 8: Batcher network in registers; larger groups are
                    // appended (warp-aggregated) to a list for 3b
                    // (OVS_NET8_X: groups per thread per iteration, their loads and networks interleaved)
                    for (u32 g0 = wg0; need_sort && g0 < wg1; g0 += BS_NT * OVS_NET8_X) {
                        u32 gs[OVS_NET8_X], len[OVS_NET8_X];
                        E a[OVS_NET8_X][8];
        #pragma unroll
                        for (int x = 0; x < OVS_NET8_X; ++x) {
                            const u32 g = g0 + x * BS_NT + threadIdx.x;
                            gs[x] = 0; len[x] = 0;
                            if (g < wg1) { const u32 s0 = g ? Sa.cnt[g - 1] : 0u; len[x] = Sa.cnt[g] - s0; gs[x] = s0 - wbase; }
                        }
        #pragma unroll
                        for (int x = 0; x < OVS_NET8_X; ++x) {
                            const u32 lx = (len[x] > 1 && len[x] <= 8) ? len[x] : 0u;
        #pragma unroll
                            for (u32 q = 0; q < 8; ++q) a[x][q] = q < lx ? sm_get<U, KV>(Sa, gs[x] + q) : E::inf();
                        }
        #pragma unroll
                        for (int x = 0; x < OVS_NET8_X; ++x) network8(a[x]);
        #pragma unroll
                        for (int x = 0; x < OVS_NET8_X; ++x) {
                            const u32 lx = (len[x] > 1 && len[x] <= 8) ? len[x] : 0u;
        #pragma unroll
                            for (u32 q = 0; q < 8; ++q)
                                if (q < lx) sm_put<U, KV>(Sa, gs[x] + q, a[x][q]);
                        }
        #pragma unroll
                        for (int x = 0; x < OVS_NET8_X; ++x) {
                            const u32 g = g0 + x * BS_NT + threadIdx.x;
                            const u32 mb = __ballot_sync(0xffffffffu, len[x] > 8);
                            if (mb) {
                                u32 base = 0;
                                if (lane == 0) base = atomicAdd(&s_nbig, __popc(mb));
                                base = __shfl_sync(0xffffffffu, base, 0) + __popc(mb & ((1u << lane) - 1));
                                if (len[x] > 8) {
                                    if (base < BS_BIGMAX) s_big[base] = g;
                                    else atomicOr(&s_over, 1u);
                                }
                            }
                        }
                    }
                    __syncthreads();
                    BS_PROBE(6)
                    // 3b. listed groups of 9..16: one thread each (63-comparator network)
                    const u32 nlisted = min(s_nbig, (u32)BS_BIGMAX);
                    const bool rescan = s_over != 0;  // list overflow (pathological skew): scan all groups
                    const u32 nwork = rescan ? wg1 - wg0 : nlisted;
                    for (u32 q = threadIdx.x; q < nwork; q += BS_NT) {
                        const u32 g = rescan ? wg0 + q : s_big[q];
                        const u32 g_s = g ? Sa.cnt[g - 1] : 0u, len = Sa.cnt[g] - g_s, gs = g_s - wbase;
                        if (len <= 8 || len > 16) continue;
                        E a[16];
        #pragma unroll
                        for (u32 t = 0; t < 16; ++t) a[t] = t < len ? sm_get<U, KV>(Sa, gs + t) : E::inf();
                        network16(a);
        #pragma unroll
                        for (u32 t = 0; t < 16; ++t)
                            if (t < len) sm_put<U, KV>(Sa, gs + t, a[t]);
                    }
                    // 3c'. groups of 17..512: one warp each (register bitonic); over 512: the CTA
                    for (u32 q = wid; q < nwork; q += BS_NT / 32) {
                        const u32 g = rescan ? wg0 + q : s_big[q];
                        const u32 g_s = g ? Sa.cnt[g - 1] : 0u, len = Sa.cnt[g] - g_s, gs = g_s - wbase;
                        if (len <= 16) continue;
                        if (len <= 32) warp_sort_group<U, KV, 1>(Sa, gs, len);
                        else if (len <= 64) warp_sort_group<U, KV, 2>(Sa, gs, len);
                        else if (len <= 128) warp_sort_group<U, KV, 4>(Sa, gs, len);
                        else if (len <= 256) warp_sort_group<U, KV, 8>(Sa, gs, len);
                        else if (len <= 512 && BS_WARPMAX >= 512) warp_sort_group<U, KV, BS_WARPMAX / 32>(Sa, gs, len);
                        else if (lane == 0) {
                            const u32 h = atomicAdd(&s_nhuge, 1u);
                            if (h < BS_HUGEMAX) s_huge[h] = g;
                            else st_set(status, ST_LIST_OVER);
                        }
                    }
                    __syncthreads();
                    BS_PROBE(7)
                    // 3c. groups over BS_WARPMAX: in-place bitonic network in shared memory, all comparators
                    // ascending (the first step of each merge compares i with its mirror), so virtual
                    // +inf padding beyond len never moves and len need not be a power of two
                    const u32 nhuge = min(s_nhuge, (u32)BS_HUGEMAX);
                    for (u32 q = 0; q < nhuge; ++q) {
                        const u32 g = s_huge[q];
                        const u32 g_s = g ? Sa.cnt[g - 1] : 0u, len = Sa.cnt[g] - g_s, gs = g_s - wbase;
                        u32 N = 1;
                        while (N < len) N <<= 1;
                        for (u32 kk = 2; kk <= N; kk <<= 1) {
                            const u32 hk = kk >> 1;
                            for (u32 t = threadIdx.x; t < N / 2; t += BS_NT) {
                                const u32 blk = t / hk, off = t % hk;
                                const u32 x = blk * kk + off, y = blk * kk + kk - 1 - off;
                                if (y < len) smem_cex<U, KV>(Sa, gs + x, gs + y);
                            }
                            __syncthreads();
                            for (u32 j = kk >> 2; j > 0; j >>= 1) {
                                for (u32 t = threadIdx.x; t < N / 2; t += BS_NT) {
                                    const u32 x = (t / j) * 2 * j + (t % j), y = x + j;
                                    if (y < len) smem_cex<U, KV>(Sa, gs + x, gs + y);
                                }
                                __syncthreads();
                            }
                        }
                    }
                    __syncthreads();
                    BS_PROBE(8)
                    // 4. write the sorted bucket (16-byte stores where the output is aligned)
                    {
                        constexpr u32 V = 16 / sizeof(U);
                        U* out = okeys + bk.beg + wbase;
                        const u32 m = wm;  // this window's items
                        const u32 mis = (u32)(((uintptr_t)out) & 15u) / (u32)sizeof(U);
                        const u32 head = mis ? min(m, V - mis) : 0u;
                        auto R = [&](U x) -> U { return out_raw ? Codec<DT>::raw(x) : x; };
                        if (threadIdx.x < head) out[threadIdx.x] = R(Sa.k[threadIdx.x]);
                        const u32 nv = (m - head) / V;
                        uint4* o4 = (uint4*)(out + head);
                        const uint4* s4 = (const uint4*)(Sa.k + head);
                        for (u32 v = threadIdx.x; v < nv; v += BS_NT) {
                            uint4 r = s4[v];
                            U* e = (U*)&r;
        #pragma unroll
                            for (u32 q = 0; q < V; ++q) e[q] = R(e[q]);
                            o4[v] = r;
                        }
                        for (u32 o = head + nv * V + threadIdx.x; o < m; o += BS_NT) out[o] = R(Sa.k[o]);
                        if (KV) {
                            for (u32 o = threadIdx.x; o < m; o += BS_NT) ovals[bk.beg + wbase + o] = Sa.v[o];
                            if (oidx)
                                for (u32 o = threadIdx.x; o < m; o += BS_NT) oidx[bk.beg + wbase + o] = Sa.i[o];
                        }
                    }
                        __syncthreads();
                    }
                    wg0 = wg1;
                }
                __syncthreads();
            }
            BS_PROBE(9)
        }
        if (threadIdx.x == 0) {
            s_work = s_next;
            s_cur = s_nxt;
            s_next = t3;
            if (t3 < nl) s_nxt = list[t3];
        }
        __syncthreads();
    }
#ifdef OVS_BS_PROF
    if (threadIdx.x == 0) atomicAdd(&g_bsprof[15], (unsigned long long)(clock64() - bs_start_));
#endif
}

// ------------------------------------------------------------------ DRO (Algorithm 1, SqDet)
// a9: the p baseline sequences X_k (first n mod p get ceil(n/p) keys, reading Q8), as
// buckets of the caller's raw keys (sorted stably by the bucket sorter into buffer 1)
__global__ void k_dro_segments(Bucket* list, u32* nlist, u32 n, u32 p) {
    PDL_PROLOGUE();
    const u32 k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= p) return;
    const u32 q = n / p, rm = n % p;
    Bucket b;
    b.beg = k * q + min(k, rm);
    b.len = q + (k < rm ? 1u : 0u);
    b.buf = 0;
    b.level = BK_RAW | BK_LOOSE;
    b.lo = 0; b.hi = ~0ull;
    list[k] = b;
    if (k == 0) *nlist = p;
}

// a10: T_k = the s = rp regular samples of the sorted X_k: the last key of each of s evenly
// sized segments (balanced reading Q9), or the Lemma 1 proof's padded positions
// (flag).  Tag = start_k + position (the (sequence id, index) order, Q6).
// 32-bit keys are packed (ord key << 32 | tag); 64-bit keys stored with a separate tag.
template <class U>
__global__ void k_dro_sample(const U* xs, u32 n, u32 p, u32 s, u32 padded, u64* t_pack, u64* t_key, u32* t_tag) {
    PDL_PROLOGUE();
    const u64 id = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= (u64)s * p) return;
    const u32 k = (u32)(id / s), j = (u32)(id % s);
    const u32 q = n / p, rm = n % p;
    const u32 beg = k * q + min(k, rm), m = q + (k < rm ? 1u : 0u);
    u32 e;
    if (padded) {
        const u32 x = ((n + p - 1) / p + s - 1) / s;
        e = (j + 1 == s) ? m - 1 : (u32)min((u64)(j + 1) * x, (u64)m) - 1;
    } else {
        const u32 qq = m / s, rr = m % s;
        e = (j + 1) * qq + min(j + 1, rr) - 1;
    }
    const U key = xs[beg + e];
    const u32 tag = beg + e;
    if (sizeof(U) == 4) t_pack[id] = ((u64)key << 32) | tag;
    else { t_key[id] = (u64)key; t_tag[id] = tag; }
}

// a11: "Merge all T_k into a sorted sequence T of rp^2 keys" (Algorithm 1 step 2, PAPER.md:266;
// the p sorted sample sequences "are then merged or sorted into T", cost
// B p^2 r lg p).  One level of a pairwise merge: runs of L records, runs 2i and 2i+1 merged into one
// run of 2L (an odd last run is copied).  Records compare by (key, tag): 32-bit keys one u64 word
// (ord key << 32 | tag), 64-bit keys the key word with the tag as tie-break (W64).  Merge path:
// each CTA writes MS_TILE outputs of one pair; warps 0 and 1 find the tile's two diagonal splits
// by a 32-ary search (a handful of dependent L2 reads), both input ranges are staged in shared
// memory, each thread merges MS_IT consecutive outputs (odd: bank-conflict-free transposes), the tile is stored coalesced.
constexpr u32 MS_NT = 256, MS_IT = 15, MS_TILE = MS_NT * MS_IT;  // odd MS_IT: the per-thread runs of u64 records start on distinct bank pairs
template <bool W64> __device__ __forceinline__ bool ms_less(u64 ka, u32 ta, u64 kb, u32 tb) {
    return ka < kb || (W64 && ka == kb && ta < tb);
}
// number of A records among the first d outputs of merge(A, B) (A first on ties): the smallest
// a with !(B[d-1-a] < A[a]) false, i.e. pred(m) = !(B[d-1-m] < A[m]) holds exactly for m < a
template <bool W64>
__device__ __forceinline__ u32 ms_split_warp(const u64* A, const u32* At, u32 la, const u64* B, const u32* Bt,
                                             u32 lb, u32 d, u32 lane) {
    u32 lo = d > lb ? d - lb : 0, hi = min(d, la);
    while (hi > lo) {
        const u32 step = (hi - lo + 31) / 32;
        const u32 m = lo + lane * step;
        bool pr = false;
        if (m < hi) pr = !ms_less<W64>(B[d - 1 - m], W64 ? Bt[d - 1 - m] : 0u, A[m], W64 ? At[m] : 0u);
        const u32 cnt = __popc(__ballot_sync(~0u, pr));
        if (cnt == 0) hi = lo;
        else {
            lo = lo + (cnt - 1) * step + 1;
            hi = min(hi, lo - 1 + step);
        }
    }
    return lo;
}
template <bool W64>
__global__ void __launch_bounds__(MS_NT) k_sample_merge(const u64* __restrict__ ik, const u32* __restrict__ it,
                                                        u64* __restrict__ ok, u32* __restrict__ ot, u32 N, u32 L,
                                                        u32 tpp) {
    PDL_PROLOGUE();
    __shared__ u64 sk[MS_TILE];
    __shared__ u32 stg[W64 ? MS_TILE : 1];
    __shared__ u32 spl[2];
    const u32 pair = blockIdx.x / tpp, tile = blockIdx.x % tpp;
    const u64 base = (u64)pair * 2 * L;
    if (base >= N) return;
    const u32 la = (u32)min((u64)L, N - base);
    const u32 lb = (u32)min((u64)L, N - base - la);
    const u32 d0 = tile * MS_TILE;
    if (d0 >= la + lb) return;
    const u32 d1 = min(d0 + MS_TILE, la + lb);
    const u64* A = ik + base;
    const u64* B = A + la;
    const u32* At = W64 ? it + base : nullptr;
    const u32* Bt = W64 ? At + la : nullptr;
    const u32 tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (warp < 2) {
        const u32 a = ms_split_warp<W64>(A, At, la, B, Bt, lb, warp ? d1 : d0, lane);
        if (lane == 0) spl[warp] = a;
    }
    __syncthreads();
    const u32 a0 = spl[0], a1 = spl[1], b0 = d0 - a0, b1 = d1 - a1;
    const u32 na = a1 - a0, nb = b1 - b0, nt = na + nb;
    {  // all MS_IT loads of a thread in flight before the shared stores
        u64 v[MS_IT];
        u32 vt[MS_IT];
#pragma unroll
        for (u32 q = 0; q < MS_IT; ++q) {
            const u32 i = tid + q * MS_NT;
            const bool fa = i < na;
            const u32 g = fa ? a0 + i : b0 + (i - na);
            if (i < nt) {
                v[q] = *((fa ? A : B) + g);
                if (W64) vt[q] = *((fa ? At : Bt) + g);
            }
        }
#pragma unroll
        for (u32 q = 0; q < MS_IT; ++q) {
            const u32 i = tid + q * MS_NT;
            if (i < nt) {
                sk[i] = v[q];
                if (W64) stg[i] = vt[q];
            }
        }
    }
    __syncthreads();
    // this thread's outputs [dl, dl + MS_IT) of the tile: split by a binary search in shared memory
    const u32 dl = min(tid * MS_IT, nt);
    u32 lo = dl > nb ? dl - nb : 0, hi = min(dl, na);
    while (lo < hi) {
        const u32 m = (lo + hi) >> 1;
        if (!ms_less<W64>(sk[na + dl - 1 - m], W64 ? stg[na + dl - 1 - m] : 0u, sk[m], W64 ? stg[m] : 0u)) lo = m + 1;
        else hi = m;
    }
    u32 i = lo, j = dl - lo;
    u64 rk[MS_IT];
    u32 rt[MS_IT];
    // the two heads stay in registers: one shared read per output (the side just consumed)
    u64 ka = i < na ? sk[i] : 0ull, kb = j < nb ? sk[na + j] : 0ull;
    u32 ta_ = (W64 && i < na) ? stg[i] : 0u, tb_ = (W64 && j < nb) ? stg[na + j] : 0u;
#pragma unroll
    for (u32 q = 0; q < MS_IT; ++q) {
        const bool ta = j >= nb || (i < na && !ms_less<W64>(kb, tb_, ka, ta_));
        rk[q] = ta ? ka : kb;
        rt[q] = ta ? ta_ : tb_;
        if (ta) {
            ++i;
            ka = i < na ? sk[i] : 0ull;
            if (W64) ta_ = i < na ? stg[i] : 0u;
        } else {
            ++j;
            kb = j < nb ? sk[na + j] : 0ull;
            if (W64) tb_ = j < nb ? stg[na + j] : 0u;
        }
    }
    __syncthreads();
#pragma unroll
    for (u32 q = 0; q < MS_IT; ++q) {
        const u32 o = tid * MS_IT + q;
        if (o < nt) {
            sk[o] = rk[q];
            if (W64) stg[o] = rt[q];
        }
    }
    __syncthreads();
    u64* O = ok + base + d0;
    u32* Ot = W64 ? ot + base + d0 : nullptr;
    for (u32 q = tid; q < nt; q += MS_NT) {
        O[q] = sk[q];
        if (W64) Ot[q] = stg[q];
    }
}

// a13: bound[k][j+1] = #{t : (X_k[t], start_k + t) <=lex S[j]} by binary search of splitter j
// into the sorted X_k; count matrix cnt[k][j] = bound[k][j+1]-bound[k][j]
// (P buckets: P - 1 splitters; P = p for the contract split, p*f for the fine split of f2)
template <class U>
__global__ void k_dro_bounds(const U* xs, u32 n, u32 p, u32 P, const U* sk, const u32* st, u32* bound, u32 tag0 = 0) {
    PDL_PROLOGUE();
    const u64 id = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= (u64)p * (P + 1)) return;
    const u32 k = (u32)(id / (P + 1)), j = (u32)(id % (P + 1));
    const u32 q = n / p, rm = n % p;
    const u32 beg = k * q + min(k, rm), m = q + (k < rm ? 1u : 0u);
    u32 r;
    if (j == 0) r = 0;
    else if (j == P) r = m;
    else {
        const U key = sk[j - 1];
        const u32 tag = st[j - 1];
        // upper bound: first t with (X_k[t], beg + t) >lex (key, tag)
        u32 lo = 0, cnt = m;
        while (cnt > 0) {
            const u32 half = cnt >> 1, mid = lo + half;
            const U x = xs[beg + mid];
            const bool le = x < key || (x == key && tag0 + beg + mid <= tag);  // tags: global positions
            if (le) { lo = mid + 1; cnt -= half + 1; } else cnt = half;
        }
        r = lo;
    }
    bound[id] = r;
}

__global__ void k_dro_counts(const u32* bound, u32 p, u32 P, u32* cnt) {
    PDL_PROLOGUE();
    const u64 id = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= (u64)p * P) return;
    const u32 k = (u32)(id / P), j = (u32)(id % P);
    cnt[id] = bound[(u64)k * (P + 1) + j + 1] - bound[(u64)k * (P + 1) + j];
}

// the single "segment" of the DRO split: p chunks (the sequences) x p buckets; key bounds of
// the whole input from the sorted sequences' first and last keys
template <class U>
__global__ void k_dro_seg(const U* xs, u32 n, u32 p, u32 P, const U* sk, u32 L, Seg* seg, u32* nseg) {
    PDL_PROLOGUE();
    __shared__ U smn[32], smx[32];
    const u32 q = n / p, rm = n % p;
    U mn = umax_of<U>(), mx = 0;
    for (u32 k = threadIdx.x; k < p; k += blockDim.x) {
        const u32 beg = k * q + min(k, rm), m = q + (k < rm ? 1u : 0u);
        mn = min(mn, xs[beg]);
        mx = max(mx, xs[beg + m - 1]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) { mn = min(mn, shfl_xor_any(mn, o)); mx = max(mx, shfl_xor_any(mx, o)); }
    if ((threadIdx.x & 31) == 0) { smn[threadIdx.x >> 5] = mn; smx[threadIdx.x >> 5] = mx; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (u32 w = 1; w < blockDim.x / 32; ++w) { mn = min(mn, smn[w]); mx = max(mx, smx[w]); }
        mn = min(mn, smn[0]); mx = max(mx, smx[0]);
        Seg g;
        g.lo = (u64)mn; g.hi = (u64)mx; g.base = 0;
        g.beg = 0; g.len = n; g.P = P; g.shift = 0; g.L = L; g.chunk0 = 0; g.nchunk = p;
        g.src = 1;  // buckets land in buffer 0
        g.loose = 0; g.pad = 0;
        *seg = g;
        nseg[0] = 1;
    }
}

// a14 (gather): run X_{k,j} (sorted X_k[bound[k][j] .. bound[k][j+1])) goes to bucket j at
// offset start_j + sum_{k'<k} cnt[k'][j] (column-scanned cnt); one warp per run
template <class U, bool KV>
__global__ void k_dro_gather(Bufs<U> B, u32 n, u32 p, const u32* bound, const u32* off, const u32* bstart) {
    PDL_PROLOGUE();
    const u64 w = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const u32 lane = threadIdx.x & 31;
    if (w >= (u64)p * p) return;
    const u32 k = (u32)(w / p), j = (u32)(w % p);
    const u32 q = n / p, rm = n % p;
    const u32 beg = k * q + min(k, rm);
    const u32 a = bound[(u64)k * (p + 1) + j], b = bound[(u64)k * (p + 1) + j + 1];
    const u32 d = bstart[j] + off[w];
    for (u32 t = a + lane; t < b; t += 32) {
        B.k[0][d + t - a] = B.k[1][beg + t];
        if (KV) { B.v[0][d + t - a] = B.v[1][beg + t]; B.i[0][d + t - a] = B.i[1][beg + t]; }
    }
}

// ------------------------------------------------------------------ f2: a14 as a p-way merge
// (Alg. 1 step 5: Y_j = the stable merge of the sorted runs X_{0,j} ..
// X_{p-1,j}, ties to the lower k.)  The DRO split is refined with P = p*f fine splitters
// taken from the same sorted regular sample (every rp/f-th record; every f-th one is a contract
// splitter, so contract bucket q is fine buckets qf .. qf+f-1).  A fine bucket's p runs are
// gathered in k order into shared memory straight from the sorted sequences (no copy pass) and
// merged by a pairwise merge tree (log2 p levels; every thread merges E outputs after a
// merge-path search on its diagonal, ties taken from the left run), then written once.  Fine
// buckets over the on-chip capacity are listed and take the gather + bucket-sort route.
constexpr int MG_NT = 512, MG_E = 8;
template <class U, bool KV> __host__ __device__ constexpr size_t merge_item_bytes() { return sizeof(U) + (KV ? 4 : 0); }
template <class U, bool KV> __host__ __device__ constexpr size_t merge_smem_bytes(u32 mcap, u32 p) {
    return 2 * a16(merge_item_bytes<U, KV>() * (size_t)mcap) + a16(8 * ((size_t)p + 1)) + 64;
}
// fine bucket j' of P: runs k = 0..p-1 are X_k[bound[k][j'] .. bound[k][j'+1]) of the sorted
// sequences (ordered keys in buffer 1), run offsets inside the bucket off[k*P + j'] (column scan),
// bucket start tot[j'] (segment scan); output = buffer 0 (raw codec), values too
template <int DT, bool KV>
__global__ void __launch_bounds__(MG_NT, 1) k_dro_merge(Bufs<typename Codec<DT>::U> B, u32 n, u32 p, u32 P,
                                                          const u32* bound, const u32* off, const u32* tot, u32 mcap) {
    PDL_PROLOGUE();
    typedef typename Codec<DT>::U U;
    extern __shared__ __align__(16) char smem[];
    U* ka = (U*)smem;
    U* kb2 = (U*)(smem + a16(sizeof(U) * (size_t)mcap));
    char* sp = smem + 2 * a16(sizeof(U) * (size_t)mcap);
    u32* va = nullptr; u32* vb = nullptr;
    if (KV) { va = (u32*)sp; sp += a16(4 * (size_t)mcap); vb = (u32*)sp; sp += a16(4 * (size_t)mcap); }
    u32* R = (u32*)sp;  // run starts inside the bucket, R[p] = bucket length
    u32* S = R + p + 1;  // run k's first item in the sorted sequences (buffer 1)
    const u32 q = n / p, rm = n % p;
    for (u32 j = blockIdx.x; j < P; j += gridDim.x) {
        const u32 bs = tot[j], len = tot[j + 1] - bs;
        if (len == 0 || len > mcap) continue;  // empty, or listed for the bucket sorter
        for (u32 k = threadIdx.x; k < p; k += MG_NT) {
            R[k] = off[(size_t)k * P + j];
            S[k] = k * q + min(k, rm) + bound[(size_t)k * (P + 1) + j];
        }
        if (threadIdx.x == 0) R[p] = len;
        __syncthreads();
        // gather the runs (k order) straight from the sorted sequences: item e of the bucket is
        // in run k = the last run starting at or before e (empty runs share a start; independent
        // loads, many in flight)
        for (u32 e = threadIdx.x; e < len; e += MG_NT) {
            u32 lo = 0, cnt = p;
            while (cnt > 1) {
                const u32 half = cnt >> 1;
                if (R[lo + half] <= e) { lo += half; cnt -= half; } else cnt = half;
            }
            const u32 src = S[lo] + (e - R[lo]);
            ka[e] = B.k[1][src];
            if (KV) va[e] = B.v[1][src];
        }
        __syncthreads();
        U* sk = ka; U* dk = kb2;
        u32* sv = va; u32* dv = vb;
        for (u32 w = 1; w < p; w <<= 1) {
            const u32 np = (p + 2 * w - 1) / (2 * w);  // pairs of sequences of w runs
            for (u32 o0 = threadIdx.x * MG_E; o0 < len; o0 += MG_NT * MG_E) {
                u32 o = o0;
                const u32 oe = min(o0 + MG_E, len);
                // pair holding output o: the last pair whose start R[2iw] <= o
                u32 lo = 0, hi = np - 1;
                while (lo < hi) {
                    const u32 mid = (lo + hi + 1) >> 1;
                    if (R[min(2 * mid * w, p)] <= o) lo = mid; else hi = mid - 1;
                }
                u32 pi = lo;
                while (o < oe) {
                    const u32 a0 = R[min(2 * pi * w, p)], a1 = R[min(2 * pi * w + w, p)], b1 = R[min(2 * pi * w + 2 * w, p)];
                    const u32 la = a1 - a0, lb = b1 - a1, d = o - a0;
                    // merge path: i outputs from the left run among the first d (ties: left first)
                    u32 l2 = d > lb ? d - lb : 0u, h2 = min(d, la);
                    while (l2 < h2) {
                        const u32 mid = (l2 + h2) >> 1;
                        if (sk[a0 + mid] <= sk[a1 + d - 1 - mid]) l2 = mid + 1; else h2 = mid;
                    }
                    u32 i = l2, jj = d - l2;
                    const u32 stop = min(oe, b1);
                    for (; o < stop; ++o) {
                        const bool left = i < la && (jj >= lb || sk[a0 + i] <= sk[a1 + jj]);
                        const u32 src = left ? a0 + i : a1 + jj;
                        dk[o] = sk[src];
                        if (KV) dv[o] = sv[src];
                        if (left) ++i; else ++jj;
                    }
                    ++pi;
                }
            }
            __syncthreads();
            U* tk = sk; sk = dk; dk = tk;
            u32* tv = sv; sv = dv; dv = tv;
        }
        // write the merged bucket (raw codec)
        U* out = B.k[0] + bs;
        for (u32 o = threadIdx.x; o < len; o += MG_NT) {
            out[o] = Codec<DT>::raw(sk[o]);
            if (KV) B.v[0][bs + o] = sv[o];
        }
        __syncthreads();
    }
}

// fine buckets over the merge capacity (the segment scan's big list): gather their runs into
// buffer 0 at the bucket position (keys, values, original indices) for the bucket sorter; the
// fine bucket index is recovered from the bucket start (starts strictly increase)
template <class U, bool KV>
__global__ void k_dro_gather_big(Bufs<U> B, u32 n, u32 p, u32 P, const u32* bound, const u32* off, const u32* tot,
                                 const Bucket* big, const u32* nbig) {
    PDL_PROLOGUE();
    const u32 lane = threadIdx.x & 31;
    const u32 nb = *nbig;
    for (u64 w = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < (u64)nb * p; w += ((u64)gridDim.x * blockDim.x) >> 5) {
    const Bucket bk = big[w / p];
    const u32 k = (u32)(w % p);
    u32 lo = 0, hi = P;  // last j with tot[j] <= beg
    while (lo < hi) {
        const u32 mid = (lo + hi + 1) >> 1;
        if (tot[mid] <= bk.beg) lo = mid; else hi = mid - 1;
    }
    const u32 j = lo;
    const u32 q = n / p, rm = n % p;
    const u32 beg = k * q + min(k, rm);
    const u32 a = bound[(size_t)k * (P + 1) + j], b = bound[(size_t)k * (P + 1) + j + 1];
    const u32 d = bk.beg + off[(size_t)k * P + j];
    for (u32 t = a + lane; t < b; t += 32) {
        B.k[0][d + t - a] = B.k[1][beg + t];
        if (KV) { B.v[0][d + t - a] = B.v[1][beg + t]; B.i[0][d + t - a] = B.i[1][beg + t]; }
    }
    }
}

// ------------------------------------------------------------------ multi-GPU building blocks
// (SURVEY.md §8(e)).  Every rank computes the same global ROS index set over n_global keys and
// contributes the records of its own shard (k_ros_take<DT, true>); after the all-reduce SUM
// the records are unpacked into the sample sort's arrays.
__global__ void k_dist_unpack(const u64* rec, u32 m, u32 words, u64* t_pack, u64* t_key, u32* t_tag) {
    PDL_PROLOGUE();
    const u32 t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m) return;
    if (words == 1) t_pack[t] = rec[t];
    else { t_key[t] = rec[2 * (u64)t]; t_tag[t] = (u32)rec[2 * (u64)t + 1]; }
}

// this rank's bucket counts -> row `rank` of the count matrix C (world x p u32) in every rank's
// window (the count all-gather as NVLink stores)
__global__ void k_put_counts(const u64* counts, u32 p, u32 rank, PeerOut po) {
    PDL_PROLOGUE();
    const u32 t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= p * po.world) return;
    const u32 d = t / p, b = t % p;
    ((u32*)(po.peers[d] + po.off))[(size_t)rank * p + b] = (u32)counts[b];
    __threadfence_system();
}

// ---- DRO across GPUs (DRO steps; the paper's McDet split): rank g
// holds the p/G whole sequences [g p/G, (g+1) p/G) of the global baseline split (equal shards, p | n).
// a10 on the local sorted sequences: record (key, global tag = tag0 + local position) of sample j of
// local sequence k goes to slot slot0 + k s + j of every rank's window (s = r p regular samples,
// balanced or padded positions of the global Alg. 1)
template <class U>
__global__ void k_dro_sample_dist(const U* xs, u32 n, u32 p, u32 s, u32 padded, u32 xpad, u32 tag0, u32 slot0,
                                  PeerOut po) {
    PDL_PROLOGUE();
    const u64 id = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= (u64)s * p) return;
    const u32 k = (u32)(id / s), j = (u32)(id % s);
    const u32 q = n / p, rm = n % p;
    const u32 beg = k * q + min(k, rm), m = q + (k < rm ? 1u : 0u);
    u32 e;
    if (padded) e = (j + 1 == s) ? m - 1 : (u32)min((u64)(j + 1) * xpad, (u64)m) - 1;
    else {
        const u32 qq = m / s, rr = m % s;
        e = (j + 1) * qq + min(j + 1, rr) - 1;
    }
    put_rec<sizeof(U) == 8>(po, slot0 + (u32)id, (u64)xs[beg + e], (u64)(tag0 + beg + e));
}

// this rank's bucket totals (u32) -> row `rank` of every window's count matrix
__global__ void k_put_counts32(const u32* tot, u32 p, u32 rank, PeerOut po) {
    PDL_PROLOGUE();
    const u32 t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= p * po.world) return;
    const u32 d = t / p, b = t % p;
    ((u32*)(po.peers[d] + po.off))[(size_t)rank * p + b] = tot[b];
    __threadfence_system();
}

// a14's exchange: run (k, j) = X_k[bound[k][j] .. bound[k][j+1]) of local sorted sequence k goes to
// bucket j's owner window at dst_off[j] + off[k][j] (the column prefix over the local sequences, so
// runs arrive in global sequence order); keys ordered, values and original indices with them
template <class U, bool KV>
__global__ void k_dro_send(Bufs<U> B, u32 n, u32 p, u32 P, const u32* bound, const u32* off, const u32* dst_off,
                           PeerOut pk, size_t off_v, size_t off_i) {
    PDL_PROLOGUE();
    const u32 lane = threadIdx.x & 31;
    const u32 q = n / p, rm = n % p;
    for (u64 w = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < (u64)p * P; w += ((u64)gridDim.x * blockDim.x) >> 5) {
        const u32 k = (u32)(w / P), j = (u32)(w % P);
        const u32 a = bound[(size_t)k * (P + 1) + j], b = bound[(size_t)k * (P + 1) + j + 1];
        if (a == b) continue;
        const u32 beg = k * q + min(k, rm);
        const u32 d = dst_off[j] + off[(size_t)k * P + j];
        char* const win = pk.peers[((u64)j * pk.world) / P];
        U* dk = (U*)(win + pk.off);
        for (u32 t = a + lane; t < b; t += 32) {
            dk[d + t - a] = B.k[1][beg + t];
            if (KV) {
                ((u32*)(win + off_v))[d + t - a] = B.v[1][beg + t];
                ((u32*)(win + off_i))[d + t - a] = B.i[1][beg + t];
            }
        }
    }
    __threadfence_system();
}

__global__ void k_add_u32(u32* a, u32 n, u32 v) {
    PDL_PROLOGUE();
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] += v;
}

// the received (owned) buckets as a work list: desc[3j..3j+2] = (begin in the receive region,
// length, global bucket id) from the host plan; bounds from the splitters around the bucket
template <class U>
__global__ void k_dist_list(const u32* desc, u32 nb, const U* sk, u32 p, Bucket* list, u32* nlist, u32 buf) {
    PDL_PROLOGUE();
    const u32 j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j == 0) { nlist[0] = nb; nlist[1] = 0; }
    if (j >= nb) return;
    Bucket bk;
    bk.beg = desc[3 * j]; bk.len = desc[3 * j + 1]; bk.buf = buf;
    const u32 g = desc[3 * j + 2];
    const bool lo_open = g == 0, hi_open = g + 1 == p;
    bk.level = (lo_open || hi_open) ? BK_LOOSE : 0u;
    bk.lo = lo_open ? 0 : (u64)sk[g - 1];
    bk.hi = hi_open ? (u64)umax_of<U>() : (u64)sk[g];
    list[j] = bk;
}

__global__ void k_fill_u32(u32* p, u32 v, u32 n) {
    PDL_PROLOGUE();
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}


__global__ void k_iota(u32* p, u32 n) {
    PDL_PROLOGUE();
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = i;
}

// internal sorts of an array that fits the bucket sorter: one bucket with loose bounds
template <class U>
__global__ void k_push_bucket(Bucket* list, u32* nlist, u32 len) {
    PDL_PROLOGUE();
    Bucket b;
    b.beg = 0; b.len = len; b.buf = 0; b.level = BK_LOOSE;
    b.lo = 0; b.hi = (u64)umax_of<U>();
    list[0] = b;
    *nlist = 1;
}

// ------------------------------------------------------------------ f3: 32-byte string keys
// The paper's own workload: keys are 32-byte strings in memcmp order.  A
// record is 4 words; word w as a big-endian number (bswap64) makes memcmp order the
// lexicographic order of (w0, w1, w2, w3).  The pipeline is ROS's: the sample index set and its
// sort run on (prefix w0, index) records (equal-prefix runs of the sorted sample re-ordered by the
// full key, k_s32_fix*), the classifier uses the prefix table and compares the full key on a prefix
// tie (classify_s32), the scatter moves whole 32-byte records (one sector each), and every bucket is
// sorted on chip by the full key (k_bucket_sort_s32).
struct K32 { u64 w[4]; };  // big-endian words
__device__ __forceinline__ K32 load_k32(const u64* recs, u64 i) {
    const uint4* r = (const uint4*)(recs + 4 * i);
    const uint4 a = r[0], b = r[1];
    K32 k;
    k.w[0] = bswap64(((u64)a.y << 32) | a.x);
    k.w[1] = bswap64(((u64)a.w << 32) | a.z);
    k.w[2] = bswap64(((u64)b.y << 32) | b.x);
    k.w[3] = bswap64(((u64)b.w << 32) | b.z);
    return k;
}
// (a, ta) <lex (b, tb) by the full key, then the tag (reading Q5)
__device__ __forceinline__ bool k32_less(const K32& a, u32 ta, const K32& b, u32 tb) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
        if (a.w[q] != b.w[q]) return a.w[q] < b.w[q];
    return ta < tb;
}

// equal-prefix runs of the sorted sample records (key word = prefix, tags = original indices):
// runs of <= 32 re-ordered by (full key, tag) by one thread; longer runs listed for k_s32_fix_long
__global__ void k_s32_fix(const u64* pk, u32* tags, u32 m, const u64* recs, u32* list, u32* nlist, u32 cap,
                          u32* status) {
    PDL_PROLOGUE();
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i + 1 >= m) return;
    if (pk[i] != pk[i + 1] || (i > 0 && pk[i - 1] == pk[i])) return;  // not the start of a run
    u32 L = 2;
    while (i + L < m && pk[i + L] == pk[i]) ++L;
    if (L > 32) {
        const u32 q = atomicAdd(nlist, 1u);
        if (q < cap) { list[2 * q] = i; list[2 * q + 1] = L; } else st_set(status, ST_LIST_OVER);
        return;
    }
    for (u32 a = 1; a < L; ++a) {  // insertion sort of the tags by (full key, tag)
        const u32 t = tags[i + a];
        const K32 kt = load_k32(recs, t);
        u32 b = a;
        while (b > 0) {
            const u32 u = tags[i + b - 1];
            if (!k32_less(kt, t, load_k32(recs, u), u)) break;
            tags[i + b] = u;
            --b;
        }
        tags[i + b] = t;
    }
}
// long runs: one CTA each, bitonic sort of the run's tags by (full key, tag) in place in global
// memory (all comparators ascending, so the length need not be a power of two)
__global__ void __launch_bounds__(1024) k_s32_fix_long(u32* tags, const u64* recs, const u32* list, const u32* nlist) {
    PDL_PROLOGUE();
    const u32 nl = *nlist;
    for (u32 r = blockIdx.x; r < nl; r += gridDim.x) {
        u32* t = tags + list[2 * r];
        const u32 len = list[2 * r + 1];
        u32 N = 1;
        while (N < len) N <<= 1;
        auto cx = [&](u32 x, u32 y) {
            const u32 a = t[x], b = t[y];
            if (k32_less(load_k32(recs, b), b, load_k32(recs, a), a)) { t[x] = b; t[y] = a; }
        };
        for (u32 kk = 2; kk <= N; kk <<= 1) {
            const u32 hk = kk >> 1;
            for (u32 q = threadIdx.x; q < N / 2; q += blockDim.x) {
                const u32 blk = q / hk, off = q % hk;
                const u32 x = blk * kk + off, y = blk * kk + kk - 1 - off;
                if (y < len) cx(x, y);
            }
            __threadfence_block();
            __syncthreads();
            for (u32 j = kk >> 2; j > 0; j >>= 1) {
                for (u32 q = threadIdx.x; q < N / 2; q += blockDim.x) {
                    const u32 x = (q / j) * 2 * j + (q % j), y = x + j;
                    if (y < len) cx(x, y);
                }
                __threadfence_block();
                __syncthreads();
            }
        }
    }
}

// full keys of the splitters (for the classifier's prefix ties and the report): rows of 4 words
// (big-endian) + the raw 32-byte records
__global__ void k_s32_splitters(const u32* st, u32 nsp, const u64* recs, u64* sfull, u64* sraw) {
    PDL_PROLOGUE();
    const u32 q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nsp) return;
    const K32 k = load_k32(recs, st[q]);
#pragma unroll
    for (int w = 0; w < 4; ++w) sfull[4 * (size_t)q + w] = k.w[w];
    if (sraw)
#pragma unroll
        for (int w = 0; w < 4; ++w) sraw[4 * (size_t)q + w] = recs[4 * (size_t)st[q] + w];
}

// bucket(key, tag) = #{q : S[q] <lex (key, tag)}: the prefix table narrows to the splitters with
// an equal prefix (or none), the full key and the tag decide among those
__device__ __forceinline__ u32 classify_s32(const ClsView<u64>& c, const u64* sfull, const K32& k, u32 tag) {
    if (c.P <= 1) return 0;
    const u64 pre = k.w[0];
    u32 lo, cnt;
    if (pre < c.base) return 0;
    const u64 x = pre - c.base;
    const u64 d = x >> c.shift;
    if (d >= (u64)c.L) return c.P - 1;
    const u32 e = c.lut[(u32)d];
    lo = e & 0x1fffu;
    cnt = (e >> 13) & 7u;
    if (cnt == 7) cnt = (c.lut[(u32)d + 1] & 0x1fffu) - lo;
    while (cnt > 0) {
        const u32 half = cnt >> 1, mid = lo + half;
        const u64 s = c.sk[mid];
        bool less;
        if (s != pre) less = s < pre;
        else {
            K32 sk;
#pragma unroll
            for (int w = 0; w < 4; ++w) sk.w[w] = sfull[4 * (size_t)mid + w];
            less = k32_less(sk, c.st[mid], k, tag);
        }
        if (less) { lo = mid + 1; cnt -= half + 1; } else { cnt = half; }
    }
    return lo;
}

// a5+a6 for strings: per chunk histogram rows and every record's bucket id (u16)
constexpr int S32_NT = 512;
__global__ void __launch_bounds__(S32_NT) k_hist_s32(const u64* recs, const Chunk* chunks, const u32* nchunks,
                                                     Seg* segs, const u64* sk_pool, const u32* st_pool,
                                                     const u32* lut_pool, u32 PS, u32 LS, u32* hist, const u64* sfull,
                                                     u16* bid) {
    PDL_PROLOGUE();
    extern __shared__ __align__(16) char smem[];
    const u32 nc = *nchunks;
    u32 loaded = 0xffffffffu;
    for (u32 c = blockIdx.x; c < nc; c += gridDim.x) {
        const Chunk ch = chunks[c];
        const Seg sg = segs[ch.seg];
        ClsView<u64> cls = load_cls<u64>(smem, sg, ch.seg, sk_pool, st_pool, lut_pool, PS, LS, loaded != ch.seg);
        loaded = ch.seg;
        u32* h = (u32*)(smem + cls_smem_bytes<u64>(PS, LS));
        for (u32 i = threadIdx.x; i < sg.P; i += S32_NT) h[i] = 0;
        __syncthreads();
        for (u32 i0 = ch.beg; i0 < ch.end; i0 += 4 * S32_NT) {
            K32 k[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const u32 i = i0 + u * S32_NT + threadIdx.x;
                if (i < ch.end) k[u] = load_k32(recs, i);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const u32 i = i0 + u * S32_NT + threadIdx.x;
                if (i < ch.end) {
                    const u32 b = classify_s32(cls, sfull, k[u], i);
                    atomicAdd(&h[b], 1u);
                    bid[i] = (u16)b;
                }
            }
        }
        __syncthreads();
        u32* row = hist + (size_t)c * PS;
        for (u32 b = threadIdx.x; b < sg.P; b += S32_NT) row[b] = h[b];
        __syncthreads();
    }
}

// a7 for strings: every record (one 32-byte sector) stored at its bucket cursor
__global__ void __launch_bounds__(S32_NT) k_scatter_s32(const u64* src, u64* dst, const Chunk* chunks,
                                                        const u32* nchunks, const Seg* segs, u32 PS, const u32* hist,
                                                        const u32* tot_pool, const u16* bid) {
    PDL_PROLOGUE();
    extern __shared__ __align__(16) char smem[];
    u32* cur = (u32*)smem;
    const u32 nc = *nchunks;
    for (u32 c = blockIdx.x; c < nc; c += gridDim.x) {
        const Chunk ch = chunks[c];
        const Seg sg = segs[ch.seg];
        const u32* hrow = hist + (size_t)c * PS;
        const u32* bst = tot_pool + (size_t)ch.seg * (PS + 1);
        for (u32 b = threadIdx.x; b < sg.P; b += S32_NT) cur[b] = sg.beg + bst[b] + hrow[b];
        __syncthreads();
        for (u32 i0 = ch.beg; i0 < ch.end; i0 += 4 * S32_NT) {
            uint4 r[4][2];
            u32 b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const u32 i = i0 + u * S32_NT + threadIdx.x;
                if (i < ch.end) {
                    const uint4* s4 = (const uint4*)(src + 4 * (size_t)i);
                    r[u][0] = s4[0]; r[u][1] = s4[1];
                    b[u] = bid[i];
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const u32 i = i0 + u * S32_NT + threadIdx.x;
                if (i < ch.end) {
                    const u32 pos = atomicAdd(&cur[b[u]], 1u);
                    uint4* d4 = (uint4*)(dst + 4 * (size_t)pos);
                    d4[0] = r[u][0]; d4[1] = r[u][1];
                }
            }
        }
        __syncthreads();
    }
}

// a8 for strings: persistent CTAs over the bucket list; a bucket of <= cap records is loaded into
// shared memory as big-endian words and its index array sorted by the full key (bitonic network,
// all comparators ascending: any length); larger buckets (outliers of the refined partition) are
// sorted through an index array in global memory (idx) the same way, slower.  Output: buffer 0.
constexpr int S32_BS_NT = 512;
__global__ void __launch_bounds__(S32_BS_NT, 1) k_bucket_sort_s32(const Bucket* list, const u32* nlist, u32* ticket,
                                                                  const u64* src, u64* dst, u32 cap, u32* gidx) {
    PDL_PROLOGUE();
    extern __shared__ __align__(16) char smem[];
    u64* kw = (u64*)smem;                         // cap x 4 words (big-endian)
    u32* ix = (u32*)(smem + 32 * (size_t)cap);    // cap indices
    __shared__ u32 s_work;
    const u32 nl = *nlist;
    for (;;) {
        if (threadIdx.x == 0) s_work = atomicAdd(ticket, 1u);
        __syncthreads();
        const u32 w = s_work;
        __syncthreads();
        if (w >= nl) break;
        const Bucket bk = list[w];
        const u32 m = bk.len;
        const u64* s = src + 4 * (size_t)bk.beg;
        u64* d = dst + 4 * (size_t)bk.beg;
        const bool on_chip = m <= cap;
        u32* id = on_chip ? ix : gidx + bk.beg;
        auto key = [&](u32 r, int q) -> u64 { return on_chip ? kw[4 * (size_t)r + q] : bswap64(s[4 * (size_t)r + q]); };
        for (u32 r = threadIdx.x; r < m; r += S32_BS_NT) {
            if (on_chip) {
                const uint4* s4 = (const uint4*)(s + 4 * (size_t)r);
                const uint4 a = s4[0], b = s4[1];
                kw[4 * (size_t)r + 0] = bswap64(((u64)a.y << 32) | a.x);
                kw[4 * (size_t)r + 1] = bswap64(((u64)a.w << 32) | a.z);
                kw[4 * (size_t)r + 2] = bswap64(((u64)b.y << 32) | b.x);
                kw[4 * (size_t)r + 3] = bswap64(((u64)b.w << 32) | b.z);
            }
            id[r] = r;
        }
        __threadfence_block();
        __syncthreads();
        auto less = [&](u32 a, u32 b) -> bool {  // record a < record b (ties: keep either)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const u64 x = key(a, q), y = key(b, q);
                if (x != y) return x < y;
            }
            return false;
        };
        u32 N = 1;
        while (N < m) N <<= 1;
        for (u32 kk = 2; kk <= N; kk <<= 1) {
            const u32 hk = kk >> 1;
            for (u32 t = threadIdx.x; t < N / 2; t += S32_BS_NT) {
                const u32 blk = t / hk, off = t % hk;
                const u32 x = blk * kk + off, y = blk * kk + kk - 1 - off;
                if (y < m) {
                    const u32 a = id[x], b = id[y];
                    if (less(b, a)) { id[x] = b; id[y] = a; }
                }
            }
            __threadfence_block();
            __syncthreads();
            for (u32 j = kk >> 2; j > 0; j >>= 1) {
                for (u32 t = threadIdx.x; t < N / 2; t += S32_BS_NT) {
                    const u32 x = (t / j) * 2 * j + (t % j), y = x + j;
                    if (y < m) {
                        const u32 a = id[x], b = id[y];
                        if (less(b, a)) { id[x] = b; id[y] = a; }
                    }
                }
                __threadfence_block();
                __syncthreads();
            }
        }
        // write out in sorted order (the raw records)
        for (u32 r = threadIdx.x; r < m; r += S32_BS_NT) {
            const uint4* s4 = (const uint4*)(s + 4 * (size_t)id[r]);
            uint4* d4 = (uint4*)(d + 4 * (size_t)r);
            d4[0] = s4[0]; d4[1] = s4[1];
        }
        __syncthreads();
    }
}

}  // namespace
}  // namespace ovs
