#pragma once
// ovs_engine.cuh — host orchestration (the sort engine) of the B200-native
// partition-first oversampling sort.  Every step of the sort runs in the kernels of
// ovs_kernels.cuh; this file only validates arguments, carves the caller's workspace and
// enqueues kernels on the caller's stream (no host synchronisation unless a report is asked).
#include "ovs.h"
#include "ovs_kernels.cuh"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>
#include <mutex>
#include <unordered_map>
#include <memory>

namespace ovs {


struct CudaFail : std::runtime_error {
    explicit CudaFail(const std::string& s) : std::runtime_error(s) {}
};
struct StatusFail {
    int code;
    std::string msg;
};

#define OVS_CK(x)                                                                                  \
    do {                                                                                           \
        cudaError_t e_ = (x);                                                                      \
        if (e_ != cudaSuccess)                                                                     \
            throw CudaFail(std::string(#x) + ": " + cudaGetErrorString(e_));                       \
    } while (0)

struct DevInfo {
    int sms = 148;
    int smem_optin = 232448;
    long long l2_bytes = 126ll << 20;
};

inline DevInfo dev_info_impl() {
    DevInfo d;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return d; }
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0) d.sms = v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) == cudaSuccess && v > 0)
        d.smem_optin = v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev) == cudaSuccess && v > 0) d.l2_bytes = v;
    cudaGetLastError();
    return d;
}

constexpr u32 OVS_NMARKS = 6;

#ifndef OVS_INT_SAMPLES
#define OVS_INT_SAMPLES 4096
#endif

// ------------------------------------------------------------------ workspace carving
// The same code path sizes the workspace (dry run) and hands out pointers (real run).
struct Ctx {
    cudaStream_t st = nullptr;
    char* ws = nullptr;
    size_t off = 0;
    bool dry = true;
    u32 launches = 0;
    DevInfo di;
    u32* status = nullptr;
    const std::vector<cudaEvent_t>* marks = nullptr;  // ovs_set_phase_events
    cudaEvent_t* rep_marks = nullptr;                  // the report's phase events (OVS_NMARKS)
    // phase boundary k (include/ovs.h, ovs_set_phase_events): 0 start, 1 sample drawn, 2 splitters,
    // 3 classify + histogram + scans, 4 scatter, 5 bucket sort (end)
    void mark(u32 k) {
        if (dry) return;
        if (marks && k < marks->size() && (*marks)[k]) OVS_CK(cudaEventRecord((*marks)[k], st));
        if (rep_marks && k < OVS_NMARKS) OVS_CK(cudaEventRecord(rep_marks[k], st));
    }
    template <class T> T* take(size_t count) {
        off = (off + 255) & ~(size_t)255;
        T* p = dry ? nullptr : (T*)(ws + off);
        off += count * sizeof(T);
        return p;
    }
    void check() {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) throw CudaFail(std::string("kernel launch: ") + cudaGetErrorString(e));
        ++launches;
    }
};

static inline u32 cdiv(u64 a, u64 b) { return (u32)((a + b - 1) / b); }

// Dynamic shared memory limit of a kernel, raised once per (device, kernel) to the most the
// kernel can use (the device's opt-in limit minus its static shared memory), so no launch pays
// for cudaFuncSetAttribute again; `need` is checked against it.  The attribute is per device, so
// the cache is keyed by the current device too.
struct SmemKey {
    int dev;
    const void* k;
    bool operator==(const SmemKey& o) const { return dev == o.dev && k == o.k; }
};
struct SmemKeyHash {
    size_t operator()(const SmemKey& x) const { return std::hash<const void*>()(x.k) ^ ((size_t)x.dev * 0x9e3779b97f4a7c15ull); }
};
template <class... KA>
static void smem_limit(void (*k)(KA...), size_t need, const DevInfo& di) {
    static std::mutex mu;
    static std::unordered_map<SmemKey, size_t, SmemKeyHash> lim;
    int dev = 0;
    OVS_CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(mu);
    auto it = lim.find(SmemKey{dev, (const void*)k});
    if (it == lim.end()) {
        cudaFuncAttributes fa;
        OVS_CK(cudaFuncGetAttributes(&fa, (const void*)k));
        const size_t mx = (size_t)di.smem_optin - fa.sharedSizeBytes;
        OVS_CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx));
        it = lim.emplace(SmemKey{dev, (const void*)k}, mx).first;
    }
    if (need > it->second) throw CudaFail("kernel shared memory " + std::to_string(need) + " > limit " + std::to_string(it->second));
}

// Kernel launch (cudaLaunchKernelEx).  With -DOVS_PDL=1 it sets programmatic dependent launch
// (cudaLaunchAttributeProgrammaticStreamSerialization): every kernel starts with PDL_PROLOGUE, so
// its successor may be scheduled while it drains; off by default (no measured gain).
template <class... KA, class... AA>
static void launch(Ctx& c, void (*k)(KA...), dim3 grid, dim3 block, size_t smem, AA&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = OVS_PDL;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    OVS_CK(cudaLaunchKernelEx(&cfg, k, std::forward<AA>(args)...));
}
// cooperative launch (every CTA resident at once: the kernel uses grid-wide barriers)
template <class... KA, class... AA>
static void launch_coop(Ctx& c, void (*k)(KA...), dim3 grid, dim3 block, size_t smem, AA&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    OVS_CK(cudaLaunchKernelEx(&cfg, k, std::forward<AA>(args)...));
}
static inline u32 pow2_at_least(u32 x) {
    u32 p = 1;
    while (p < x) p <<= 1;
    return p;
}
static inline u32 bits_for(u64 n) {  // bits needed for the values 0 .. n-1 (>= 1)
    u32 b = 1;
    while (b < 32 && (1ull << b) < n) ++b;
    return b;
}
static inline u32 ilog2(u32 x) {
    u32 l = 0;
    while ((1u << (l + 1)) <= x) ++l;
    return l;
}

// shared-memory capacity (items) of the bucket sorter
template <class U, bool KV> static u32 bucket_cap(const DevInfo& di) {
    const size_t reserve = 8192;  // static shared memory of k_bucket_sort (~5.5 KB)
    size_t avail = (size_t)di.smem_optin - bucket_smem_fixed<U, KV>() - reserve;
    u32 cap = (u32)(avail / bucket_item_bytes<U, KV>());
    return cap & ~31u;
}
template <class U, bool KV> static size_t bucket_smem(u32 cap) {
    return bucket_smem_fixed<U, KV>() + (size_t)cap * bucket_item_bytes<U, KV>();
}

#ifndef OVS_WC_NT
#define OVS_WC_NT 1024
#endif
// write-combining scatter: WC_NT threads x WC_ITEMS (u32) keys per sub-tile
#ifndef OVS_WC_TILE
#define OVS_WC_TILE 8192
#endif
constexpr int WC_NT = OVS_WC_NT, WC_ITEMS = OVS_WC_TILE / OVS_WC_NT;
#ifndef OVS_REFINE_WC  // ROS refinement stays within the write-combining scatter's bucket count
#define OVS_REFINE_WC 1
#endif
#ifndef OVS_SEL_FUSED  // a3+a4 of 32-bit-key ROS samples in one cooperative launch (k_sel_fused)
#define OVS_SEL_FUSED 1
#endif
#ifndef OVS_SEL_PER_BUCKET
#define OVS_SEL_PER_BUCKET 2048u
#endif
// partition tile shape: 512 threads x ITEMS per sub-tile
constexpr int PT_NT = 512;
template <class U, bool KV> struct PartItems { static constexpr int v = (sizeof(U) == 4 && !KV) ? 16 : 8; };

static void fill_u32(Ctx& c, u32* p, u32 v, u32 n) {
    if (c.dry || n == 0) return;
    launch(c, k_fill_u32, cdiv(n, 256), 256, 0, p, v, n);
    c.check();
}

// Number of candidate draws for the ROS sample (reading Q1: the first ps-1 distinct values of
// the counter stream): the expected number of draws to collect m distinct indices out of n
// (coupon collector, E = n(H_n - H_{n-m})) plus 10 standard deviations and 64; a shortfall
// (probability below 1e-20, never observed) is caught on the device (ST_SAMPLE_SHORT).
inline u64 ros_draws(u64 n, u64 m) {
    const double N = (double)n, a = (double)(n - m) + 0.5, b = N + 0.5;
    const double E = N * std::log(b / a);
    const double var = std::max(0.0, N * N * (1.0 / a - 1.0 / b) - E);
    const double M = std::ceil(E + 10.0 * std::sqrt(var) + 64.0);
    return (u64)std::max<double>(M, (double)m);  // < 2^37 for n < 2^32: inside the 2^40 stream
}

// ------------------------------------------------------------------ the sort engine
// Sorts an array held in buffer 0 of B (codec DT: the caller's raw keys, or internal ordered
// keys with DT_U64) into buffer 0, through a level-0 partition and the bucket sorter.
// Splitters for level 0 come either from the caller (the contract ROS / DRO splitters) or
// from an internal random sample (p == 1 and the internal sorts of sample arrays).
template <int DT, bool KV> struct Engine {
    typedef typename Codec<DT>::U U;

    Ctx& c;
    Bufs<U> B;
    u32 n;
    u32 cap;
    bool mark_phases = false;  // the contract-level engine records the phase events
    u32 tag_base = 0;          // level-0 tag of item i = tag_base + i (multi-GPU: global index)
    u32 ixbits = 32;           // key-value sorts: original indices are < 2^ixbits
    explicit Engine(Ctx& ctx) : c(ctx) {}

    struct Level0 {
        u32 P = 1, L = 0, log2L = 0, nchunk = 0, chunk = 0;
        U* sk = nullptr; u32* st = nullptr; u32* lut = nullptr;
        Seg* seg = nullptr; Chunk* chunks = nullptr; u32* nchunks = nullptr;
        u32* hist = nullptr; u32* tot = nullptr; u32* nseg = nullptr;
        u16* bid = nullptr;  // keys only: every key's bucket, from the histogram pass (scatter input)
    };
    struct Lists {
        Bucket* fit = nullptr; u32* nfit = nullptr; u32* ticket = nullptr; u32 fit_cap = 0;
        Bucket* stack = nullptr; u32 grid = 0;
        Bucket* wl = nullptr; u32* nwl = nullptr; u32 wl_cap = 0;  // buckets sorted in windows
    };

    // keys-only sorts use the write-combining scatter when its shared memory fits
    bool use_wc(u32 P) const {
        return !KV && P > 1 && wc_smem_bytes<U>(P) + 512 <= (size_t)c.di.smem_optin;
    }
    static size_t scatter_smem(u32 P, u32 L) {
        return scatter_smem_bytes<U, KV, PartItems<U, KV>::v, PT_NT>(P, L);
    }
    u32 max_p_one_level() const {
        // largest P whose scatter working set fits shared memory (with the smallest table)
        u32 lo = 1, hi = 8192;  // 13-bit classifier table entries
        while (lo < hi) {
            u32 mid = (lo + hi + 1) / 2;
            if (use_wc(mid) || scatter_smem(mid, 64) + 1024 <= (size_t)c.di.smem_optin) lo = mid; else hi = mid - 1;
        }
        return lo;
    }

    void carve_level0(Level0& z, u32 P) {
        z.P = P;
        // classifier table: ~8 entries per splitter for keys-only sorts (only the histogram pass
        // holds it), ~4 for key-value sorts (the scatter holds it next to its staging area)
        // (the write-combining scatter does not classify; the generic scatter does)
        const bool wc = use_wc(P);
        z.L = P > 1 ? std::min<u32>(wc ? 32768 : 16384, std::max<u32>(64, pow2_at_least((wc ? 8 : 4) * P))) : 1;
        while (z.L > 64 && (wc ? cls_smem_bytes<U>(P, z.L) + 4 * (size_t)P : scatter_smem(P, z.L)) + 1024 >
                               (size_t)c.di.smem_optin)
            z.L >>= 1;
        z.log2L = ilog2(z.L);
        // chunks: one per resident CTA slot, whole sub-tiles
        const u32 ts = PT_NT * PartItems<U, KV>::v;
        u32 want = (u32)c.di.sms * (wc ? OVS_WC_MINB : 1);  // one chunk per resident scatter CTA
        z.chunk = std::max<u32>(ts, cdiv(cdiv(n, want), ts) * ts);
        z.nchunk = std::max<u32>(1, cdiv(n, z.chunk));
        z.sk = c.take<U>(std::max<u32>(P, 1));
        z.st = c.take<u32>(std::max<u32>(P, 1));
        z.lut = c.take<u32>(z.L + 1);
        z.seg = c.take<Seg>(1);
        z.chunks = c.take<Chunk>(z.nchunk);
        z.nchunks = c.take<u32>(2);
        z.nseg = z.nchunks + 1;
        z.hist = c.take<u32>((size_t)z.nchunk * P);
        z.tot = c.take<u32>(P + 1);
        if (!KV && P > 1) z.bid = c.take<u16>(n);
    }
    void carve_lists(Lists& l, u32 P) {
        l.fit_cap = P + 64;
        l.fit = c.take<Bucket>(l.fit_cap);
        l.nfit = c.take<u32>(2);
        l.ticket = l.nfit + 1;
        l.grid = (u32)c.di.sms;  // bucket sorter: one CTA per SM (shared-memory bound)
        l.stack = c.take<Bucket>((size_t)l.grid * BS_STACK);
        l.wl_cap = std::max<u32>(64, n / std::max<u32>(cap, 1) + 64);  // windowed buckets exceed cap
        l.wl = c.take<Bucket>(l.wl_cap);
        l.nwl = c.take<u32>(2);
    }

    // internal splitters for level 0 (P-1 of them) from a one-CTA sorted random sample
    void internal_splitters(Level0& z, u64 seed) {
        if (c.dry || z.P <= 1) return;
        // up to 32 samples per internal splitter, at most OVS_INT_SAMPLES in all, sorted by one CTA
        // (a power-of-two bitonic network)
        const u32 si = std::max<u32>(1, std::min<u32>(32, OVS_INT_SAMPLES / z.P));
        const u32 N = pow2_at_least(z.P * si);
        const size_t sm = (sizeof(U) + 4) * (size_t)N;
        smem_limit(k_internal_sample<DT, KV>, sm, c.di);
        launch(c, k_internal_sample<DT, KV>, 1, 1024, sm, B, n, z.P, si, N, seed, z.sk, z.st);
        c.check();
    }

    // level 0: classifier build, histogram, scans, scatter buffer 0 -> buffer 1
    void level0_hist(Level0& z, Lists& l, u64* counts_out) {
        if (c.dry) return;
        const size_t sm_cls = std::max<size_t>(sizeof(U) * std::max<u32>(z.P, 1), 16);
        smem_limit(k_build_cls0<U>, sm_cls, c.di);
        launch(c, k_build_cls0<U>, std::max<u32>(16, std::min<u32>(z.L / 1024 + 1, 64)), 1024, sm_cls,
            z.sk, z.P, z.L, z.log2L, z.lut, z.seg, n, z.nchunk, z.chunk, z.chunks, z.nchunks, l.nfit, z.hist,
            z.nchunk * z.P);
        c.check();
        const size_t sm_h = cls_smem_bytes<U>(z.P, z.L) + 4 * (size_t)z.P;
        const u32 hsplit = 2;  // two 1024-thread CTAs per chunk
        smem_limit(k_hist<DT, KV, true, 1024>, sm_h, c.di);
        launch(c, k_hist<DT, KV, true, 1024>, z.nchunk * hsplit, 1024, sm_h, B, z.chunks, z.nchunks, z.seg, z.sk, z.st,
                                                                           z.lut, z.P, z.L, z.hist, hsplit, tag_base,
                                                                           use_wc(z.P) ? z.bid : nullptr);
        c.check();
        launch(c, k_colscan, std::min<u32>(cdiv(z.P, 32), 4 * c.di.sms), 1024, 0, z.hist, z.seg, z.nseg, z.P, z.tot);
        c.check();
        launch(c, k_segscan<U>, 1, 1024, 0, z.seg, z.nseg, z.P, z.tot, z.sk, 0, cap, l.fit, l.nfit, l.fit_cap, nullptr,
                                          nullptr, 0, counts_out, c.status);
        c.check();
        if (mark_phases) c.mark(3);
    }
    void level0(Level0& z, Lists& l, u64* counts_out) {
        level0_hist(z, l, counts_out);
        level0_scatter(z);
    }
    // a7: buffer 0 -> buffer 1 at the scanned positions; DIST: straight into the owners' windows
    // (dst_off[b]: this rank's run of bucket b in its owner's receive region)
    template <bool DIST = false>
    void level0_scatter(Level0& z, const u32* dst_off = nullptr, PeerOut pk = PeerOut{nullptr, 0, 1},
                        size_t off_v = 0, size_t off_i = 0) {
        if (c.dry) return;
        if (use_wc(z.P)) {
            constexpr int IT = WC_ITEMS * 4 / (int)sizeof(U);  // u32: WC_ITEMS keys per thread
            const size_t sm_w = wc_smem_bytes<U>(z.P);
            auto kw = k_scatter_wc<DT, WC_NT, IT, true, DIST>;
            smem_limit(kw, sm_w, c.di);
            launch(c, kw, z.nchunk, WC_NT, sm_w, B, z.chunks, z.nchunks, z.seg, z.P, z.hist, z.tot, (const u16*)z.bid,
                   dst_off, pk);
            c.check();
        } else {
            constexpr int IT = PartItems<U, KV>::v;
            const size_t sm_s = scatter_smem(z.P, z.L);
            auto ks = k_scatter<DT, KV, true, PT_NT, IT, DIST>;
            smem_limit(ks, sm_s, c.di);
            launch(c, ks, z.nchunk, PT_NT, sm_s, B, z.chunks, z.nchunks, z.seg, z.sk, z.st, z.lut, z.P, z.L, z.hist,
                                                z.tot, tag_base, dst_off, pk, off_v, off_i);
            c.check();
        }
        if (mark_phases) c.mark(4);
    }


    // sorts every bucket of the list into okeys (+ ovals, + oidx) at the bucket's position;
    // out_raw applies the codec's inverse (the caller's dtype) on the way out
    void bucket_sort(Lists& l, u64 seed, U* okeys = nullptr, u32* ovals = nullptr, u32* oidx = nullptr,
                     bool out_raw = true) {
        if (c.dry) return;
        if (!okeys) { okeys = B.k[0]; ovals = KV ? B.v[0] : nullptr; }
        const size_t sm = bucket_smem<U, KV>(cap);
        smem_limit(k_bucket_sort<DT, KV, false>, sm, c.di);
        smem_limit(k_bucket_sort<DT, KV, true>, sm, c.di);
        fill_u32(c, l.nwl, 0, 2);
        launch(c, k_bucket_sort<DT, KV, false>, l.grid, BS_NT, sm, l.fit, l.nfit, l.ticket, B, okeys, ovals, oidx, out_raw,
                                                          cap, l.stack, seed, c.status, ixbits, l.wl, l.nwl, l.wl_cap);
        c.check();
        launch(c, k_bucket_sort<DT, KV, true>, l.grid, BS_NT, sm, l.wl, l.nwl, l.nwl + 1, B, okeys, ovals, oidx, out_raw,
               cap, l.stack, seed, c.status, ixbits, l.wl, l.nwl, 0u);
        c.check();
    }
};

// ------------------------------------------------------------------ level 1 (k_l1_setup, ...)
// Re-splits every bucket of a device list by the whole GPU; the sub-buckets (in buffer
// 1 - bucket.buf) are appended to out (its own fit list, sized for maxseg * L1_PS entries).
template <int DT, bool KV> struct Level1 {
    typedef typename Codec<DT>::U U;
    static constexpr u32 PS = 256, LS = 1024, CH = 1u << 16;
    Engine<DT, KV>& e;
    u32 maxseg = 0, maxchunk = 0;
    U* sk = nullptr; u32* st = nullptr; u32* lut = nullptr; Seg* segs = nullptr; u32* nsegs = nullptr;
    Chunk* chunks = nullptr; u32* hist = nullptr; u32* tot = nullptr;
    u16* bid = nullptr;  // keys only: sub-bucket ids (the write-combining scatter's input)
    Level1(Engine<DT, KV>& eng, u32 max_segments) : e(eng) {
        Ctx& c = e.c;
        maxseg = std::max<u32>(1, max_segments);
        maxchunk = e.n / CH + maxseg + 1;
        sk = c.take<U>((size_t)maxseg * PS);
        st = c.take<u32>((size_t)maxseg * PS);
        lut = c.take<u32>((size_t)maxseg * (LS + 1));
        segs = c.take<Seg>(maxseg);
        nsegs = c.take<u32>(2);
        chunks = c.take<Chunk>(maxchunk);
        hist = c.take<u32>((size_t)maxchunk * PS);
        tot = c.take<u32>((size_t)maxseg * (PS + 1));
        if (!KV) bid = c.take<u16>(e.n);
    }
    static size_t setup_smem() { return (sizeof(U) + 4) * (size_t)PS * L1_SI; }
    void run(const Bucket* list, const u32* nlist, typename Engine<DT, KV>::Lists& out, u64 seed) {
        Ctx& c = e.c;
        if (c.dry) return;
        const u32 part = (u32)(e.cap * 6ull / 10);
        const size_t sm0 = setup_smem();
        smem_limit(k_l1_setup<DT, KV>, sm0, c.di);
        launch(c, k_l1_setup<DT, KV>, maxseg, 1024, sm0, e.B, list, nlist, part, PS, LS, 10u, sk, st, lut, segs, nsegs,
               seed, CH);
        c.check();
        launch(c, k_l1_chunks, 1, 1024, 0, segs, nsegs, CH, chunks, nsegs + 1);
        c.check();
        OVS_CK(cudaMemsetAsync(hist, 0, sizeof(u32) * (size_t)maxchunk * PS, c.st));
        const size_t sm_h = cls_smem_bytes<U>(PS, LS) + 4 * (size_t)PS;
        smem_limit(k_hist<DT, KV, false, 1024>, sm_h, c.di);
        launch(c, k_hist<DT, KV, false, 1024>, std::min<u32>(maxchunk, 4 * (u32)c.di.sms), 1024, sm_h, e.B, chunks,
               nsegs + 1, segs, sk, st, lut, PS, LS, hist, 1u, 0u, bid);
        c.check();
        launch(c, k_colscan, std::min<u32>(maxseg * (PS / 32), 4 * (u32)c.di.sms), 1024, 0, hist, segs, nsegs, PS, tot);
        c.check();
        launch(c, k_segscan<U>, std::min<u32>(maxseg, 2 * (u32)c.di.sms), 1024, 0, segs, nsegs, PS, tot, sk, 1u, e.cap,
               out.fit, out.nfit, out.fit_cap, (Bucket*)nullptr, (u32*)nullptr, 0u, (u64*)nullptr, c.status);
        c.check();
        if (!KV) {
            constexpr int IT = WC_ITEMS * 4 / (int)sizeof(U);
            const size_t sm_w = wc_smem_bytes<U>(PS);
            auto kw = k_scatter_wc<DT, WC_NT, IT, false>;
            smem_limit(kw, sm_w, c.di);
            launch(c, kw, std::min<u32>(maxchunk, (u32)c.di.sms), WC_NT, sm_w, e.B, chunks, nsegs + 1, segs, PS, hist, tot,
                   (const u16*)bid, (const u32*)nullptr, PeerOut{nullptr, 0, 1});
        } else {
            constexpr int IT = PartItems<U, KV>::v;
            const size_t sm_s = Engine<DT, KV>::scatter_smem(PS, LS);
            auto ks = k_scatter<DT, KV, false, PT_NT, IT>;
            smem_limit(ks, sm_s, c.di);
            launch(c, ks, std::min<u32>(maxchunk, 2 * (u32)c.di.sms), PT_NT, sm_s, e.B, chunks, nsegs + 1, segs, sk, st,
                   lut, PS, LS, hist, tot, 0u, (const u32*)nullptr, PeerOut{nullptr, 0, 1}, (size_t)0, (size_t)0);
        }
        c.check();
    }
};

// ------------------------------------------------------------------ internal sort of an array
// keys (ordered u64) [+ u32 values, sorted stably] in buffer 0 of B; buffer 1 scratch.
template <bool KV> struct InternalSort {
    Engine<DT_U64, KV> e;
    typename Engine<DT_U64, KV>::Level0 z;
    typename Engine<DT_U64, KV>::Lists l;
    bool direct = false;
    InternalSort(Ctx& c, u32 n, u64* k0, u32* v0) : e(c) {
        e.n = n;
        e.cap = bucket_cap<u64, KV>(c.di);
        e.B.k[0] = k0;
        e.B.k[1] = c.take<u64>(n);
        e.B.v[0] = v0;
        e.B.v[1] = KV ? c.take<u32>(n) : nullptr;
        e.B.i[0] = KV ? c.take<u32>(n) : nullptr;
        e.B.i[1] = KV ? c.take<u32>(n) : nullptr;
        direct = n <= e.cap;
        // internal buckets of ~cap/8 keys: enough of them to occupy every SM
        u32 P = direct ? 1 : std::min<u32>(1024, cdiv(n, e.cap / 8));
        if (!direct) e.carve_level0(z, P);
        e.carve_lists(l, direct ? 1 : P);
    }
    void run(u64 seed) {
        Ctx& c = e.c;
        if (c.dry || e.n == 0) return;
        if (direct) {
            if (KV) { launch(c, k_iota, cdiv(e.n, 256), 256, 0, e.B.i[0], e.n); c.check(); }
            launch(c, k_fill_u32, 1, 2, 0, l.nfit, 0, 2);
            c.check();
            launch(c, k_push_bucket<u64>, 1, 1, 0, l.fit, l.nfit, e.n);
            c.check();
        } else {
            e.internal_splitters(z, seed);
            e.level0(z, l, nullptr);
        }
        e.bucket_sort(l, seed);
    }
};

// DRO's sample T (p sorted runs of s records): merged (SampleMerge) while the merge's two arrays
// fit in half the L2, else sorted by the generic internal sort — measured on B200: C2 (12.6 MB of
// records) 0.20 -> 0.11 ms merged; C4 (56.6 MB, 9 levels that miss L2) 0.43 ms sorted, 0.42 ms
// merged (break-even).  OVS_DRO_SAMPLE_SORT=1 / =0 forces the sort / the merge (experiments and tests).
static inline bool sample_sorted(const DevInfo& di, u64 ns, bool w64) {
    const char* v = getenv("OVS_DRO_SAMPLE_SORT");
    if (v && (v[0] == '0' || v[0] == '1')) return v[0] == '1';
    return 2 * ns * (w64 ? 12 : 8) > (u64)di.l2_bytes / 2;
}
// ------------------------------------------------------------------ a11: merge of the DRO sample
// The p sorted regular samples T_k (s records each, contiguous, run k at k*s) merged into T by
// ceil(lg p) levels of the pairwise merge k_sample_merge (Algorithm 1 step 2, PAPER.md:266,
// PAPER.md:359-364), ping-ponging between the sample arrays and one scratch pair.  T is identical
// to a sort of the sample (records are unique by their tag).  run() returns the buffer holding T.
struct SampleMerge {
    Ctx& c;
    u32 ns, s;
    bool w64;
    u64* k[2] = {nullptr, nullptr};
    u32* t[2] = {nullptr, nullptr};
    SampleMerge(Ctx& c_, u32 ns_, u32 s_, u64* k0, u32* t0, bool w64_) : c(c_), ns(ns_), s(s_), w64(w64_) {
        k[0] = k0;
        t[0] = t0;
        k[1] = c.take<u64>(ns);
        t[1] = w64 ? c.take<u32>(ns) : nullptr;
    }
    int run() {
        int cur = 0;
        if (c.dry || ns == 0 || s == 0) return cur;
        for (u64 L = s; L < ns; L *= 2) {
            const u32 tpp = (u32)cdiv(2 * L, (u64)MS_TILE), pairs = (u32)cdiv((u64)ns, 2 * L);
            if (w64)
                launch(c, k_sample_merge<true>, pairs * tpp, MS_NT, 0, (const u64*)k[cur], (const u32*)t[cur], k[cur ^ 1],
                       t[cur ^ 1], ns, (u32)L, tpp);
            else
                launch(c, k_sample_merge<false>, pairs * tpp, MS_NT, 0, (const u64*)k[cur], (const u32*)nullptr,
                       k[cur ^ 1], (u32*)nullptr, ns, (u32)L, tpp);
            c.check();
            cur ^= 1;
        }
        return cur;
    }
};

// ------------------------------------------------------------------ a3+a4: sample sort + splitters
// The m sample records (key word [, tag]) in draw order -> G coarse buckets (k_sel_count,
// k_sel_scatter) -> every coarse bucket sorted by the bucket sorter -> S[q] = T[(q+1)s - 1].
// 32-bit keys: one word (ord key << 32 | tag), sorted as u64 keys; 64-bit keys: key word + tag,
// sorted as (key, tag) pairs (the tag rides as the value and is the tie-break index).
template <bool TAG> struct Selector {
    Engine<DT_U64, TAG> e;
    typename Engine<DT_U64, TAG>::Lists l;
    u32 m, G;
    const u64* tk = nullptr;
    const u32* tt = nullptr;
    u64* csk = nullptr; u32* cst = nullptr; uint8_t* cb = nullptr;
    u32* gcnt = nullptr; u32* gcur = nullptr;  // zeroed by the owner before run()
    u32 stride = 1;  // coarse subsample: T[i] (1, T in random order) or random positions (0)
    Selector(Ctx& c, u32 m_, const u64* tk_, const u32* tt_, u32* gcnt_, u32* gcur_)
        : e(c), m(m_), tk(tk_), tt(tt_), gcnt(gcnt_), gcur(gcur_) {
        u32 g = 1;
        while (g * 2 <= m / OVS_SEL_PER_BUCKET && g * 2 <= SEL_GMAX) g *= 2;
        G = g;
        e.n = m;
        e.cap = bucket_cap<u64, TAG>(c.di);
        e.B.k[0] = c.take<u64>(m);
        e.B.k[1] = c.take<u64>(m);
        e.B.v[0] = TAG ? c.take<u32>(m) : nullptr;
        e.B.v[1] = TAG ? c.take<u32>(m) : nullptr;
        e.B.i[0] = TAG ? c.take<u32>(m) : nullptr;
        e.B.i[1] = TAG ? c.take<u32>(m) : nullptr;
        csk = c.take<u64>(SEL_GMAX);
        cst = c.take<u32>(SEL_GMAX);
        cb = c.take<uint8_t>(m);
        e.carve_lists(l, G);
    }
    template <class U> void run(u32 P, u32 s, u32 f, u64 seed, U* sk, u32* st) {
        Ctx& c = e.c;
        if (c.dry) return;
        sort(seed);
        pick<U>(P, s, f, sk, st);
    }
    // the sorted records (key word e.B.k[0], tag e.B.v[0]) without picking splitters
    void sort(u64 seed) {
        Ctx& c = e.c;
        if (c.dry) return;
        const u32 grid = cdiv(m, SEL_PER);
        launch(c, k_sel_count<TAG>, grid, 1024, 0, tk, tt, m, G, stride, csk, cst, cb, gcnt);
        c.check();
        launch(c, k_sel_scatter<TAG>, grid, 1024, 0, tk, tt, m, G, cb, gcnt, gcur, csk, e.B.k[1], e.B.v[1], e.B.i[1],
                                                    l.fit, l.nfit);
        c.check();
        e.bucket_sort(l, seed);
    }
    // 32-bit keys (packed records) drawn in random order: a3+a4 in one cooperative launch
    // (its own coarse bucket count: <= 2048 records per bucket on average, one CTA each)
    u32 fused_G() const {
        u32 g = 1;
        while ((u64)g * SF_NT * SF_IT < m) g *= 2;
        return g;
    }
    bool fused_ok() const { return !TAG && stride == 1 && fused_G() <= std::min<u32>(SEL_GMAX, (u32)e.c.di.sms); }
    template <int DT>
    void run_fused(u32 P, u32 s, u32 f, typename Codec<DT>::U* sk, u32* st) {
        Ctx& c = e.c;
        if (c.dry) return;
        const size_t sm = 16 * (size_t)SF_MAXB + 4 * (size_t)SF_NG;
        auto k = k_sel_fused<DT>;
        smem_limit(k, sm, c.di);
        launch_coop(c, k, fused_G(), SF_NT, sm, tk, m, gcnt, gcur, e.B.k[1], e.B.k[0], P, s, f, sk, st, c.status);
        c.check();
    }
    // S[q] = T[(q+1)s - 1], q < P-1, from the sorted records
    template <class U> void pick(u32 P, u32 s, u32 f, U* sk, u32* st) {
        Ctx& c = e.c;
        if (c.dry) return;
        launch(c, k_pick_splitters<U>, cdiv(P, 256), 256, 0, e.B.k[0], e.B.k[0], e.B.v[0], P, s, f, sk, st);
        c.check();
    }
};

// a1+a2: the ROS sample index set I (first ps-1 distinct draws, reading Q1) and the records
// T = [(x[i], i)], hash-set form (k_ros_draw, k_ros_first, k_ros_take); DIST: the global index
// set over n_global keys, each rank contributing the records of its own shard.
template <int DT, bool DIST> struct RosSampler {
    typedef typename Codec<DT>::U U;
    static constexpr bool TAG = sizeof(U) == 8;
    Ctx& c;
    u64 n, Mfull;
    u32 m, M = 0, lg = 0, nb = 0;
    u64* zero = nullptr; u32* bits = nullptr; u32* bcnt = nullptr;
    u64* tk = nullptr; u32* tt = nullptr;
    Selector<TAG>* sel = nullptr;
    // direct-address form (k_ros_draw_direct ...): when the draws outnumber the indices or the
    // hash set would be too large (samples that are a large fraction of n, up to ps-1 = n)
    bool direct = false;
    u64* minj = nullptr; RSel* rsel = nullptr; u32* ghist = nullptr; u32* dbcnt = nullptr;
    u32 dnb = 0, Lr = 0;
    RosSampler(Ctx& ctx, u64 n_, u32 p, u32 s) : c(ctx), n(n_) {
        m = p * s - 1;
        Mfull = ros_draws(n, m);
        direct = Mfull > (1ull << 26) || Mfull > n;
        u32* gcnt = nullptr;
        if (!direct) {
            M = (u32)Mfull;
            lg = ilog2(pow2_at_least(std::max<u32>(1024, M + M / 2)));
            nb = cdiv(M, TK_NT);
            zero = c.take<u64>(((size_t)1 << lg) + SEL_GMAX);
            bits = c.take<u32>((size_t)nb * (TK_NT / 32));
            bcnt = c.take<u32>(nb);
            gcnt = zero ? (u32*)(zero + ((size_t)1 << lg)) : nullptr;
        } else {
            zero = c.take<u64>(SEL_GMAX);
            gcnt = zero ? (u32*)zero : nullptr;
            minj = c.take<u64>(n);
            rsel = c.take<RSel>(1);
            ghist = c.take<u32>(RS_BINS);
            dnb = (u32)((n + DT_NT * DT_PER - 1) / (DT_NT * DT_PER));
            dbcnt = c.take<u32>(dnb + 1);
            u32 L = 1;
            while (L < 64 && (Mfull - 1) >> L) ++L;  // bits of the largest draw number
            Lr = (L + RS_BITS - 1) / RS_BITS * RS_BITS;
        }
        tk = c.take<u64>(m);
        tt = TAG ? c.take<u32>(m) : nullptr;
        sel = new Selector<TAG>(c, m, tk, tt, gcnt, gcnt ? gcnt + SEL_GMAX : nullptr);
        if (direct) sel->stride = 0;  // T in index order: coarse splitters from random positions
    }
    ~RosSampler() { delete sel; }
    size_t zero_bytes() const { return 8 * ((direct ? 0 : ((size_t)1 << lg)) + SEL_GMAX); }
    // the hash set of the draws and the first-draw masks (direct: the table and j*)
    void draw(u64 seed) {
        if (c.dry) return;
        OVS_CK(cudaMemsetAsync(zero, 0, zero_bytes(), c.st));
        if (direct) {
            OVS_CK(cudaMemsetAsync(minj, 0xff, 8 * (size_t)n, c.st));
            const u64 g = std::min<u64>((Mfull + 255) / 256, (u64)c.di.sms * 16);
            launch(c, k_ros_draw_direct, (u32)g, 256, 0, minj, Mfull, n, seed);
            c.check();
            launch(c, k_rsel_init, 1, 1024, 0, rsel, (u64)(m - 1), ghist);
            c.check();
            const u32 hg = std::min<u32>(cdiv(n, 1024 * 8), (u32)c.di.sms * 2);
            for (int sh = (int)Lr - (int)RS_BITS; sh >= 0; sh -= (int)RS_BITS) {
                launch(c, k_rsel_hist, std::max<u32>(hg, 1), 1024, 0, (const u64*)minj, n, (const RSel*)rsel, (u32)sh, ghist);
                c.check();
                launch(c, k_rsel_pick, 1, 1024, 0, rsel, (u32)sh, ghist, c.status, sh == 0 ? 1u : 0u);
                c.check();
            }
            return;
        }
        launch(c, k_ros_draw, cdiv(M, 256), 256, 0, zero, lg, M, n, seed);
        c.check();
        launch(c, k_ros_first, nb, TK_NT, 0, zero, lg, M, n, seed, bits, bcnt);
        c.check();
    }
    // records of the members of I (DIST: of the shard [offset, offset + nl), into rec)
    void take(u64 seed, const U* x, u64 offset, u32 nl, PeerOut po = PeerOut{nullptr, 0, 1}) {
        if (c.dry) return;
        if (direct) {
            launch(c, k_direct_count, dnb, DT_NT, 0, (const u64*)minj, n, (const RSel*)rsel, dbcnt);
            c.check();
            launch(c, k_direct_scan, 1, 1024, 0, dbcnt, dnb, m, c.status);
            c.check();
            launch(c, k_direct_take<DT, DIST>, dnb, DT_NT, 0, (const u64*)minj, n, (const RSel*)rsel,
                   (const u32*)dbcnt, x, offset, nl, tk, tt, po);
            c.check();
            return;
        }
        launch(c, k_ros_take<DT, DIST>, nb, TK_NT, 0, bits, bcnt, M, n, seed, m, x, offset, nl, tk, tt, c.status, po);
        c.check();
    }
    void select(u32 P, u32 s, u32 f, u64 seed, U* sk, u32* st) {
        if (OVS_SEL_FUSED && !DIST && !TAG && sel->fused_ok()) {
            sel->template run_fused<DT>(P, s, f, sk, st);
        } else {
            sel->template run<U>(P, s, f, seed, sk, st);
        }
    }
};

// ------------------------------------------------------------------ ROS contract sort
template <int DT, bool KV> struct RosSort {
    typedef typename Codec<DT>::U U;
    Ctx& c;
    Engine<DT, KV> e;
    typename Engine<DT, KV>::Level0 z;
    typename Engine<DT, KV>::Lists l;
    u32 n, p, s;
    u64 seed;
    u64* counts = nullptr;
    RosSampler<DT, false>* smp = nullptr;  // a1-a4
    // Refinement: when the contract's buckets (n/p keys) cannot be sorted on chip, level 0
    // partitions into p*f buckets with the splitters T[floor((i+1)s/f) - 1] (>= 8 samples each),
    // a superset of the contract's T[(q+1)s - 1] (i = (q+1)f - 1).  Contract bucket q is
    // exactly the concatenation of level-0 buckets qf .. qf+f-1, so the output is unchanged and
    // the contract's splitters and counts are read off (k_pick_splitters, k_fold_counts).
    u32 f = 1;
    U* rep_sk = nullptr;
    u32* rep_st = nullptr;
    u64* int_counts = nullptr;

    RosSort(Ctx& ctx, U* keys, u32* vals, u32 n_, u32 p_, u32 s_, u64 seed_) : c(ctx), e(ctx), n(n_), p(p_), s(s_), seed(seed_) {
        e.n = n;
        e.ixbits = bits_for(n);
        e.cap = bucket_cap<U, KV>(c.di);
        e.B.k[0] = keys;
        e.B.v[0] = vals;
        e.B.k[1] = c.take<U>(n);
        e.B.v[1] = KV ? c.take<u32>(n) : nullptr;
        e.B.i[0] = KV ? c.take<u32>(n) : nullptr;
        e.B.i[1] = KV ? c.take<u32>(n) : nullptr;
        counts = c.take<u64>(std::max<u32>(p, 1));
        u32 P0 = p;
        if (p == 1) P0 = n > e.cap ? std::min<u32>(std::min<u32>(1024, e.max_p_one_level()),
                                                   cdiv(n, (u32)(e.cap * 45ull / 100))) : 1;
        if (p > 1) {
            // refine while the buckets exceed the on-chip capacity, within the bucket count the
            // fast scatter handles (keys only: the write-combining one)
            u32 pmax = std::min<u32>(8192, e.max_p_one_level());
            if (OVS_REFINE_WC && !KV && e.use_wc(p)) while (pmax > p && !e.use_wc(pmax)) --pmax;
            while (s / (2 * f) >= 8 && (u64)p * 2 * f <= pmax && (u64)n > (u64)p * f * e.cap)
                f *= 2;
            P0 = p * f;
            if (f > 1) {
                rep_sk = c.take<U>(p);
                rep_st = c.take<u32>(p);
                int_counts = c.take<u64>(P0);
            }
        }
        e.carve_level0(z, P0);
        e.carve_lists(l, P0);
        if (p > 1) smp = new RosSampler<DT, false>(c, n, p, s);
    }
    ~RosSort() { delete smp; }

    void run() {
        if (c.dry) return;
        e.mark_phases = true;
        c.mark(0);
        if (p > 1) {
            // a1+a2: ps-1 distinct random indices and their records T = [(x[i], i)]
            smp->draw(seed);
            smp->take(seed, e.B.k[0], 0, n);
            c.mark(1);
            // a3+a4: sort T by (key, i); S[q] = T[(q+1)s - 1] (refined: every (s/f)-th)
            smp->select(p * f, s, f, seed ^ 0x5eed, z.sk, z.st);
            if (f > 1) smp->sel->template pick<U>(p, s, 1, rep_sk, rep_st);
        } else {
            e.internal_splitters(z, seed);
            c.mark(1);
        }
        c.mark(2);
        // a5-a7: classify, histogram, scan, scatter;  a8: bucket sort
        e.level0(z, l, p > 1 ? (f > 1 ? int_counts : counts) : nullptr);
        if (f > 1) {
            launch(c, k_fold_counts, cdiv(p, 256), 256, 0, int_counts, f, p, counts);
            c.check();
        }
        e.bucket_sort(l, seed);
        c.mark(5);
    }
};

// ------------------------------------------------------------------ f3: ROS on 32-byte strings
// (the paper's workload).  Same contract as RosSort:
// sample index set I (reading Q1), T sorted by (full key, index), S[q] = T[(q+1)s - 1], buckets by
// the tagged lower bound, every bucket sorted, concatenated.  Keys only (equal strings are equal
// bytes).  Refinement f as in RosSort keeps buckets on chip.
struct RosSortS32 {
    Ctx& c;
    u32 n, p, s, f = 1, P0 = 1, L = 64, log2L = 6, nchunk = 1, chunk = 0, cap = 0;
    u64 seed;
    u64* recs = nullptr; u64* buf1 = nullptr;
    u16* bid = nullptr; u32* gidx = nullptr;
    u64* sk = nullptr; u32* st = nullptr; u32* lut = nullptr; Seg* seg = nullptr; Chunk* chunks = nullptr;
    u32* nchunks = nullptr; u32* nseg = nullptr; u32* hist = nullptr; u32* tot = nullptr;
    u64* sfull = nullptr;
    u64* counts = nullptr; u64* int_counts = nullptr;
    u64* rep_sk = nullptr; u32* rep_st = nullptr; u64* rep_raw = nullptr; u64* rep_full = nullptr;
    u32* fixl = nullptr; u32* nfix = nullptr; u32 fix_cap = 0;
    Bucket* fit = nullptr; u32* nfit = nullptr; u32 fit_cap = 0;
    RosSampler<DT_S32, false>* smp = nullptr;

    static u32 cap_s32(const DevInfo& di) {
        return (u32)(((size_t)di.smem_optin - 2048) / 36) & ~31u;
    }
    u32 pc = 1;  // the contract's p (p == 1, a plain sort: an internal p keeps the buckets on chip)
    RosSortS32(Ctx& ctx, void* keys, u32 n_, u32 p_, u32 s_, u64 seed_) : c(ctx), n(n_), p(p_), s(s_), seed(seed_) {
        recs = (u64*)keys;
        cap = cap_s32(c.di);
        pc = p;
        if (p == 1 && n > cap) {
            p = std::min<u32>(4096, pow2_at_least(cdiv(n, cap * 6 / 10)));
            s = 16;
            while (p > 2 && (u64)p * s - 1 > n) p >>= 1;
        }
        buf1 = c.take<u64>(4 * (size_t)n);
        bid = c.take<u16>(n);
        gidx = c.take<u32>(n);
        counts = c.take<u64>(std::max<u32>(p, 1));
        if (p > 1) {
            while (s / (2 * f) >= 8 && (u64)p * 2 * f <= 8192 && (u64)n * 10 > (u64)p * f * cap * 6) f *= 2;
            P0 = p * f;
        } else {
            P0 = 1;
        }
        // classifier table: ~4 entries per splitter within the histogram kernel's shared memory
        L = P0 > 1 ? std::min<u32>(16384, std::max<u32>(64, pow2_at_least(4 * P0))) : 1;
        while (L > 64 && cls_smem_bytes<u64>(P0, L) + 4 * (size_t)P0 + 1024 > (size_t)c.di.smem_optin) L >>= 1;
        log2L = ilog2(L);
        chunk = std::max<u32>(4 * S32_NT, cdiv(cdiv(n, (u32)c.di.sms), 4 * S32_NT) * 4 * S32_NT);
        nchunk = std::max<u32>(1, cdiv(n, chunk));
        sk = c.take<u64>(std::max<u32>(P0, 1));
        st = c.take<u32>(std::max<u32>(P0, 1));
        lut = c.take<u32>(L + 1);
        seg = c.take<Seg>(1);
        chunks = c.take<Chunk>(nchunk);
        nchunks = c.take<u32>(2);
        nseg = nchunks + 1;
        hist = c.take<u32>((size_t)nchunk * P0);
        tot = c.take<u32>(P0 + 1);
        sfull = c.take<u64>(4 * (size_t)std::max<u32>(P0, 1));
        rep_sk = c.take<u64>(std::max<u32>(p, 1));
        rep_st = c.take<u32>(std::max<u32>(p, 1));
        rep_raw = c.take<u64>(4 * (size_t)std::max<u32>(p, 1));
        rep_full = c.take<u64>(4 * (size_t)std::max<u32>(p, 1));
        if (f > 1) int_counts = c.take<u64>(P0);
        fit_cap = P0 + 64;
        fit = c.take<Bucket>(fit_cap);
        nfit = c.take<u32>(2);
        if (p > 1) {
            smp = new RosSampler<DT_S32, false>(c, n, p, s);
            fix_cap = 4096;
            fixl = c.take<u32>(2 * (size_t)fix_cap);
            nfix = c.take<u32>(2);
        }
    }
    ~RosSortS32() { delete smp; }

    void run() {
        if (c.dry) return;
        c.mark(0);
        if (p > 1) {
            // a1+a2: the index set I and the records (prefix, index)
            smp->draw(seed);
            smp->take(seed, recs, 0, n);
            c.mark(1);
            // a3: sort by (prefix, index); runs of equal prefixes re-ordered by the full key
            Selector<true>* sel = smp->sel;
            sel->sort(seed ^ 0x5eed);
            fill_u32(c, nfix, 0, 2);
            launch(c, k_s32_fix, cdiv(smp->m, 256), 256, 0, (const u64*)sel->e.B.k[0], sel->e.B.v[0], smp->m,
                   (const u64*)recs, fixl, nfix, fix_cap, c.status);
            c.check();
            launch(c, k_s32_fix_long, (u32)c.di.sms, 1024, 0, sel->e.B.v[0], (const u64*)recs, (const u32*)fixl,
                   (const u32*)nfix);
            c.check();
            // a4: S[q] = T[(q+1)s - 1] (level 0 refined: every (s/f)-th record), their full keys
            sel->template pick<u64>(P0, s, f, sk, st);
            sel->template pick<u64>(p, s, 1, rep_sk, rep_st);
            launch(c, k_s32_splitters, cdiv(P0, 256), 256, 0, (const u32*)st, P0 - 1, (const u64*)recs, sfull,
                   (u64*)nullptr);
            c.check();
            launch(c, k_s32_splitters, cdiv(p, 256), 256, 0, (const u32*)rep_st, p - 1, (const u64*)recs, rep_full,
                   rep_raw);
            c.check();
        } else {
            c.mark(1);
        }
        c.mark(2);
        // a5+a6: classify (prefix table + full-key ties), histogram, scans
        const size_t sm_cls = std::max<size_t>(8 * (size_t)std::max<u32>(P0, 1), 16);
        smem_limit(k_build_cls0<u64>, sm_cls, c.di);
        launch(c, k_build_cls0<u64>, std::max<u32>(16, std::min<u32>(L / 1024 + 1, 64)), 1024, sm_cls, (const u64*)sk,
               P0, L, log2L, lut, seg, n, nchunk, chunk, chunks, nchunks, nfit, hist, nchunk * P0);
        c.check();
        const size_t sm_h = cls_smem_bytes<u64>(P0, L) + 4 * (size_t)P0;
        smem_limit(k_hist_s32, sm_h, c.di);
        launch(c, k_hist_s32, nchunk, S32_NT, sm_h, (const u64*)recs, (const Chunk*)chunks, (const u32*)nchunks, seg,
               (const u64*)sk, (const u32*)st, (const u32*)lut, P0, L, hist, (const u64*)sfull, bid);
        c.check();
        launch(c, k_colscan, std::min<u32>(cdiv(P0, 32), 4 * c.di.sms), 1024, 0, hist, (const Seg*)seg,
               (const u32*)nseg, P0, tot);
        c.check();
        launch(c, k_segscan<u64>, 1, 1024, 0, (const Seg*)seg, (const u32*)nseg, P0, tot, (const u64*)sk, 0u,
               0xffffffffu, fit, nfit, fit_cap, (Bucket*)nullptr, (u32*)nullptr, 0u,
               p > 1 ? (f > 1 ? int_counts : counts) : (u64*)nullptr, c.status);
        c.check();
        c.mark(3);
        // a7: whole records to their bucket positions (buffer 1)
        const size_t sm_s = 4 * (size_t)P0 + 16;
        smem_limit(k_scatter_s32, sm_s, c.di);
        launch(c, k_scatter_s32, nchunk, S32_NT, sm_s, (const u64*)recs, buf1, (const Chunk*)chunks,
               (const u32*)nchunks, (const Seg*)seg, P0, (const u32*)hist, (const u32*)tot, (const u16*)bid);
        c.check();
        c.mark(4);
        // a8: every bucket sorted by the full key into the caller's array
        const size_t sm_b = 36 * (size_t)cap + 64;
        smem_limit(k_bucket_sort_s32, sm_b, c.di);
        launch(c, k_bucket_sort_s32, (u32)c.di.sms, S32_BS_NT, sm_b, (const Bucket*)fit, (const u32*)nfit, nfit + 1,
               (const u64*)buf1, recs, cap, gidx);
        c.check();
        if (pc == 1 && p > 1) {  // internal buckets of a plain sort: one count
            launch(c, k_fold_counts, 1, 32, 0, (const u64*)(f > 1 ? int_counts : counts), P0, 1u, counts);
            c.check();
        } else if (p > 1 && f > 1) {
            launch(c, k_fold_counts, cdiv(p, 256), 256, 0, (const u64*)int_counts, f, p, counts);
            c.check();
        }
        c.mark(5);
    }
};

// ------------------------------------------------------------------ parameter validation
inline int validate_impl(size_t n, int dtype, const ovs_params* prm) {
    if (!prm) return OVS_EINVAL;
    if (dtype != OVS_U32 && dtype != OVS_I32 && dtype != OVS_F64 && dtype != OVS_S32) return OVS_EDTYPE;
    if (dtype == OVS_S32 && prm->method != OVS_ROS) return OVS_EDTYPE;  // strings: ROS (f3)
    if (prm->p == 0) return OVS_EINVAL;
    // positions are u32 counted from a 32-byte-aligned base (the write-combining scatter adds up
    // to 7 slots): n + 32 must stay below 2^32
    if (n >= 0xffffffffull - 32) return OVS_EINVAL;
    if (prm->method != OVS_ROS && prm->method != OVS_DRO) return OVS_EINVAL;
    if (prm->flags & ~(OVS_DRO_PADDED_POSITIONS | OVS_DRO_MERGE)) return OVS_EINVAL;
    if (n == 0 || prm->p == 1) return OVS_OK;
    if (prm->method == OVS_ROS) {
        if (prm->s == 0) return OVS_ESAMPLE;
        if ((uint64_t)prm->p * prm->s - 1 > n) return OVS_ESAMPLE;
    } else {
        if (prm->s == 0) return OVS_ESAMPLE;
        if ((uint64_t)prm->s * prm->p > n / prm->p) return OVS_ESAMPLE;
    }
    return OVS_OK;
}

// ordered bits -> the caller's dtype on the host (the report's splitter keys)
template <int DT> inline typename Codec<DT>::U host_raw(typename Codec<DT>::U o) {
    if constexpr (DT == DT_I32) return (typename Codec<DT>::U)(o ^ 0x80000000u);
    else if constexpr (DT == DT_F64) return (typename Codec<DT>::U)((o >> 63) ? (o & 0x7fffffffffffffffull) : ~o);
    else return o;
}

struct Out {
    void* sk = nullptr;    // device U[p-1]
    u32* st = nullptr;     // device u32[p-1]
    u64* counts = nullptr; // device u64[p]
    size_t ws = 0;
};


// ------------------------------------------------------------------ DRO contract sort (SqDet)
// Algorithm 1 on the device: (a9) the p sequences are sorted stably by the
// bucket sorter into buffer 1; (a10) rp regular samples per sequence; (a11) the rp^2 samples
// are sorted; (a12) S[q] = T[(q+1)rp - 1]; (a13) every splitter is binary-searched into every
// sorted sequence; (a14) bucket j gathers its runs X_{k,j} in k order and is sorted (instead
// of the paper's p-way merge; the result is the same stable order).
template <int DT, bool KV> struct DroSort {
    typedef typename Codec<DT>::U U;
    Ctx& c;
    Engine<DT, KV> e;
    typename Engine<DT, KV>::Lists l1, l2;
    u32 n, p, r, s, ns, flags;
    u64* counts = nullptr;
    U* sk = nullptr;
    u32* st = nullptr;
    u64* t_pack = nullptr; u64* t_key = nullptr; u32* t_tag = nullptr;
    InternalSort<false>* ts32 = nullptr;
    InternalSort<true>* ts64 = nullptr;
    SampleMerge* smg = nullptr;
    const u64* fin_pack = nullptr; const u64* fin_key = nullptr; const u32* fin_tag = nullptr;  // sorted T
    u32* bound = nullptr; u32* cnt = nullptr; u32* tot = nullptr; u32* nseg = nullptr;
    Seg* seg = nullptr;
    // sequences and buckets of n/p keys far over the on-chip capacity: level 1 re-splits them
    // with the whole GPU before the bucket sorter (instead of one CTA re-splitting each)
    bool big = false;
    Level1<DT, KV>* l1x = nullptr;
    typename Engine<DT, KV>::Lists lb;
    // f2 (OVS_DRO_MERGE): step 5 as an on-chip p-way merge over P = p*f fine buckets
    bool merge = false;  // OVS_DRO_MERGE flag (include/ovs.h)
    u32 f = 1, P = 0, mcap = 0;
    U* fsk = nullptr; u32* fst = nullptr; u64* fcounts = nullptr;
    typename Engine<DT, KV>::Lists lfine, lbig;

    DroSort(Ctx& ctx, U* keys, u32* vals, u32 n_, u32 p_, u32 r_, u32 flags_)
        : c(ctx), e(ctx), n(n_), p(p_), r(r_), flags(flags_) {
        merge = (flags & OVS_DRO_MERGE) != 0;
        e.n = n;
        e.ixbits = bits_for(n);
        e.cap = bucket_cap<U, KV>(c.di);
        e.B.k[0] = keys;
        e.B.v[0] = vals;
        e.B.k[1] = c.take<U>(n);
        e.B.v[1] = KV ? c.take<u32>(n) : nullptr;
        e.B.i[0] = KV ? c.take<u32>(n) : nullptr;
        e.B.i[1] = KV ? c.take<u32>(n) : nullptr;
        s = r * p;
        ns = s * p;
        counts = c.take<u64>(p);
        sk = c.take<U>(p);
        st = c.take<u32>(p);
        // (the sample of sorted runs is sorted by the generic internal sort; the ROS coarse-bucket
        // selector measured slower here: its buckets of ~n/(128 r p) records overflow the chip)
        if (sizeof(U) == 4) t_pack = c.take<u64>(ns);
        else { t_key = c.take<u64>(ns); t_tag = c.take<u32>(ns); }
        if (sample_sorted(c.di, ns, sizeof(U) == 8)) {
            if (sizeof(U) == 4) ts32 = new InternalSort<false>(c, ns, t_pack, nullptr);
            else ts64 = new InternalSort<true>(c, ns, t_key, t_tag);
        } else {
            smg = new SampleMerge(c, ns, s, sizeof(U) == 4 ? t_pack : t_key, t_tag, sizeof(U) == 8);
        }
        if (merge) {
            // merge capacity (items in shared memory, two buffers) and the refinement f: the
            // smallest power of two whose worst-case fine bucket fits it, by the tight count of the
            // Lemma 1 proof (reading Q10): ceil(s/f) sample segments of x keys plus x - 1 keys of
            // every other sequence, x = ceil(ceil(n/p)/s)
            const size_t item = merge_item_bytes<U, KV>();
            const size_t fixed = merge_smem_bytes<U, KV>(0, p) + 2 * 16;
            mcap = (u32)(((size_t)c.di.smem_optin - 1024 - fixed) / (2 * item)) & ~15u;
            const u64 x = ((n + p - 1) / p + s - 1) / s;
            auto worst = [&](u64 ff) { return ((s + ff - 1) / ff) * x + (u64)(p - 1) * (x > 0 ? x - 1 : 0); };
            while (2 * f <= s && f < 4096 && worst(f) > mcap) f *= 2;  // f <= s: every fine splitter is a sample
            P = p * f;
            fsk = c.take<U>(P);
            fst = c.take<u32>(P);
            fcounts = c.take<u64>(P);
            e.carve_lists(lfine, P);
            e.carve_lists(lbig, P);
        } else {
            P = p;
        }
        bound = c.take<u32>((size_t)p * (P + 1));
        cnt = c.take<u32>((size_t)p * P);
        tot = c.take<u32>(P + 1);
        seg = c.take<Seg>(1);
        nseg = c.take<u32>(2);
        e.carve_lists(l1, p);
        e.carve_lists(l2, p);
        big = (n / p) > BS_WMAX * e.cap;
        if (big) {
            l1x = new Level1<DT, KV>(e, p);
            e.carve_lists(lb, p * Level1<DT, KV>::PS);
        }
    }
    ~DroSort() { delete ts32; delete ts64; delete smg; delete l1x; }

    // f2: a13 against the P - 1 fine splitters, then a14 as an on-chip p-way merge per fine
    // bucket (k_dro_merge); fine buckets over the merge capacity: gather + bucket sorter
    void run_merge() {
        Bufs<U>& B = e.B;
        launch(c, k_dro_bounds<U>, cdiv((u64)p * (P + 1), 256), 256, 0, B.k[1], n, p, P, (const U*)fsk, (const u32*)fst,
               bound, 0u);
        c.check();
        launch(c, k_dro_counts, cdiv((u64)p * P, 256), 256, 0, (const u32*)bound, p, P, cnt);
        c.check();
        launch(c, k_dro_seg<U>, 1, 1024, 0, B.k[1], n, p, P, (const U*)fsk, 0u, seg, nseg);
        c.check();
        launch(c, k_colscan, std::min<u32>(cdiv(P, 32), 4 * c.di.sms), 1024, 0, cnt, seg, nseg, P, tot);
        c.check();
        fill_u32(c, lfine.nfit, 0, 2);
        fill_u32(c, lbig.nfit, 0, 2);
        launch(c, k_segscan<U>, 1, 1024, 0, seg, nseg, P, tot, (const U*)fsk, 0u, mcap, lfine.fit, lfine.nfit,
               lfine.fit_cap, lbig.fit, lbig.nfit, lbig.fit_cap, fcounts, c.status);
        c.check();
        launch(c, k_fold_counts, cdiv(p, 256), 256, 0, (const u64*)fcounts, f, p, counts);
        c.check();
        c.mark(3);
        const size_t sm = merge_smem_bytes<U, KV>(mcap, p);
        smem_limit(k_dro_merge<DT, KV>, sm, c.di);
        launch(c, k_dro_merge<DT, KV>, (u32)c.di.sms, MG_NT, sm, B, n, p, P, (const u32*)bound, (const u32*)cnt,
               (const u32*)tot, mcap);
        c.check();
        // fine buckets over the merge capacity (rare): gathered into place, then the bucket sorter
        launch(c, k_dro_gather_big<U, KV>, 4 * (u32)c.di.sms, 256, 0, B, n, p, P, (const u32*)bound, (const u32*)cnt,
               (const u32*)tot, (const Bucket*)lbig.fit, (const u32*)lbig.nfit);
        c.check();
        c.mark(4);
        e.bucket_sort(lbig, 0x5e9u);
    }
    // sort the buckets of list l (all far over capacity) through level 1
    void sort_big(typename Engine<DT, KV>::Lists& l, u64 seed, U* okeys, u32* ovals, u32* oidx, bool out_raw) {
        fill_u32(c, lb.nfit, 0, 2);
        l1x->run(l.fit, l.nfit, lb, seed);
        e.bucket_sort(lb, seed, okeys, ovals, oidx, out_raw);
    }

    void run() {
        if (c.dry) return;
        Bufs<U>& B = e.B;
        c.mark(0);
        // a9: BaselineSorting of the p sequences -> buffer 1 (ordered keys, values, indices)
        fill_u32(c, l1.nfit, 0, 2);
        launch(c, k_dro_segments, cdiv(p, 256), 256, 0, l1.fit, l1.nfit, n, p);
        c.check();
        if (big) {
            // ordered keys (+ values, indices) in buffer 1, sequences re-split 1 -> 0, sorted -> 1
            launch(c, k_to_ordered<DT, KV>, 4 * c.di.sms, 1024, 0, B, n);
            c.check();
            launch(c, k_list_flip, cdiv(p, 256), 256, 0, l1.fit, l1.nfit);
            c.check();
            sort_big(l1, 0x5e9u, B.k[1], KV ? B.v[1] : nullptr, KV ? B.i[1] : nullptr, false);
        } else {
            e.bucket_sort(l1, 0x5e9u, B.k[1], KV ? B.v[1] : nullptr, KV ? B.i[1] : nullptr, false);
        }
        c.mark(1);
        // a10-a12: regular sample, sample sort, splitters
        launch(c, k_dro_sample<U>, cdiv((u64)ns, 256), 256, 0, B.k[1], n, p, s, flags & OVS_DRO_PADDED_POSITIONS,
                                                             t_pack, t_key, t_tag);
        c.check();
        fin_pack = t_pack; fin_key = t_key; fin_tag = t_tag;
        if (smg) {
            const int b = smg->run();
            if (sizeof(U) == 4) fin_pack = smg->k[b];
            else { fin_key = smg->k[b]; fin_tag = smg->t[b]; }
        } else if (ts32) ts32->run(0xd0d0);
        else ts64->run(0xd0d0);
        launch(c, k_pick_splitters<U>, cdiv(p, 256), 256, 0, fin_pack, fin_key, fin_tag, p, s, 1u, sk, st);
        c.check();
        if (merge) {
            // fine splitters T[floor((i+1) s / f) - 1]: the contract's S[q] is fine splitter (q+1)f - 1
            launch(c, k_pick_splitters<U>, cdiv(P, 256), 256, 0, fin_pack, fin_key, fin_tag, P, s, f, fsk, fst);
            c.check();
            c.mark(2);
            run_merge();
            c.mark(5);
            return;
        }
        c.mark(2);
        // a13: split every sorted sequence by binary search; bucket starts and run offsets
        launch(c, k_dro_bounds<U>, cdiv((u64)p * (p + 1), 256), 256, 0, B.k[1], n, p, p, sk, st, bound, 0u);
        c.check();
        launch(c, k_dro_counts, cdiv((u64)p * p, 256), 256, 0, bound, p, p, cnt);
        c.check();
        launch(c, k_dro_seg<U>, 1, 1024, 0, B.k[1], n, p, p, sk, 0, seg, nseg);
        c.check();
        launch(c, k_colscan, std::min<u32>(cdiv(p, 32), 4 * c.di.sms), 1024, 0, cnt, seg, nseg, p, tot);
        c.check();
        fill_u32(c, l2.nfit, 0, 2);
        launch(c, k_segscan<U>, 1, 1024, 0, seg, nseg, p, tot, sk, 0, e.cap, l2.fit, l2.nfit, l2.fit_cap, nullptr,
                                          nullptr, 0, counts, c.status);
        c.check();
        c.mark(3);
        // a14: gather the runs X_{k,j} of every bucket (k order) into buffer 0, sort each bucket
        launch(c, k_dro_gather<U, KV>, cdiv((u64)p * p * 32, 256), 256, 0, B, n, p, bound, cnt, tot);
        c.check();
        c.mark(4);
        if (big) {
            sort_big(l2, 0x5e9u, B.k[0], KV ? B.v[0] : nullptr, nullptr, true);
        } else if (n / p > e.cap) {
            // buckets mostly over the on-chip capacity: sorted out of place into the free buffer 1
            // (so they can be sorted in windows instead of re-split by their CTA), then copied back
            e.bucket_sort(l2, 0x5e9u, B.k[1], KV ? B.v[1] : nullptr, nullptr, true);
            OVS_CK(cudaMemcpyAsync(B.k[0], B.k[1], n * sizeof(U), cudaMemcpyDeviceToDevice, c.st));
            if (KV) OVS_CK(cudaMemcpyAsync(B.v[0], B.v[1], n * sizeof(u32), cudaMemcpyDeviceToDevice, c.st));
        } else {
            e.bucket_sort(l2, 0x5e9u);
        }
        c.mark(5);
    }
};

// ------------------------------------------------------------------ multi-GPU
// One rank's distributed ROS sort, in phases that ovs_dist.cu runs with barriers between them
// (the paper's multi-core split, with GPUs in place of cores):
//   sample   every rank draws the same global index set over n_global keys (a1) and stores the
//            records of its own shard into slot `rank` of EVERY rank's window (NVLink stores)
//   select   records -> sample sort -> splitters (a3-a4, identical on every rank)
//   count    classify + histogram of the local shard (a5-a6, tags = global indices); the bucket
//            counts -> row `rank` of the count matrix in every rank's window
//   scatter  (after the host plan) every key straight into its owner's window (a7 fused with the
//            exchange: bucket j lives on rank floor(j*world/p), p a multiple of world)
//   finish   the owned buckets (runs in source-rank order, so the order of equal keys is the
//            global index order) are sorted from the window into the caller's output (a8)
// Window layout (every rank the same; byte offsets): the sample records, the count matrix, then
// the received keys (+ values + original indices).
struct WinLayout {
    size_t rec = 0, C = 0, rk = 0, rv = 0, ri = 0, end = 0;
    u64 cap = 0;  // received items that fit
};
inline WinLayout win_layout(size_t win_bytes, u64 m, u32 kb, bool kv, u32 world, u32 p) {
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    WinLayout L;
    size_t o = 0;
    L.rec = o; o = al(o + 8 * (size_t)m * (kb == 8 ? 2 : 1));
    L.C = o; o = al(o + 4 * (size_t)world * p);
    const size_t per = kb + (kv ? 8 : 0);
    const size_t rem = win_bytes > o + 3 * 256 ? win_bytes - o - 3 * 256 : 0;
    L.cap = std::min<u64>(rem / per, 0xffffffffull - 64);
    L.rk = o; o = al(o + kb * L.cap);
    L.rv = o; o = kv ? al(o + 4 * L.cap) : o;
    L.ri = o; o = kv ? al(o + 4 * L.cap) : o;
    L.end = o;
    return L;
}
// the host part of the exchange plan (also exported as ovs_dist_plan for the CPU tests):
// dst_off[b] = where this rank's run of bucket b starts inside owner(b)'s receive region,
// desc = (begin, length, global id) of every non-empty owned bucket, recv[r] = items rank r gets
struct DistPlanHost {
    std::vector<u32> dst_off, desc;
    std::vector<u64> recv;
};
inline void dist_plan_host(const u32* C, u32 world, u32 p, u32 rank, DistPlanHost& P) {
    P.dst_off.assign(p, 0);
    P.desc.clear();
    P.recv.assign(world, 0);
    std::vector<u64> tot(p, 0);
    for (u32 g = 0; g < world; ++g)
        for (u32 b = 0; b < p; ++b) tot[b] += C[(size_t)g * p + b];
    for (u32 d = 0; d < world; ++d) {
        const u32 b0 = (u32)((u64)d * p / world), b1 = (u32)((u64)(d + 1) * p / world);
        u64 run = 0;
        for (u32 b = b0; b < b1; ++b) {
            u64 before = 0;
            for (u32 g = 0; g < rank; ++g) before += C[(size_t)g * p + b];
            P.dst_off[b] = (u32)(run + before);
            if (d == rank && tot[b] > 0) { P.desc.push_back((u32)run); P.desc.push_back((u32)tot[b]); P.desc.push_back(b); }
            run += tot[b];
        }
        P.recv[d] = run;
    }
}

struct DistCfg {
    const void* keys; const u32* vals; u64 n_local, n_global, offset;
    u32 p, s, world, rank; u64 seed;
    u32 method, flags;  // OVS_ROS / OVS_DRO (s = r for DRO), OVS_DRO_PADDED_POSITIONS
    u64 out_cap;  // output items (d_out) the caller provides
    WinLayout W;
    void* out_k; u32* out_v;
};

struct DistRun {
    virtual ~DistRun() {}
    virtual void sample(char* const* d_peer) = 0;            // records -> every window
    virtual void select(const char* win) = 0;                // this rank's window
    virtual void count(char* const* d_peer) = 0;             // counts -> every window
    virtual void scatter(char* const* d_peer, const DistPlanHost& P, u32* h_stage) = 0;
    virtual void finish(const char* win, u32 n_owned) = 0;   // owned buckets -> out
    virtual void splitters(void* h_keys, uint64_t* h_tags) = 0;  // raw dtype (after select)
    virtual size_t ws() const = 0;
};

template <int DT, bool KV> struct DistSort : DistRun {
    typedef typename Codec<DT>::U U;
    Ctx& c;
    DistCfg g;
    Engine<DT, KV> e;   // local partition: buffer 0 = the local shard (read only)
    Engine<DT, KV> f;   // receive side: buffer 1 = the window's received items, buffer 0 = the output
    typename Engine<DT, KV>::Level0 z;
    typename Engine<DT, KV>::Lists l, lf, lb;
    u32 m = 0;
    u64* counts64 = nullptr;
    u32* dst_off = nullptr;   // p (device)
    u32* desc = nullptr;      // 3p (device)
    RosSampler<DT, true>* smp = nullptr;
    Level1<DT, KV>* l1x = nullptr;

    DistSort(Ctx& ctx, const DistCfg& cfg) : c(ctx), g(cfg), e(ctx), f(ctx) {
        const u32 nl = (u32)g.n_local, p = g.p;
        m = p * g.s - 1;
        e.n = nl;
        e.cap = bucket_cap<U, KV>(c.di);
        e.tag_base = (u32)g.offset;
        e.B.k[0] = (U*)g.keys;  // read only: the fused scatter writes to the windows
        e.B.v[0] = (u32*)g.vals;
        e.B.k[1] = nullptr; e.B.v[1] = nullptr; e.B.i[0] = nullptr; e.B.i[1] = nullptr;
        counts64 = c.take<u64>(p);
        dst_off = c.take<u32>(p);
        desc = c.take<u32>(3 * (size_t)p);
        smp = new RosSampler<DT, true>(c, g.n_global, p, g.s);
        e.carve_level0(z, p);
        e.carve_lists(l, p);
        // receive side: items in the window (buffer 1), output in buffer 0
        const u32 oc = (u32)std::min<u64>(g.out_cap, 0xffffffffull - 64);
        f.n = oc;
        f.cap = e.cap;
        f.ixbits = bits_for(g.n_global);
        f.B.k[0] = (U*)g.out_k;
        f.B.v[0] = g.out_v;
        f.B.k[1] = nullptr; f.B.v[1] = nullptr; f.B.i[1] = nullptr;
        f.B.i[0] = KV ? c.take<u32>(oc) : nullptr;  // level-1 scratch of the original indices
        f.carve_lists(lf, p);
        // owned buckets (n_global/p keys) over the on-chip capacity: one GPU-wide level-1 re-split (measured
        // on emulated ranks: far faster than sorting 1.4-4x-capacity buckets in windows)
        if (g.n_global / p > f.cap) {
            l1x = new Level1<DT, KV>(f, p / g.world + 1);
            f.carve_lists(lb, (p / g.world + 1) * Level1<DT, KV>::PS);
        }
    }
    ~DistSort() { delete smp; delete l1x; }
    size_t ws() const override { return c.off + 256; }

    void sample(char* const* d_peer) override {
        if (c.dry) return;
        smp->draw(g.seed);
        smp->take(g.seed, (const U*)g.keys, g.offset, (u32)g.n_local, PeerOut{d_peer, g.W.rec, g.world});
    }
    void select(const char* win) override {
        if (c.dry) return;
        const u32 words = sizeof(U) == 4 ? 1 : 2;
        launch(c, k_dist_unpack, cdiv(m, 256), 256, 0, (const u64*)(win + g.W.rec), m, words, smp->tk, smp->tk, smp->tt);
        c.check();
        OVS_CK(cudaMemsetAsync(smp->sel->gcnt, 0, 8 * SEL_GMAX, c.st));
        smp->select(g.p, g.s, 1, g.seed ^ 0x5eed, z.sk, z.st);
    }
    void count(char* const* d_peer) override {
        if (c.dry) return;
        e.level0_hist(z, l, counts64);
        launch(c, k_put_counts, cdiv(g.p * g.world, 256), 256, 0, (const u64*)counts64, g.p, g.rank,
               PeerOut{d_peer, g.W.C, g.world});
        c.check();
    }
    void scatter(char* const* d_peer, const DistPlanHost& P, u32* h_stage) override {
        if (c.dry) return;
        // the plan: dst_off (p) and the owned-bucket descriptors, staged in pinned host memory
        std::memcpy(h_stage, P.dst_off.data(), 4 * (size_t)g.p);
        if (!P.desc.empty()) std::memcpy(h_stage + g.p, P.desc.data(), 4 * P.desc.size());
        OVS_CK(cudaMemcpyAsync(dst_off, h_stage, 4 * (size_t)g.p, cudaMemcpyHostToDevice, c.st));
        if (!P.desc.empty())
            OVS_CK(cudaMemcpyAsync(desc, h_stage + g.p, 4 * P.desc.size(), cudaMemcpyHostToDevice, c.st));
        e.template level0_scatter<true>(z, dst_off, PeerOut{d_peer, g.W.rk, g.world}, g.W.rv, g.W.ri);
    }
    void finish(const char* win, u32 n_owned) override {
        if (c.dry) return;
        f.B.k[1] = (U*)(win + g.W.rk);
        f.B.v[1] = KV ? (u32*)(win + g.W.rv) : nullptr;
        f.B.i[1] = KV ? (u32*)(win + g.W.ri) : nullptr;
        launch(c, k_dist_list<U>, std::max<u32>(1, cdiv(n_owned, 256)), 256, 0, (const u32*)desc, n_owned,
               (const U*)z.sk, g.p, lf.fit, lf.nfit, 1u);
        c.check();
        fill_u32(c, lf.ticket, 0, 1);
        if (l1x) {
            fill_u32(c, lb.nfit, 0, 2);
            l1x->run(lf.fit, lf.nfit, lb, g.seed ^ 0xf2);
            f.bucket_sort(lb, g.seed ^ 0xf1);
        } else {
            f.bucket_sort(lf, g.seed ^ 0xf1);
        }
    }
    void splitters(void* h_keys, uint64_t* h_tags) override {
        if (c.dry || g.p < 2) return;
        std::vector<U> kb(g.p - 1);
        std::vector<u32> tb(g.p - 1);
        OVS_CK(cudaMemcpyAsync(kb.data(), z.sk, sizeof(U) * (g.p - 1), cudaMemcpyDeviceToHost, c.st));
        OVS_CK(cudaMemcpyAsync(tb.data(), z.st, 4 * (size_t)(g.p - 1), cudaMemcpyDeviceToHost, c.st));
        OVS_CK(cudaStreamSynchronize(c.st));
        for (u32 q = 0; q + 1 < g.p; ++q) {
            if (h_keys) ((U*)h_keys)[q] = host_raw<DT>(kb[q]);
            if (h_tags) h_tags[q] = tb[q];
        }
    }
};

template <int DT, bool KV>
Out plan_or_run(Ctx& c, void* keys, u32* vals, size_t n, const ovs_params* prm) {
    typedef typename Codec<DT>::U U;
    if (prm->method == OVS_DRO && prm->p > 1) {
        DroSort<DT, KV> d(c, (U*)keys, vals, (u32)n, prm->p, prm->s, prm->flags);
        Out o;
        o.sk = d.sk;
        o.st = d.st;
        o.counts = d.counts;
        if (!c.dry) d.run();
        o.ws = c.off + 256;
        return o;
    }
    RosSort<DT, KV> r(c, (U*)keys, vals, (u32)n, prm->p, prm->s, prm->seed);
    if (prm->p > 1 && r.z.P > r.e.max_p_one_level())
        throw StatusFail{OVS_EINVAL, "p too large for the one-level classifier in shared memory"};
    Out o;
    o.sk = r.f > 1 ? r.rep_sk : r.z.sk;
    o.st = r.f > 1 ? r.rep_st : r.z.st;
    o.counts = r.counts;
    if (!c.dry) r.run();
    o.ws = c.off + 256;
    return o;
}


// ---- DRO across GPUs (SURVEY.md §8(e) DRO steps 1-6; the paper's McDet): rank g owns the
// p/G whole sequences [g p/G, (g+1) p/G) of Algorithm 1's baseline split (equal shards and p | n_global,
// so every sequence is local).  Phases, as DistSort's:
//   sample   a9: sort the local sequences (tags = global positions); a10: their r p regular samples
//            (global s = r p per sequence) -> every rank's window, rank g's block of slots
//   select   a11-a12: sort all r p^2 records, S[q] = T[(q+1) r p - 1] (identical on every rank)
//   count    a13: split the local sequences, column prefix over them, bucket totals -> every window
//   scatter  a14's exchange: every run X_{k,j} straight into the owner of bucket j (k_dro_send)
//   finish   every owned bucket (runs in global sequence order) sorted into the output by (key,
//            original index) - the stable result of the paper's p-way merge
template <int DT, bool KV> struct DistDroSort : DistRun {
    typedef typename Codec<DT>::U U;
    Ctx& c;
    DistCfg g;
    Engine<DT, KV> e;   // local: buffer 0 = the shard (raw, read only), buffer 1 = sorted sequences
    Engine<DT, KV> f;   // receive side (as DistSort)
    typename Engine<DT, KV>::Lists l1, lb1, lf, lb;
    u32 pl = 1, r = 1, s = 1, ns = 0;   // local sequences, r, s = r p, records r p^2
    u64* t_pack = nullptr; u64* t_key = nullptr; u32* t_tag = nullptr;
    InternalSort<false>* ts32 = nullptr;
    InternalSort<true>* ts64 = nullptr;
    SampleMerge* smg = nullptr;
    const u64* fin_pack = nullptr; const u64* fin_key = nullptr; const u32* fin_tag = nullptr;  // sorted T
    U* sk = nullptr; u32* st = nullptr;
    u32* bound = nullptr; u32* cnt = nullptr; u32* tot = nullptr; u32* nseg = nullptr; Seg* seg = nullptr;
    u32* dst_off = nullptr; u32* desc = nullptr;
    bool big = false;
    Level1<DT, KV>* l1s = nullptr;   // local sequences far over capacity
    Level1<DT, KV>* l1x = nullptr;   // owned buckets over capacity
    DistDroSort(Ctx& ctx, const DistCfg& cfg) : c(ctx), g(cfg), e(ctx), f(ctx) {
        const u32 nl = (u32)g.n_local, p = g.p;
        pl = p / g.world;
        r = g.s;
        s = r * p;
        ns = s * p;
        e.n = nl;
        e.ixbits = bits_for(g.n_global);
        e.cap = bucket_cap<U, KV>(c.di);
        e.B.k[0] = (U*)g.keys;
        e.B.v[0] = (u32*)g.vals;
        e.B.k[1] = c.take<U>(nl);
        e.B.v[1] = KV ? c.take<u32>(nl) : nullptr;
        e.B.i[0] = KV ? c.take<u32>(nl) : nullptr;
        e.B.i[1] = KV ? c.take<u32>(nl) : nullptr;
        sk = c.take<U>(p);
        st = c.take<u32>(p);
        if (sizeof(U) == 4) t_pack = c.take<u64>(ns);
        else { t_key = c.take<u64>(ns); t_tag = c.take<u32>(ns); }
        if (sample_sorted(c.di, ns, sizeof(U) == 8)) {
            if (sizeof(U) == 4) ts32 = new InternalSort<false>(c, ns, t_pack, nullptr);
            else ts64 = new InternalSort<true>(c, ns, t_key, t_tag);
        } else {
            smg = new SampleMerge(c, ns, s, sizeof(U) == 4 ? t_pack : t_key, t_tag, sizeof(U) == 8);
        }
        bound = c.take<u32>((size_t)pl * (p + 1));
        cnt = c.take<u32>((size_t)pl * p);
        tot = c.take<u32>(p + 1);
        seg = c.take<Seg>(1);
        nseg = c.take<u32>(2);
        dst_off = c.take<u32>(p);
        desc = c.take<u32>(3 * (size_t)p);
        e.carve_lists(l1, pl);
        big = (nl / std::max<u32>(pl, 1)) > BS_WMAX * e.cap;
        if (big) {
            l1s = new Level1<DT, KV>(e, pl);
            e.carve_lists(lb1, pl * Level1<DT, KV>::PS);
        }
        // receive side
        const u32 oc = (u32)std::min<u64>(g.out_cap, 0xffffffffull - 64);
        f.n = oc;
        f.cap = e.cap;
        f.ixbits = bits_for(g.n_global);
        f.B.k[0] = (U*)g.out_k;
        f.B.v[0] = g.out_v;
        f.B.k[1] = nullptr; f.B.v[1] = nullptr; f.B.i[1] = nullptr;
        f.B.i[0] = KV ? c.take<u32>(oc) : nullptr;
        f.carve_lists(lf, p);
        if (g.n_global / p > f.cap) {
            l1x = new Level1<DT, KV>(f, p / g.world + 1);
            f.carve_lists(lb, (p / g.world + 1) * Level1<DT, KV>::PS);
        }
    }
    ~DistDroSort() { delete ts32; delete ts64; delete smg; delete l1s; delete l1x; }
    size_t ws() const override { return c.off + 256; }

    void sample(char* const* d_peer) override {
        if (c.dry) return;
        Bufs<U>& B = e.B;
        const u32 nl = (u32)g.n_local;
        // a9: the local sequences sorted into buffer 1 (ordered keys; values, original indices)
        fill_u32(c, l1.nfit, 0, 2);
        launch(c, k_dro_segments, cdiv(pl, 256), 256, 0, l1.fit, l1.nfit, nl, pl);
        c.check();
        if (big) {
            launch(c, k_to_ordered<DT, KV>, 4 * c.di.sms, 1024, 0, B, nl);
            c.check();
            launch(c, k_list_flip, cdiv(pl, 256), 256, 0, l1.fit, l1.nfit);
            c.check();
            fill_u32(c, lb1.nfit, 0, 2);
            l1s->run(l1.fit, l1.nfit, lb1, 0x5e9u);
            e.bucket_sort(lb1, 0x5e9u, B.k[1], KV ? B.v[1] : nullptr, KV ? B.i[1] : nullptr, false);
        } else {
            e.bucket_sort(l1, 0x5e9u, B.k[1], KV ? B.v[1] : nullptr, KV ? B.i[1] : nullptr, false);
        }
        if (KV && g.offset) {  // original indices of the shard -> global
            launch(c, k_add_u32, cdiv(nl, 256), 256, 0, B.i[1], nl, (u32)g.offset);
            c.check();
        }
        // a10: regular samples of the local sorted sequences -> every window (slots of this rank)
        const u32 xpad = (u32)((((u64)g.n_global + g.p - 1) / g.p + s - 1) / s);
        launch(c, k_dro_sample_dist<U>, cdiv((u64)s * pl, 256), 256, 0, (const U*)B.k[1], nl, pl, s,
               (u32)((g.flags & OVS_DRO_PADDED_POSITIONS) ? 1 : 0), xpad, (u32)g.offset, g.rank * pl * s,
               PeerOut{d_peer, g.W.rec, g.world});
        c.check();
    }
    void select(const char* win) override {
        if (c.dry) return;
        const u32 words = sizeof(U) == 4 ? 1 : 2;
        launch(c, k_dist_unpack, cdiv(ns, 256), 256, 0, (const u64*)(win + g.W.rec), ns, words, t_pack, t_key, t_tag);
        c.check();
        fin_pack = t_pack; fin_key = t_key; fin_tag = t_tag;
        if (smg) {
            const int b = smg->run();
            if (sizeof(U) == 4) fin_pack = smg->k[b];
            else { fin_key = smg->k[b]; fin_tag = smg->t[b]; }
        } else if (ts32) ts32->run(0xd0d0);
        else ts64->run(0xd0d0);
        launch(c, k_pick_splitters<U>, cdiv(g.p, 256), 256, 0, fin_pack, fin_key, fin_tag,
               g.p, s, 1u, sk, st);
        c.check();
    }
    void count(char* const* d_peer) override {
        if (c.dry) return;
        const u32 nl = (u32)g.n_local, p = g.p;
        launch(c, k_dro_bounds<U>, cdiv((u64)pl * (p + 1), 256), 256, 0, (const U*)e.B.k[1], nl, pl, p, (const U*)sk,
               (const u32*)st, bound, (u32)g.offset);
        c.check();
        launch(c, k_dro_counts, cdiv((u64)pl * p, 256), 256, 0, (const u32*)bound, pl, p, cnt);
        c.check();
        launch(c, k_dro_seg<U>, 1, 1024, 0, (const U*)e.B.k[1], nl, pl, p, (const U*)sk, 0u, seg, nseg);
        c.check();
        launch(c, k_colscan, std::min<u32>(cdiv(p, 32), 4 * c.di.sms), 1024, 0, cnt, (const Seg*)seg,
               (const u32*)nseg, p, tot);
        c.check();
        launch(c, k_put_counts32, cdiv(p * g.world, 256), 256, 0, (const u32*)tot, p, g.rank,
               PeerOut{d_peer, g.W.C, g.world});
        c.check();
    }
    void scatter(char* const* d_peer, const DistPlanHost& P, u32* h_stage) override {
        if (c.dry) return;
        std::memcpy(h_stage, P.dst_off.data(), 4 * (size_t)g.p);
        if (!P.desc.empty()) std::memcpy(h_stage + g.p, P.desc.data(), 4 * P.desc.size());
        OVS_CK(cudaMemcpyAsync(dst_off, h_stage, 4 * (size_t)g.p, cudaMemcpyHostToDevice, c.st));
        if (!P.desc.empty())
            OVS_CK(cudaMemcpyAsync(desc, h_stage + g.p, 4 * P.desc.size(), cudaMemcpyHostToDevice, c.st));
        launch(c, k_dro_send<U, KV>, 8 * (u32)c.di.sms, 256, 0, e.B, (u32)g.n_local, pl, g.p, (const u32*)bound,
               (const u32*)cnt, (const u32*)dst_off, PeerOut{d_peer, g.W.rk, g.world}, g.W.rv, g.W.ri);
        c.check();
    }
    void finish(const char* win, u32 n_owned) override {
        if (c.dry) return;
        f.B.k[1] = (U*)(win + g.W.rk);
        f.B.v[1] = KV ? (u32*)(win + g.W.rv) : nullptr;
        f.B.i[1] = KV ? (u32*)(win + g.W.ri) : nullptr;
        launch(c, k_dist_list<U>, std::max<u32>(1, cdiv(n_owned, 256)), 256, 0, (const u32*)desc, n_owned,
               (const U*)sk, g.p, lf.fit, lf.nfit, 1u);
        c.check();
        fill_u32(c, lf.ticket, 0, 1);
        if (l1x) {
            fill_u32(c, lb.nfit, 0, 2);
            l1x->run(lf.fit, lf.nfit, lb, g.seed ^ 0xf2);
            f.bucket_sort(lb, g.seed ^ 0xf1);
        } else {
            f.bucket_sort(lf, g.seed ^ 0xf1);
        }
    }
    void splitters(void* h_keys, uint64_t* h_tags) override {
        if (c.dry || g.p < 2) return;
        std::vector<U> kb(g.p - 1);
        std::vector<u32> tb(g.p - 1);
        OVS_CK(cudaMemcpyAsync(kb.data(), sk, sizeof(U) * (g.p - 1), cudaMemcpyDeviceToHost, c.st));
        OVS_CK(cudaMemcpyAsync(tb.data(), st, 4 * (size_t)(g.p - 1), cudaMemcpyDeviceToHost, c.st));
        OVS_CK(cudaStreamSynchronize(c.st));
        for (u32 q = 0; q + 1 < g.p; ++q) {
            if (h_keys) ((U*)h_keys)[q] = host_raw<DT>(kb[q]);
            if (h_tags) h_tags[q] = tb[q];
        }
    }
};

// multi-GPU: one rank's distributed sort object (per (dtype, keys/pairs) translation unit)
template <int DT, bool KV> DistRun* make_dist(Ctx& c, const DistCfg& cfg) {
    if (cfg.method == OVS_DRO) return new DistDroSort<DT, KV>(c, cfg);
    return new DistSort<DT, KV>(c, cfg);
}
DistRun* dist_u32_k(Ctx& c, const DistCfg& cfg);
DistRun* dist_u32_v(Ctx& c, const DistCfg& cfg);
DistRun* dist_i32_k(Ctx& c, const DistCfg& cfg);
DistRun* dist_i32_v(Ctx& c, const DistCfg& cfg);
DistRun* dist_f64_k(Ctx& c, const DistCfg& cfg);
DistRun* dist_f64_v(Ctx& c, const DistCfg& cfg);

// per-(dtype, keys/pairs) entry points (ovs_<dtype>_<k|v>.cu)
Out plan_u32_k(Ctx& c, void* keys, u32* vals, size_t n, const ovs_params* prm);
Out plan_u32_v(Ctx& c, void* keys, u32* vals, size_t n, const ovs_params* prm);
Out plan_i32_k(Ctx& c, void* keys, u32* vals, size_t n, const ovs_params* prm);
Out plan_i32_v(Ctx& c, void* keys, u32* vals, size_t n, const ovs_params* prm);
Out plan_f64_k(Ctx& c, void* keys, u32* vals, size_t n, const ovs_params* prm);
Out plan_f64_v(Ctx& c, void* keys, u32* vals, size_t n, const ovs_params* prm);
Out plan_s32_k(Ctx& c, void* keys, u32* vals, size_t n, const ovs_params* prm);
int validate(size_t n, int dtype, const ovs_params* prm);
DevInfo dev_info();
extern thread_local std::string g_err;
extern thread_local std::vector<cudaEvent_t> g_marks;

}  // namespace ovs

