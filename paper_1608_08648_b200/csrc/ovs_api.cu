// ovs_api.cu — the C ABI of include/ovs.h: argument validation, workspace sizing (dry run of
// the same carving code), the enqueue of the sort, and the optional report.
#include "ovs_engine.cuh"

namespace ovs {
thread_local std::string g_err;
thread_local std::vector<cudaEvent_t> g_marks;
DevInfo dev_info() { return dev_info_impl(); }
int validate(size_t n, int dtype, const ovs_params* prm) { return validate_impl(n, dtype, prm); }
}  // namespace ovs

using namespace ovs;

// ------------------------------------------------------------------ C ABI
static Out plan_dispatch(Ctx& c, void* keys, u32* vals, size_t n, int dtype, const ovs_params* prm) {
    const bool kv = vals != nullptr || (c.dry && keys == (void*)1);
    if (dtype == OVS_S32) {
        if (kv) throw StatusFail{OVS_EDTYPE, "32-byte string keys: keys only"};
        return plan_s32_k(c, keys, vals, n, prm);
    }
    if (dtype == OVS_U32) return kv ? plan_u32_v(c, keys, vals, n, prm) : plan_u32_k(c, keys, vals, n, prm);
    if (dtype == OVS_I32) return kv ? plan_i32_v(c, keys, vals, n, prm) : plan_i32_k(c, keys, vals, n, prm);
    return kv ? plan_f64_v(c, keys, vals, n, prm) : plan_f64_k(c, keys, vals, n, prm);
}

static int sort_impl(void* d_keys, uint32_t* d_vals, bool kv, size_t n, int dtype, const ovs_params* prm, void* d_ws,
                     size_t ws_bytes, void* stream, ovs_report* rep) {
    g_err.clear();
    int v = validate(n, dtype, prm);
    if (v != OVS_OK) { g_err = "invalid arguments"; return v; }
    if (n > 0 && (d_keys == nullptr || (kv && d_vals == nullptr))) { g_err = "NULL buffer"; return OVS_EINVAL; }
    try {
        Ctx c;
        c.di = dev_info();
        c.st = (cudaStream_t)stream;
        c.marks = &g_marks;
        if (n == 0) {
            if (rep) {
                std::memset(rep->phase_ms, 0, sizeof(rep->phase_ms));
                if (rep->bucket_counts) for (u32 j = 0; j < prm->p; ++j) rep->bucket_counts[j] = 0;
                rep->max_bucket = 0; rep->kernel_launches = 0; rep->device_status = 0; rep->exchange_bytes = 0;
            }
            return OVS_OK;
        }
        // dry run: size
        Ctx d = c;
        d.dry = true;
        d.take<u32>(4);           // status
        Out od = plan_dispatch(d, kv ? (void*)1 : nullptr, nullptr, n, dtype, prm);
        if (ws_bytes < od.ws || d_ws == nullptr) { g_err = "workspace too small"; return OVS_EWORKSPACE; }
        // real run
        c.dry = false;
        c.ws = (char*)d_ws;
        c.status = c.take<u32>(4);
        // the report's phase events: boundaries 0..5 of Ctx::mark (include/ovs.h)
        struct Evs {
            cudaEvent_t e[OVS_NMARKS] = {};
            ~Evs() { for (auto x : e) if (x) cudaEventDestroy(x); }
        } ev;
        if (rep) {
            for (auto& x : ev.e) {
                OVS_CK(cudaEventCreate(&x));
                OVS_CK(cudaEventRecord(x, c.st));  // a phase a path skips reads as 0 ms
            }
            c.rep_marks = ev.e;
        }
        OVS_CK(cudaMemsetAsync(c.status, 0, 4, c.st));  // this call's bits (status[1] is sticky)
        Out o = plan_dispatch(c, d_keys, kv ? d_vals : nullptr, n, dtype, prm);
        if (rep) {
            OVS_CK(cudaStreamSynchronize(c.st));
            std::memset(rep->phase_ms, 0, sizeof(rep->phase_ms));
            for (u32 k = 0; k + 1 < OVS_NMARKS; ++k) {
                float ms = 0;
                OVS_CK(cudaEventElapsedTime(&ms, ev.e[k], ev.e[k + 1]));
                rep->phase_ms[k] = ms;  // sample, sample_sort, classify_hist, scatter, bucket_sort
            }
            float tot = 0;
            OVS_CK(cudaEventElapsedTime(&tot, ev.e[0], ev.e[OVS_NMARKS - 1]));
            rep->phase_ms[7] = tot;
            u32 stv = 0;
            OVS_CK(cudaMemcpy(&stv, c.status, 4, cudaMemcpyDeviceToHost));
            rep->device_status = stv;
            rep->kernel_launches = c.launches;
            rep->exchange_bytes = 0;
            const u32 p = prm->p;
            std::vector<u64> cnt(p, 0);
            if (p > 1) OVS_CK(cudaMemcpy(cnt.data(), o.counts, 8 * (size_t)p, cudaMemcpyDeviceToHost));
            else cnt[0] = n;
            u64 mx = 0;
            for (u64 x : cnt) mx = std::max(mx, x);
            rep->max_bucket = (u32)mx;
            if (rep->bucket_counts) std::memcpy(rep->bucket_counts, cnt.data(), 8 * (size_t)p);
            if (p > 1 && (rep->splitter_keys || rep->splitter_tags)) {
                const size_t kb = dtype == OVS_S32 ? 32 : dtype == OVS_F64 ? 8 : 4;
                std::vector<unsigned char> kbuf(kb * (p - 1));
                std::vector<u32> tbuf(p - 1);
                OVS_CK(cudaMemcpy(kbuf.data(), o.sk, kb * (p - 1), cudaMemcpyDeviceToHost));
                OVS_CK(cudaMemcpy(tbuf.data(), o.st, 4 * (size_t)(p - 1), cudaMemcpyDeviceToHost));
                if (rep->splitter_keys) {
                    // splitters are held as ordered bits: convert back to the raw dtype
                    if (dtype == OVS_U32 || dtype == OVS_S32) std::memcpy(rep->splitter_keys, kbuf.data(), kbuf.size());
                    else if (dtype == OVS_I32) {
                        u32* d = (u32*)rep->splitter_keys;
                        const u32* s = (const u32*)kbuf.data();
                        for (u32 q = 0; q + 1 < p; ++q) d[q] = s[q] ^ 0x80000000u;
                    } else {
                        u64* d = (u64*)rep->splitter_keys;
                        const u64* s = (const u64*)kbuf.data();
                        for (u32 q = 0; q + 1 < p; ++q)
                            d[q] = (s[q] >> 63) ? (s[q] & 0x7fffffffffffffffull) : ~s[q];
                    }
                }
                if (rep->splitter_tags)
                    for (u32 q = 0; q + 1 < p; ++q) rep->splitter_tags[q] = tbuf[q];
            }
            if (stv != 0) { g_err = "device-side check failed (status bits " + std::to_string(stv) + ")"; return OVS_EINTERNAL; }
        }
        return OVS_OK;
    } catch (const CudaFail& e) {
        g_err = e.what();
        return OVS_ECUDA;
    } catch (const StatusFail& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return OVS_ECUDA;
    } catch (...) {
        g_err = "unknown exception";
        return OVS_ECUDA;
    }
}

// ovs_auto_params: the smallest power-of-two p whose buckets fit on chip with margin
template <class U, bool KV> static u32 auto_p(size_t n, const DevInfo& di) {
    const u64 cap = bucket_cap<U, KV>(di);
    if (n <= cap) return 1;
    const u64 part = cap * 6 / 10;
    u32 pmax = 8192;  // 13-bit classifier entries; keys only: the write-combining scatter's range
    if (!KV) while (pmax > 2 && wc_smem_bytes<U>(pmax) + 512 > (size_t)di.smem_optin) pmax >>= 1;
    else
        while (pmax > 2 && scatter_smem_bytes<U, KV, PartItems<U, KV>::v, PT_NT>(pmax, 64) + 1024 > (size_t)di.smem_optin)
            pmax >>= 1;
    u32 p = 2;
    while ((u64)p < pmax && (n + p - 1) / p > part) p <<= 1;
    return p;
}

extern "C" {

size_t ovs_workspace_bytes(size_t n, int dtype, int with_values, const ovs_params* prm) {
    if (validate(n, dtype, prm) != OVS_OK) return 0;
    if (n == 0) return 0;
    try {
        Ctx d;
        d.di = dev_info();
        d.dry = true;
        d.take<u32>(4);
        Out o = plan_dispatch(d, with_values ? (void*)1 : nullptr, nullptr, n, dtype, prm);
        return o.ws;
    } catch (...) {
        return 0;
    }
}

int ovs_sort_keys(void* d_keys, size_t n, int dtype, const ovs_params* prm, void* d_ws, size_t ws_bytes, void* stream,
                  ovs_report* rep) {
    return sort_impl(d_keys, nullptr, false, n, dtype, prm, d_ws, ws_bytes, stream, rep);
}

int ovs_sort_pairs_stable(void* d_keys, uint32_t* d_vals, size_t n, int dtype, const ovs_params* prm, void* d_ws,
                          size_t ws_bytes, void* stream, ovs_report* rep) {
    return sort_impl(d_keys, d_vals, true, n, dtype, prm, d_ws, ws_bytes, stream, rep);
}

int ovs_device_status(const void* d_ws, void* stream, uint32_t* status, int reset) {
    g_err.clear();
    if (!d_ws) { g_err = "NULL workspace"; return OVS_EINVAL; }
    try {
        u32 w[2] = {0, 0};
        const cudaStream_t st = (cudaStream_t)stream;
        OVS_CK(cudaMemcpyAsync(w, d_ws, 8, cudaMemcpyDeviceToHost, st));
        OVS_CK(cudaStreamSynchronize(st));
        if (reset) OVS_CK(cudaMemsetAsync((char*)d_ws + 4, 0, 4, st));
        if (status) *status = w[1];
        if (w[1] != 0) {
            g_err = "device-side check failed (sticky status bits " + std::to_string(w[1]) + ")";
            return OVS_EINTERNAL;
        }
        return OVS_OK;
    } catch (const CudaFail& e) {
        g_err = e.what();
        return OVS_ECUDA;
    }
}

const char* ovs_last_error(void) { return g_err.c_str(); }

void ovs_set_phase_events(void* const* events, int count) {
    g_marks.assign(count > 0 ? count : 0, nullptr);
    for (int i = 0; i < count; ++i) g_marks[i] = (cudaEvent_t)events[i];
}

const char* ovs_version(void) { return "ovs 0.1 sm_100a"; }

int ovs_auto_params(size_t n, int dtype, int with_values, int method, ovs_params* out) {
    if (!out || (method != OVS_ROS && method != OVS_DRO) || n == 0 || n >= 0xffffffffull) return OVS_EINVAL;
    if (dtype != OVS_U32 && dtype != OVS_I32 && dtype != OVS_F64) return OVS_EDTYPE;
    const DevInfo di = dev_info();
    const bool kv = with_values != 0;
    u32 p = dtype == OVS_F64 ? (kv ? auto_p<u64, true>(n, di) : auto_p<u64, false>(n, di))
                             : (kv ? auto_p<u32, true>(n, di) : auto_p<u32, false>(n, di));
    u32 s = 1;
    if (method == OVS_ROS) {
        s = 64;
        while (p > 1 && s > 1 && (u64)p * s - 1 > n) s >>= 1;
    } else {
        while (p > 1 && (u64)p * p > n) p >>= 1;  // r >= 1 needs r*p <= n/p
        u32 lg = 0;
        while (lg < 32 && (1ull << lg) < n) ++lg;
        const u64 rmax = p > 1 ? n / ((u64)p * p) : 1;
        s = (u32)std::max<u64>(1, std::min<u64>(lg, rmax));
    }
    out->method = (uint32_t)method;
    out->p = p;
    out->s = s;
    out->flags = 0;
    out->seed = 1;
    return OVS_OK;
}

}  // extern "C"
