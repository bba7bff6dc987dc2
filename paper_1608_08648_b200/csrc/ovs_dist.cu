// ovs_dist.cu — the multi-GPU C ABI of include/ovs.h: the NCCL
// communicator, the symmetric receive window every rank writes into over NVLink, the barriers
// between the phases of DistSort (ovs_engine.cuh), the host part of the exchange plan, and the
// single-GPU emulation of several ranks used by the tests.
#include "ovs_engine.cuh"

#include <nccl.h>
#include <nccl_device.h>

#include <cstdlib>

using namespace ovs;

struct ovs_comm {
    int rank = 0, world = 1, device = 0;
    ncclComm_t nccl = nullptr;
    ncclDevComm dev{};
    bool dev_ok = false;
    void* win_buf = nullptr;   // ncclMemAlloc'd, registered as a symmetric window
    size_t win_bytes = 0;
    ncclWindow_t win = nullptr;
    char** d_peer = nullptr;   // device [world]: every rank's window base (NVLink peer mappings)
    u64* d_tmp = nullptr;      // device scratch: the sizes all-gather, the window-size all-reduce
    u64* h_tmp = nullptr;      // pinned host mirror of d_tmp
    u32* h_stage = nullptr;    // pinned: the count matrix read-back and the plan upload
    size_t h_stage_words = 0;
};

namespace ovsd {

#define OVS_NCCK(x)                                                                                \
    do {                                                                                           \
        ncclResult_t r_ = (x);                                                                     \
        if (r_ != ncclSuccess) throw NcclFail(std::string(#x) + ": " + ncclGetErrorString(r_));    \
    } while (0)

struct NcclFail : std::runtime_error {
    explicit NcclFail(const std::string& s) : std::runtime_error(s) {}
};

// every rank's window base as seen from this GPU (ncclGetLsaPointer: the NVLink peer mapping of
// the symmetric window; LSA = load/store accessible, here all ranks of the NVSwitch node)
__global__ void k_peer_ptrs(ncclWindow_t w, char** out, int world) {
    for (int i = threadIdx.x; i < world; i += blockDim.x) out[i] = (char*)ncclGetLsaPointer(w, 0, i);
}

// barrier over all ranks: every rank's earlier work on its stream (including its NVLink stores
// into the others' windows, fenced system-wide by the storing kernels) is visible after it
__global__ void k_lsa_barrier(ncclDevComm dc) {
    ncclLsaBarrierSession<ncclCoopCta> bar{ncclCoopCta(), dc, ncclTeamTagLsa(), 0u};
    bar.sync(ncclCoopCta(), cuda::memory_order_seq_cst);
}

void barrier(ovs_comm* c, cudaStream_t st) {
    if (c->world == 1) return;
    k_lsa_barrier<<<1, 128, 0, st>>>(c->dev);
    OVS_CK(cudaGetLastError());
}

DistRun* make_run(Ctx& c, int dtype, bool kv, const DistCfg& g) {
    if (dtype == OVS_U32) return kv ? dist_u32_v(c, g) : dist_u32_k(c, g);
    if (dtype == OVS_I32) return kv ? dist_i32_v(c, g) : dist_i32_k(c, g);
    return kv ? dist_f64_v(c, g) : dist_f64_k(c, g);
}

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

// parameter checks that need only the call's own arguments
int dist_args(int dtype, const ovs_params* prm, int world) {
    if (!prm) return OVS_EINVAL;
    if (dtype != OVS_U32 && dtype != OVS_I32 && dtype != OVS_F64) return OVS_EDTYPE;
    if (prm->method != OVS_ROS && prm->method != OVS_DRO) return OVS_EINVAL;
    if (prm->flags & ~(u32)OVS_DRO_PADDED_POSITIONS) return OVS_EINVAL;  // (no merge flag across GPUs)
    if (prm->method == OVS_ROS && prm->flags) return OVS_EINVAL;
    if (prm->p < 2 || prm->p % (uint32_t)world != 0) return OVS_EINVAL;  // "p ... a multiple of m"
    if (prm->s == 0) return OVS_ESAMPLE;
    return OVS_OK;
}
// checks on the global size (identical on every rank: the sizes are all-gathered)
int dist_global(u64 n_global, const ovs_params* prm) {
    if (n_global >= 0xffffffffull - 32) return OVS_EINVAL;  // global indices are the u32 tags
    if (prm->method == OVS_DRO) {
        // every rank holds whole sequences of Algorithm 1's baseline split: p | n_global (the shard
        // sizes are checked to be n_global / world by the caller of this), r p <= n / p
        if (n_global % prm->p != 0) return OVS_EINVAL;
        if ((u64)prm->s * prm->p > n_global / prm->p) return OVS_ESAMPLE;
        return OVS_OK;
    }
    if ((u64)prm->p * prm->s - 1 > n_global) return OVS_ESAMPLE;
    return OVS_OK;
}
// sample records in the window: ROS ps - 1, DRO r p^2
u64 rec_count(const ovs_params* prm) {
    return prm->method == OVS_DRO ? (u64)prm->s * prm->p * prm->p : (u64)prm->p * prm->s - 1;
}

DistCfg make_cfg(u64 n_local, u64 n_global, u64 offset, const ovs_params* prm, int world, int rank, u64 out_cap,
                 const WinLayout& W) {
    DistCfg g{};
    g.n_local = n_local; g.n_global = n_global; g.offset = offset;
    g.p = prm->p; g.s = prm->s; g.world = (u32)world; g.rank = (u32)rank; g.seed = prm->seed;
    g.method = prm->method; g.flags = prm->flags;
    g.out_cap = out_cap; g.W = W;
    return g;
}

size_t ws_need(int dtype, bool kv, const DistCfg& g) {
    Ctx d;
    d.di = dev_info();
    d.dry = true;
    d.take<u32>(4);
    std::unique_ptr<DistRun> r(make_run(d, dtype, kv, g));
    return r->ws();
}

void stage(ovs_comm* c, size_t words) {
    if (c->h_stage_words >= words) return;
    if (c->h_stage) cudaFreeHost(c->h_stage);
    c->h_stage = nullptr;
    OVS_CK(cudaMallocHost(&c->h_stage, 4 * words));
    c->h_stage_words = words;
}

// all-gather of (n_local, out_capacity, ws_bytes) of every rank, on the host
void gather_sizes(ovs_comm* c, u64 a, u64 b, u64 w, std::vector<u64>& out, cudaStream_t st) {
    out.assign(3 * (size_t)c->world, 0);
    if (c->world == 1) { out[0] = a; out[1] = b; out[2] = w; return; }
    c->h_tmp[0] = a; c->h_tmp[1] = b; c->h_tmp[2] = w;
    u64* src = c->d_tmp + 3 * (size_t)c->world;
    OVS_CK(cudaMemcpyAsync(src, c->h_tmp, 24, cudaMemcpyHostToDevice, st));
    OVS_NCCK(ncclAllGather(src, c->d_tmp, 3, ncclUint64, c->nccl, st));
    OVS_CK(cudaMemcpyAsync(c->h_tmp, c->d_tmp, 24 * (size_t)c->world, cudaMemcpyDeviceToHost, st));
    OVS_CK(cudaStreamSynchronize(st));
    std::memcpy(out.data(), c->h_tmp, 24 * (size_t)c->world);
}

struct Evs {
    cudaEvent_t e[OVS_NMARKS] = {};
    ~Evs() { for (auto x : e) if (x) cudaEventDestroy(x); }
};

// One rank's distributed sort (see DistSort): sizes all-gather (host sync 1), sample records to
// every window, barrier, splitters, counts to every window, barrier, count matrix read-back
// (host sync 2: the capacity check and the plan), fused scatter into the owners' windows,
// barrier, sort of the owned buckets into the output.  Failures found after the sizes
// all-gather are decided from all-gathered data, so every rank returns the same code.
int dist_impl(ovs_comm* c, const void* keys, const u32* vals, bool kv, size_t n_local, int dtype,
              const ovs_params* prm, void* out_k, u32* out_v, size_t out_cap, size_t* n_out, void* d_ws,
              size_t ws_bytes, void* stream, ovs_report* rep) {
    g_err.clear();
    if (!c) return fail(OVS_EINVAL, "NULL communicator");
    int v = dist_args(dtype, prm, c->world);
    if (v != OVS_OK) return fail(v, "invalid arguments (ROS only, p a multiple of world, s >= 1)");
    if ((n_local > 0 && (!keys || (kv && !vals))) || !n_out) return fail(OVS_EINVAL, "NULL buffer");
    try {
        OVS_CK(cudaSetDevice(c->device));
        const cudaStream_t st = (cudaStream_t)stream;
        std::vector<u64> sz;
        gather_sizes(c, n_local, out_cap, ws_bytes, sz, st);
        const u32 world = (u32)c->world, rank = (u32)c->rank, p = prm->p;
        u64 n_global = 0, offset = 0;
        for (u32 r = 0; r < world; ++r) {
            if (r < rank) offset += sz[3 * r];
            n_global += sz[3 * r];
        }
        v = dist_global(n_global, prm);
        if (v != OVS_OK) return fail(v, "invalid global size or sample size (ps-1 <= n_global < 2^32-33; DRO: p | n)");
        if (prm->method == OVS_DRO)
            for (u32 r = 0; r < world; ++r)
                if (sz[3 * r] != n_global / world)
                    return fail(OVS_EINVAL, "DRO across GPUs: every rank holds n_global / world keys (whole sequences)");
        *n_out = 0;
        if (rep) {
            std::memset(rep->phase_ms, 0, sizeof(rep->phase_ms));
            rep->max_bucket = 0; rep->kernel_launches = 0; rep->device_status = 0;
        }
        const u32 kb = dtype == OVS_F64 ? 8 : 4;
        const u64 m = rec_count(prm);
        const WinLayout W = win_layout(c->win_bytes, m, kb, kv, world, p);
        if (W.end > c->win_bytes || W.cap == 0)
            return fail(OVS_ECAPACITY, "the window cannot hold the sample and the count matrix (ovs_comm_reserve)");
        // every rank's workspace requirement, from the all-gathered sizes (same verdict everywhere)
        for (u32 r = 0; r < world; ++r) {
            u64 off_r = 0;
            for (u32 q = 0; q < r; ++q) off_r += sz[3 * q];
            const size_t need = ws_need(dtype, kv, make_cfg(sz[3 * r], n_global, off_r, prm, c->world, (int)r, sz[3 * r + 1], W));
            if (sz[3 * r + 2] < need || (r == rank && !d_ws))
                return fail(OVS_EWORKSPACE, "workspace too small on rank " + std::to_string(r) + " (" +
                                                std::to_string(sz[3 * r + 2]) + " < " + std::to_string(need) + ")");
        }
        Ctx cx;
        cx.di = dev_info();
        cx.dry = false;
        cx.ws = (char*)d_ws;
        cx.st = st;
        cx.marks = &g_marks;
        Evs ev;
        if (rep) {
            for (auto& x : ev.e) {
                OVS_CK(cudaEventCreate(&x));
                OVS_CK(cudaEventRecord(x, st));
            }
            cx.rep_marks = ev.e;
        }
        cx.status = cx.take<u32>(4);
        DistCfg g = make_cfg(n_local, n_global, offset, prm, c->world, c->rank, out_cap, W);
        g.keys = keys; g.vals = vals; g.out_k = out_k; g.out_v = out_v;
        std::unique_ptr<DistRun> run(make_run(cx, dtype, kv, g));
        OVS_CK(cudaMemsetAsync(cx.status, 0, 4, st));
        char* const win = (char*)c->win_buf;
        cx.mark(0);
        run->sample(c->d_peer);
        barrier(c, st);
        cx.mark(1);
        run->select(win);
        cx.mark(2);
        run->count(c->d_peer);
        barrier(c, st);
        // the count matrix -> host: capacity check and the exchange plan
        stage(c, (size_t)world * p + 4 * (size_t)p + 16);
        OVS_CK(cudaMemcpyAsync(c->h_stage, win + W.C, 4 * (size_t)world * p, cudaMemcpyDeviceToHost, st));
        OVS_CK(cudaStreamSynchronize(st));
        std::vector<u32> C(c->h_stage, c->h_stage + (size_t)world * p);
        cx.mark(3);
        DistPlanHost P;
        dist_plan_host(C.data(), world, p, rank, P);
        *n_out = (size_t)P.recv[rank];
        for (u32 r = 0; r < world; ++r)
            if (P.recv[r] > W.cap || P.recv[r] > sz[3 * r + 1])
                return fail(OVS_ECAPACITY, "rank " + std::to_string(r) + " receives " + std::to_string(P.recv[r]) +
                                               " items: window capacity " + std::to_string(W.cap) + ", output capacity " +
                                               std::to_string(sz[3 * r + 1]));
        run->scatter(c->d_peer, P, c->h_stage);
        barrier(c, st);
        cx.mark(4);
        run->finish(win, (u32)(P.desc.size() / 3));
        cx.mark(5);
        if (rep) {
            OVS_CK(cudaStreamSynchronize(st));
            for (u32 k = 0; k + 1 < OVS_NMARKS; ++k) {
                float ms = 0;
                OVS_CK(cudaEventElapsedTime(&ms, ev.e[k], ev.e[k + 1]));
                rep->phase_ms[k] = ms;
            }
            rep->phase_ms[6] = rep->phase_ms[3];  // the exchange is the fused scatter
            OVS_CK(cudaEventElapsedTime(&rep->phase_ms[7], ev.e[0], ev.e[OVS_NMARKS - 1]));
            u64 mx = 0;
            for (u32 b = 0; b < p; ++b) {
                u64 t = 0;
                for (u32 r = 0; r < world; ++r) t += C[(size_t)r * p + b];
                if (rep->bucket_counts) rep->bucket_counts[b] = t;
                mx = std::max(mx, t);
            }
            rep->max_bucket = (u32)mx;
            rep->kernel_launches = cx.launches;
            // NVLink bytes out of this GPU: records of this shard, count rows, items of other owners
            u64 xb = 0;
            for (u32 b = 0; b < p; ++b)
                if ((u64)b * world / p != rank) xb += (u64)C[(size_t)rank * p + b] * (kb + (kv ? 8 : 0));
            xb += (u64)(world - 1) * (4 * (u64)p);
            rep->exchange_bytes = xb;
            run->splitters(rep->splitter_keys, rep->splitter_tags);
            u32 stv = 0;
            OVS_CK(cudaMemcpy(&stv, cx.status, 4, cudaMemcpyDeviceToHost));
            rep->device_status = stv;
            if (stv) return fail(OVS_EINTERNAL, "device-side check failed (status bits " + std::to_string(stv) + ")");
        }
        return OVS_OK;
    } catch (const NcclFail& e) {
        return fail(OVS_ENCCL, e.what());
    } catch (const CudaFail& e) {
        return fail(OVS_ECUDA, e.what());
    } catch (const StatusFail& e) {
        return fail(e.code, e.msg);
    } catch (const std::exception& e) {
        return fail(OVS_ECUDA, e.what());
    } catch (...) {
        return fail(OVS_ECUDA, "unknown exception");
    }
}

}  // namespace ovsd

using namespace ovsd;

extern "C" {

int ovs_comm_unique_id(void* out) {
    g_err.clear();
    if (!out) return fail(OVS_EINVAL, "NULL id buffer");
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return fail(OVS_ENCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    std::memcpy(out, &id, sizeof(id));
    return OVS_OK;
}

int ovs_comm_reserve(ovs_comm* c, size_t window_bytes, void* stream) {
    g_err.clear();
    if (!c) return fail(OVS_EINVAL, "NULL communicator");
    try {
        OVS_CK(cudaSetDevice(c->device));
        const cudaStream_t st = (cudaStream_t)stream;
        u64 want = window_bytes;
        if (c->world > 1) {  // the window is symmetric: the largest request of any rank
            c->h_tmp[0] = want;
            OVS_CK(cudaMemcpyAsync(c->d_tmp, c->h_tmp, 8, cudaMemcpyHostToDevice, st));
            OVS_NCCK(ncclAllReduce(c->d_tmp, c->d_tmp, 1, ncclUint64, ncclMax, c->nccl, st));
            OVS_CK(cudaMemcpyAsync(c->h_tmp, c->d_tmp, 8, cudaMemcpyDeviceToHost, st));
            OVS_CK(cudaStreamSynchronize(st));
            want = c->h_tmp[0];
        }
        want = (want + NCCL_WIN_REQUIRED_ALIGNMENT - 1) / NCCL_WIN_REQUIRED_ALIGNMENT * NCCL_WIN_REQUIRED_ALIGNMENT;
        if (want <= c->win_bytes) return OVS_OK;
        OVS_CK(cudaStreamSynchronize(st));
        if (c->win) { OVS_NCCK(ncclCommWindowDeregister(c->nccl, c->win)); c->win = nullptr; }
        if (c->win_buf) { OVS_NCCK(ncclMemFree(c->win_buf)); c->win_buf = nullptr; }
        c->win_bytes = 0;
        OVS_NCCK(ncclMemAlloc(&c->win_buf, want));
        OVS_NCCK(ncclCommWindowRegister(c->nccl, c->win_buf, want, &c->win, NCCL_WIN_COLL_SYMMETRIC));
        k_peer_ptrs<<<1, 32, 0, st>>>(c->win, c->d_peer, c->world);
        OVS_CK(cudaGetLastError());
        OVS_CK(cudaStreamSynchronize(st));
        c->win_bytes = want;
        return OVS_OK;
    } catch (const NcclFail& e) {
        return fail(OVS_ENCCL, e.what());
    } catch (const CudaFail& e) {
        return fail(OVS_ECUDA, e.what());
    } catch (const std::exception& e) {
        return fail(OVS_ECUDA, e.what());
    }
}

int ovs_comm_create(ovs_comm** out, const void* nccl_unique_id, int rank, int world, int device, size_t window_bytes) {
    g_err.clear();
    if (!out || !nccl_unique_id || world < 1 || rank < 0 || rank >= world) return fail(OVS_EINVAL, "invalid arguments");
    *out = nullptr;
    ovs_comm* c = new ovs_comm();
    c->rank = rank; c->world = world; c->device = device;
    try {
        OVS_CK(cudaSetDevice(device));
        ncclUniqueId id;
        std::memcpy(&id, nccl_unique_id, sizeof(id));
        OVS_NCCK(ncclCommInitRank(&c->nccl, world, id, rank));
        ncclDevCommRequirements reqs = {};
        reqs.lsaBarrierCount = 1;
        OVS_NCCK(ncclDevCommCreate(c->nccl, &reqs, &c->dev));
        c->dev_ok = true;
        if (c->dev.lsaSize != world)
            throw NcclFail("not every rank is load/store reachable (NVLink) from every other: lsa size " +
                           std::to_string(c->dev.lsaSize) + " of " + std::to_string(world));
        OVS_CK(cudaMalloc(&c->d_peer, sizeof(char*) * (size_t)world));
        OVS_CK(cudaMalloc(&c->d_tmp, sizeof(u64) * (4 * (size_t)world + 8)));
        OVS_CK(cudaMallocHost(&c->h_tmp, sizeof(u64) * (4 * (size_t)world + 8)));
        const int r = ovs_comm_reserve(c, std::max<size_t>(window_bytes, 1 << 20), nullptr);
        if (r != OVS_OK) { std::string e = g_err; ovs_comm_destroy(c); return fail(r, e); }
        *out = c;
        return OVS_OK;
    } catch (const NcclFail& e) {
        std::string m = e.what();
        ovs_comm_destroy(c);
        return fail(OVS_ENCCL, m);
    } catch (const CudaFail& e) {
        std::string m = e.what();
        ovs_comm_destroy(c);
        return fail(OVS_ECUDA, m);
    } catch (const std::exception& e) {
        std::string m = e.what();
        ovs_comm_destroy(c);
        return fail(OVS_ECUDA, m);
    }
}

int ovs_comm_destroy(ovs_comm* c) {
    if (!c) return OVS_OK;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    if (c->win) ncclCommWindowDeregister(c->nccl, c->win);
    if (c->win_buf) ncclMemFree(c->win_buf);
    if (c->dev_ok) ncclDevCommDestroy(c->nccl, &c->dev);
    if (c->nccl) ncclCommDestroy(c->nccl);
    if (c->d_peer) cudaFree(c->d_peer);
    if (c->d_tmp) cudaFree(c->d_tmp);
    if (c->h_tmp) cudaFreeHost(c->h_tmp);
    if (c->h_stage) cudaFreeHost(c->h_stage);
    delete c;
    return OVS_OK;
}

size_t ovs_comm_window_bytes(const ovs_comm* c) { return c ? c->win_bytes : 0; }

size_t ovs_dist_window_bytes(size_t n_recv, int dtype, int with_values, const ovs_params* prm, int world) {
    if (!prm || world < 1 || prm->p < 1) return 0;
    const u32 kb = dtype == OVS_F64 ? 8 : 4;
    const u64 m = rec_count(prm);
    const WinLayout L0 = win_layout(0, m, kb, with_values != 0, (u32)world, prm->p);
    return L0.rk + (size_t)n_recv * (kb + (with_values ? 8 : 0)) + 4 * 256;
}

size_t ovs_dist_workspace_bytes(ovs_comm* c, size_t n_local, int dtype, int with_values, const ovs_params* prm,
                                size_t out_capacity, void* stream) {
    g_err.clear();
    if (!c || dist_args(dtype, prm, c->world) != OVS_OK) return 0;
    try {
        OVS_CK(cudaSetDevice(c->device));
        std::vector<u64> sz;
        gather_sizes(c, n_local, out_capacity, 0, sz, (cudaStream_t)stream);
        u64 n_global = 0, offset = 0;
        for (int r = 0; r < c->world; ++r) {
            if (r < c->rank) offset += sz[3 * r];
            n_global += sz[3 * r];
        }
        if (dist_global(n_global, prm) != OVS_OK) return 0;
        const u32 kb = dtype == OVS_F64 ? 8 : 4;
        const WinLayout W = win_layout(c->win_bytes, rec_count(prm), kb, with_values != 0, (u32)c->world, prm->p);
        return ws_need(dtype, with_values != 0, make_cfg(n_local, n_global, offset, prm, c->world, c->rank, out_capacity, W));
    } catch (const std::exception& e) {
        g_err = e.what();
        return 0;
    } catch (...) {
        return 0;
    }
}

int ovs_dist_sort_keys(ovs_comm* c, const void* d_in, size_t n_local, int dtype, const ovs_params* prm, void* d_out,
                       size_t out_capacity, size_t* n_out, void* d_ws, size_t ws_bytes, void* stream, ovs_report* rep) {
    return dist_impl(c, d_in, nullptr, false, n_local, dtype, prm, d_out, nullptr, out_capacity, n_out, d_ws, ws_bytes,
                     stream, rep);
}

int ovs_dist_sort_pairs_stable(ovs_comm* c, const void* d_keys, const uint32_t* d_vals, size_t n_local, int dtype,
                               const ovs_params* prm, void* d_out_keys, uint32_t* d_out_vals, size_t out_capacity,
                               size_t* n_out, void* d_ws, size_t ws_bytes, void* stream, ovs_report* rep) {
    if (!d_out_vals && n_local) return fail(OVS_EINVAL, "NULL output values");
    return dist_impl(c, d_keys, d_vals, true, n_local, dtype, prm, d_out_keys, d_out_vals, out_capacity, n_out, d_ws,
                     ws_bytes, stream, rep);
}

int ovs_dist_plan(const uint32_t* counts, int world, uint32_t p, int rank, uint32_t* dst_off, uint64_t* recv) {
    if (!counts || world < 1 || rank < 0 || rank >= world || p < 1 || p % (uint32_t)world) return OVS_EINVAL;
    DistPlanHost P;
    dist_plan_host(counts, (u32)world, p, (u32)rank, P);
    if (dst_off) std::memcpy(dst_off, P.dst_off.data(), 4 * (size_t)p);
    if (recv) for (int r = 0; r < world; ++r) recv[r] = P.recv[r];
    return OVS_OK;
}

// Single-GPU emulation of `world` ranks for the tests: the same DistSort phases, the same kernels
// (the fused scatter writes into the other emulated ranks' windows), every phase run for rank 0,
// 1, ... in turn (stream order replaces the barriers: no kernel waits on another).
int ovs_dist_sort_virtual(int world, const void* const* d_keys, const uint32_t* const* d_vals, const size_t* n_local,
                          int dtype, const ovs_params* prm, void* const* d_out_keys, uint32_t* const* d_out_vals,
                          const size_t* out_capacity, size_t* n_out, void* const* d_ws, const size_t* ws_bytes,
                          void* const* d_win, size_t win_bytes, void* stream, uint64_t* counts, void* split_keys,
                          uint64_t* split_tags, float* rank_ms) {
    g_err.clear();
    if (world < 1 || !d_keys || !n_local || !d_out_keys || !out_capacity || !n_out || !d_ws || !ws_bytes || !d_win)
        return fail(OVS_EINVAL, "NULL argument");
    const bool kv = d_vals != nullptr;
    int v = dist_args(dtype, prm, world);
    if (v != OVS_OK) return fail(v, "invalid arguments");
    char** d_peer = nullptr;
    try {
        const cudaStream_t st = (cudaStream_t)stream;
        u64 n_global = 0;
        for (int r = 0; r < world; ++r) n_global += n_local[r];
        v = dist_global(n_global, prm);
        if (v != OVS_OK) return fail(v, "invalid global size");
        if (prm->method == OVS_DRO)
            for (int r = 0; r < world; ++r)
                if (n_local[r] != n_global / world) return fail(OVS_EINVAL, "DRO: equal shards of whole sequences");
        const u32 kb = dtype == OVS_F64 ? 8 : 4, p = prm->p;
        const WinLayout W = win_layout(win_bytes, rec_count(prm), kb, kv, (u32)world, p);
        if (W.end > win_bytes || W.cap == 0) return fail(OVS_ECAPACITY, "window too small");
        OVS_CK(cudaMalloc(&d_peer, sizeof(char*) * (size_t)world));
        OVS_CK(cudaMemcpyAsync(d_peer, d_win, sizeof(char*) * (size_t)world, cudaMemcpyHostToDevice, st));
        std::vector<Ctx> cx(world);
        std::vector<std::unique_ptr<DistRun>> runs;
        u64 off = 0;
        for (int r = 0; r < world; ++r) {
            DistCfg g = make_cfg(n_local[r], n_global, off, prm, world, r, out_capacity[r], W);
            g.keys = d_keys[r]; g.vals = kv ? d_vals[r] : nullptr; g.out_k = d_out_keys[r];
            g.out_v = kv ? d_out_vals[r] : nullptr;
            if (ws_bytes[r] < ws_need(dtype, kv, g)) { cudaFree(d_peer); return fail(OVS_EWORKSPACE, "workspace too small"); }
            cx[r].di = dev_info(); cx[r].dry = false; cx[r].ws = (char*)d_ws[r]; cx[r].st = st;
            cx[r].status = cx[r].take<u32>(4);
            runs.emplace_back(make_run(cx[r], dtype, kv, g));
            OVS_CK(cudaMemsetAsync(cx[r].status, 0, 4, st));
            off += n_local[r];
        }
        // per-rank device time of every phase (rank_ms): events around each rank's launches
        std::vector<cudaEvent_t> evs;
        auto tick = [&]() -> cudaEvent_t {
            if (!rank_ms) return nullptr;
            cudaEvent_t e;
            OVS_CK(cudaEventCreate(&e));
            OVS_CK(cudaEventRecord(e, st));
            evs.push_back(e);
            return e;
        };
        std::vector<std::pair<cudaEvent_t, cudaEvent_t>> span[3];  // per phase group, per rank
        for (int r = 0; r < world; ++r) {
            cudaEvent_t a = tick();
            runs[r]->sample(d_peer);
            span[0].push_back({a, tick()});
        }
        for (int r = 0; r < world; ++r) {
            cudaEvent_t a = tick();
            runs[r]->select((const char*)d_win[r]);
            runs[r]->count(d_peer);
            span[1].push_back({a, tick()});
        }
        std::vector<u32> C((size_t)world * p);
        OVS_CK(cudaMemcpyAsync(C.data(), (const char*)d_win[0] + W.C, 4 * C.size(), cudaMemcpyDeviceToHost, st));
        OVS_CK(cudaStreamSynchronize(st));
        std::vector<DistPlanHost> P(world);
        std::vector<u32*> hs(world, nullptr);
        for (int r = 0; r < world; ++r) {
            dist_plan_host(C.data(), (u32)world, p, (u32)r, P[r]);
            n_out[r] = P[r].recv[r];
        }
        for (int r = 0; r < world; ++r)
            if (P[0].recv[r] > W.cap || P[0].recv[r] > out_capacity[r]) {
                cudaFree(d_peer);
                return fail(OVS_ECAPACITY, "rank " + std::to_string(r) + " receives " + std::to_string(P[0].recv[r]));
            }
        std::vector<std::vector<u32>> hsv(world);
        for (int r = 0; r < world; ++r) {
            hsv[r].assign(4 * (size_t)p + 16, 0);
            hs[r] = hsv[r].data();
            cudaEvent_t a = tick();
            runs[r]->scatter(d_peer, P[r], hs[r]);
            OVS_CK(cudaStreamSynchronize(st));  // pageable staging: keep it alive until the upload is done
            span[2].push_back({a, tick()});
        }
        std::vector<std::pair<cudaEvent_t, cudaEvent_t>> fin;
        for (int r = 0; r < world; ++r) {
            cudaEvent_t a = tick();
            runs[r]->finish((const char*)d_win[r], (u32)(P[r].desc.size() / 3));
            fin.push_back({a, tick()});
        }
        if (counts)
            for (u32 b = 0; b < p; ++b) {
                u64 t = 0;
                for (int r = 0; r < world; ++r) t += C[(size_t)r * p + b];
                counts[b] = t;
            }
        runs[0]->splitters(split_keys, split_tags);
        OVS_CK(cudaStreamSynchronize(st));
        u32 stv = 0;
        for (int r = 0; r < world; ++r) {
            u32 x = 0;
            OVS_CK(cudaMemcpy(&x, cx[r].status, 4, cudaMemcpyDeviceToHost));
            stv |= x;
        }
        if (rank_ms) {
            for (int r = 0; r < world; ++r) {
                float tot = 0, ms = 0;
                for (int g = 0; g < 3; ++g) {
                    OVS_CK(cudaEventElapsedTime(&ms, span[g][r].first, span[g][r].second));
                    tot += ms;
                }
                OVS_CK(cudaEventElapsedTime(&ms, fin[r].first, fin[r].second));
                rank_ms[r] = tot + ms;
                if (std::getenv("OVS_DIST_PHASES")) {  // experiments: the phase split of every rank
                    float ph[4] = {0, 0, 0, ms};
                    for (int g = 0; g < 3; ++g) OVS_CK(cudaEventElapsedTime(&ph[g], span[g][r].first, span[g][r].second));
                    std::fprintf(stderr, "rank %d: sample %.3f select+count %.3f scatter %.3f finish %.3f ms\n", r, ph[0],
                                 ph[1], ph[2], ph[3]);
                }
            }
            for (auto e : evs) cudaEventDestroy(e);
        }
        cudaFree(d_peer);
        if (stv) return fail(OVS_EINTERNAL, "device-side check failed (status bits " + std::to_string(stv) + ")");
        return OVS_OK;
    } catch (const CudaFail& e) {
        if (d_peer) cudaFree(d_peer);
        return fail(OVS_ECUDA, e.what());
    } catch (const StatusFail& e) {
        if (d_peer) cudaFree(d_peer);
        return fail(e.code, e.msg);
    } catch (const std::exception& e) {
        if (d_peer) cudaFree(d_peer);
        return fail(OVS_ECUDA, e.what());
    }
}

size_t ovs_dist_virtual_workspace_bytes(int world, const size_t* n_local, int dtype, int with_values,
                                        const ovs_params* prm, const size_t* out_capacity, size_t win_bytes) {
    if (world < 1 || !n_local || !out_capacity || dist_args(dtype, prm, world) != OVS_OK) return 0;
    try {
        u64 n_global = 0;
        for (int r = 0; r < world; ++r) n_global += n_local[r];
        if (dist_global(n_global, prm) != OVS_OK) return 0;
        const u32 kb = dtype == OVS_F64 ? 8 : 4;
        const WinLayout W = win_layout(win_bytes, rec_count(prm), kb, with_values != 0, (u32)world, prm->p);
        size_t mx = 0;
        u64 off = 0;
        for (int r = 0; r < world; ++r) {
            mx = std::max(mx, ws_need(dtype, with_values != 0, make_cfg(n_local[r], n_global, off, prm, world, r, out_capacity[r], W)));
            off += n_local[r];
        }
        return mx;
    } catch (...) {
        return 0;
    }
}

}  // extern "C"
