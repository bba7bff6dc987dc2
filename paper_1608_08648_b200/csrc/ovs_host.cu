// ovs_host.cu — the host-buffer entry of include/ovs.h (ovs_host_pipe_*): a stream of sorts from and to
// pinned host memory.  Step k's host->device copy, the sorts, and step k-1's device->host copy run on three
// streams of the pipe (the two PCIe directions have their own copy engines), over nbuf rotating device
// buffers of the caller's; the sort itself is ovs_sort_keys on the pipe's sort stream.  No kernels here.
#include <cuda_runtime.h>

#include <new>
#include <string>
#include <vector>

#include "ovs.h"

namespace ovs {
extern thread_local std::string g_err;
}
using ovs::g_err;

struct ovs_host_pipe {
    size_t n = 0, bytes = 0, wsb = 0, k = 0;
    int dtype = 0, dev = 0;
    ovs_params prm{};
    std::vector<void*> bufs;
    void* ws = nullptr;
    cudaStream_t s_in = nullptr, s_sort = nullptr, s_out = nullptr;
    std::vector<cudaEvent_t> loaded, sorted, freed;
    cudaEvent_t t0 = nullptr, t1 = nullptr;  // first copy-in start / last copy-out end since the last wait
    bool timing = false, ended = false;
};

namespace {
struct DevGuard {  // the pipe's device current for the call, the caller's restored after
    int prev = -1;
    bool ok = true;
    explicit DevGuard(int dev) {
        ok = cudaGetDevice(&prev) == cudaSuccess && (prev == dev || cudaSetDevice(dev) == cudaSuccess);
        if (!ok) prev = -1;
        want = dev;
    }
    ~DevGuard() { if (prev >= 0 && prev != want) cudaSetDevice(prev); }
    int want = 0;
};
int cuda_fail(cudaError_t e, const char* what) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    cudaGetLastError();
    return OVS_ECUDA;
}
#define HP_CK(x)                                        \
    do {                                                \
        cudaError_t e_ = (x);                           \
        if (e_ != cudaSuccess) return cuda_fail(e_, #x); \
    } while (0)
size_t key_bytes(int dtype) { return dtype == OVS_F64 ? 8 : dtype == OVS_S32 ? 32 : 4; }
void release(ovs_host_pipe* hp) {
    for (auto* v : {&hp->loaded, &hp->sorted, &hp->freed})
        for (cudaEvent_t e : *v) if (e) cudaEventDestroy(e);
    if (hp->t0) cudaEventDestroy(hp->t0);
    if (hp->t1) cudaEventDestroy(hp->t1);
    for (cudaStream_t s : {hp->s_in, hp->s_sort, hp->s_out}) if (s) cudaStreamDestroy(s);
    delete hp;
}
}  // namespace

extern "C" {

int ovs_host_pipe_create(ovs_host_pipe** out, size_t n, int dtype, const ovs_params* prm, void* const* d_bufs,
                         int nbuf, void* d_ws, size_t ws_bytes) {
    g_err.clear();
    if (!out) { g_err = "NULL out"; return OVS_EINVAL; }
    *out = nullptr;
    if (!prm || !d_bufs || !d_ws || n == 0 || nbuf < 1 || nbuf > 16) { g_err = "invalid arguments"; return OVS_EINVAL; }
    if (dtype != OVS_U32 && dtype != OVS_I32 && dtype != OVS_F64 && dtype != OVS_S32) { g_err = "dtype"; return OVS_EDTYPE; }
    for (int i = 0; i < nbuf; ++i)
        if (!d_bufs[i]) { g_err = "NULL device buffer"; return OVS_EINVAL; }
    const size_t need = ovs_workspace_bytes(n, dtype, 0, prm);
    if (need == 0) { g_err = "invalid sort parameters"; return OVS_EINVAL; }
    if (ws_bytes < need) { g_err = "workspace too small"; return OVS_EWORKSPACE; }
    ovs_host_pipe* hp = new (std::nothrow) ovs_host_pipe;
    if (!hp) { g_err = "out of host memory"; return OVS_ECUDA; }
    try {
        hp->bufs.assign(d_bufs, d_bufs + nbuf);
        hp->loaded.assign(nbuf, nullptr);
        hp->sorted.assign(nbuf, nullptr);
        hp->freed.assign(nbuf, nullptr);
    } catch (...) {
        delete hp;
        g_err = "out of host memory";
        return OVS_ECUDA;
    }
    hp->n = n; hp->bytes = n * key_bytes(dtype); hp->dtype = dtype; hp->prm = *prm; hp->ws = d_ws; hp->wsb = ws_bytes;
    int rc = OVS_OK;
    auto ck = [&](cudaError_t e, const char* what) { if (rc == OVS_OK && e != cudaSuccess) rc = cuda_fail(e, what); };
    ck(cudaGetDevice(&hp->dev), "cudaGetDevice");
    ck(cudaStreamCreateWithFlags(&hp->s_in, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaStreamCreateWithFlags(&hp->s_sort, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaStreamCreateWithFlags(&hp->s_out, cudaStreamNonBlocking), "cudaStreamCreate");
    for (int i = 0; i < nbuf && rc == OVS_OK; ++i) {
        ck(cudaEventCreateWithFlags(&hp->loaded[i], cudaEventDisableTiming), "cudaEventCreate");
        ck(cudaEventCreateWithFlags(&hp->sorted[i], cudaEventDisableTiming), "cudaEventCreate");
        ck(cudaEventCreateWithFlags(&hp->freed[i], cudaEventDisableTiming), "cudaEventCreate");
    }
    ck(cudaEventCreate(&hp->t0), "cudaEventCreate");
    ck(cudaEventCreate(&hp->t1), "cudaEventCreate");
    if (rc == OVS_OK) {  // the sticky status word of the workspace starts clear
        const int st = ovs_device_status(d_ws, hp->s_sort, nullptr, 1);
        if (st == OVS_ECUDA) rc = st;
    }
    if (rc != OVS_OK) { const std::string keep = g_err; release(hp); g_err = keep; return rc; }
    g_err.clear();
    *out = hp;
    return OVS_OK;
}

int ovs_host_pipe_submit(ovs_host_pipe* hp, const void* h_in, void* h_out) {
    g_err.clear();
    if (!hp || !h_in || !h_out) { g_err = "NULL argument"; return OVS_EINVAL; }
    DevGuard g(hp->dev);
    if (!g.ok) return cuda_fail(cudaGetLastError(), "cudaSetDevice");
    const size_t b = hp->k % hp->bufs.size();
    if (hp->k >= hp->bufs.size()) HP_CK(cudaStreamWaitEvent(hp->s_in, hp->freed[b], 0));
    if (!hp->timing) { HP_CK(cudaEventRecord(hp->t0, hp->s_in)); hp->timing = true; hp->ended = false; }
    HP_CK(cudaMemcpyAsync(hp->bufs[b], h_in, hp->bytes, cudaMemcpyHostToDevice, hp->s_in));
    HP_CK(cudaEventRecord(hp->loaded[b], hp->s_in));
    HP_CK(cudaStreamWaitEvent(hp->s_sort, hp->loaded[b], 0));
    const int rc = ovs_sort_keys(hp->bufs[b], hp->n, hp->dtype, &hp->prm, hp->ws, hp->wsb, hp->s_sort, nullptr);
    if (rc != OVS_OK) return rc;
    HP_CK(cudaEventRecord(hp->sorted[b], hp->s_sort));
    HP_CK(cudaStreamWaitEvent(hp->s_out, hp->sorted[b], 0));
    HP_CK(cudaMemcpyAsync(h_out, hp->bufs[b], hp->bytes, cudaMemcpyDeviceToHost, hp->s_out));
    HP_CK(cudaEventRecord(hp->freed[b], hp->s_out));
    HP_CK(cudaEventRecord(hp->t1, hp->s_out));
    hp->ended = true;
    ++hp->k;
    return OVS_OK;
}

int ovs_host_pipe_wait(ovs_host_pipe* hp, float* ms) {
    g_err.clear();
    if (!hp) { g_err = "NULL pipe"; return OVS_EINVAL; }
    DevGuard g(hp->dev);
    if (!g.ok) return cuda_fail(cudaGetLastError(), "cudaSetDevice");
    HP_CK(cudaStreamSynchronize(hp->s_out));  // the last copy-out follows every copy-in and sort
    HP_CK(cudaStreamSynchronize(hp->s_in));
    if (ms) {
        *ms = 0.f;
        if (hp->timing && hp->ended) HP_CK(cudaEventElapsedTime(ms, hp->t0, hp->t1));
    }
    hp->timing = false;
    return ovs_device_status(hp->ws, hp->s_sort, nullptr, 1);
}

int ovs_host_pipe_destroy(ovs_host_pipe* hp) {
    g_err.clear();
    if (!hp) return OVS_OK;
    DevGuard g(hp->dev);
    cudaStreamSynchronize(hp->s_in);
    cudaStreamSynchronize(hp->s_sort);
    cudaStreamSynchronize(hp->s_out);
    cudaGetLastError();
    release(hp);
    return OVS_OK;
}

}  // extern "C"
