// ovs_u32_k.cu — instantiation of the sort engine for u32 keys, keys only (one
// translation unit per (dtype, keys/pairs) so the build runs in parallel).
#include "ovs_engine.cuh"

namespace ovs {
Out plan_u32_k(Ctx& c, void* keys, u32* vals, size_t n, const ovs_params* prm) {
    return plan_or_run<DT_U32, false>(c, keys, vals, n, prm);
}
DistRun* dist_u32_k(Ctx& c, const DistCfg& cfg) { return make_dist<DT_U32, false>(c, cfg); }
}  // namespace ovs

#ifdef OVS_BS_PROF  // experiments only: bucket-sorter phase cycles of this translation unit's kernels
extern "C" int ovs_debug_bsprof_u32_k(unsigned long long* out, int reset) {
    unsigned long long v[16];
    if (cudaMemcpyFromSymbol(v, ovs::g_bsprof, sizeof(v)) != cudaSuccess) return 1;
    for (int i = 0; i < 16; ++i) out[i] += v[i];
    if (reset) {
        unsigned long long z[16] = {0};
        cudaMemcpyToSymbol(ovs::g_bsprof, z, sizeof(z));
    }
    return 0;
}
#endif
#ifdef OVS_SF_PROF
extern "C" int ovs_debug_sfprof(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, ovs::g_sfprof, 8 * sizeof(unsigned long long)) != cudaSuccess;
}
#endif
