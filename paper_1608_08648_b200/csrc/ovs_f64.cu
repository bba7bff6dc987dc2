// ovs_f64.cu — instantiation of the sort engine for f64 keys (keys only / key-value).
#include "ovs_engine.cuh"

namespace ovs {
Out plan_f64(Ctx& c, void* keys, u32* vals, size_t n, const ovs_params* prm, bool kv) {
    return kv ? plan_or_run<DT_F64, true>(c, keys, vals, n, prm) : plan_or_run<DT_F64, false>(c, keys, vals, n, prm);
}
}  // namespace ovs
