// ovs_s32_k.cu — instantiation of the string sort (32-byte keys in memcmp order, SURVEY.md §8(f) f3;
// the paper's workload): ROS, keys only.
#include "ovs_engine.cuh"

namespace ovs {
Out plan_s32_k(Ctx& c, void* keys, u32* vals, size_t n, const ovs_params* prm) {
    (void)vals;
    RosSortS32 r(c, keys, (u32)n, prm->p, prm->s, prm->seed);
    Out o;
    o.sk = r.rep_raw;
    o.st = r.rep_st;
    o.counts = r.counts;
    if (!c.dry) r.run();
    o.ws = c.off + 256;
    return o;
}
}  // namespace ovs
