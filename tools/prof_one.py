"""One sort of the metric workload (for ncu captures): python tools/prof_one.py [p] [s] [n]"""
import sys
sys.path.insert(0, ".")
import torch
import ovs_inputs
import paper_1608_08648_b200 as ovs

p = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
s = int(sys.argv[2]) if len(sys.argv) > 2 else 64
n = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 27
x = torch.from_numpy(ovs_inputs.keys("u32", n, seed=51)).cuda()
srt = ovs.Sorter(n, torch.uint32, False, "ros", p, s, 1)
srt(x)
torch.cuda.synchronize()
print("ok")
