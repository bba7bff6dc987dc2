"""f3: the paper's own workload — 32-byte string keys in memcmp order — through
the C ABI (dtype OVS_S32, ROS), element by element against the oracle: output bytes, splitter
records and tags, bucket counts."""
import numpy as np
import pytest
import torch

import ovs_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ovs():
    import paper_1608_08648_b200 as m
    m.lib()
    return m


def run(ovs, orc, dist, n, p, s, seed=3):
    x = ovs_inputs.keys(dist, n, seed=n % 97)
    ref = orc.ros_sort(x, p, s, seed)
    t = torch.from_numpy(np.frombuffer(x.tobytes(), dtype=np.uint8).copy()).cuda()
    rep = ovs.sort_strings32(t, p, s, seed)
    torch.cuda.synchronize()
    out = t.cpu().numpy().view("V32")
    assert rep.device_status == 0
    assert out.tobytes() == ref.keys.tobytes()
    np.testing.assert_array_equal(rep.counts, ref.counts)
    if p > 1:
        assert rep.splitter_keys.tobytes() == ref.split_keys.tobytes()
        np.testing.assert_array_equal(rep.splitter_tags, ref.split_tags)
    return rep


@pytest.mark.parametrize("dist", ["s32", "s32_prefix", "s32_few"])
@pytest.mark.parametrize("n,p,s", [(1, 1, 1), (7, 2, 4), (1000, 4, 8), (100_003, 64, 32), (300_000, 256, 16),
                                   (200_000, 1, 1), (1_000_000, 1000, 8), (65_537, 7, 64)])
def test_strings_ros(ovs, orc, dist, n, p, s):
    if p * s - 1 > n:
        pytest.skip("sample larger than the input")
    run(ovs, orc, dist, n, p, s)


def test_strings_exhaustive_sample(ovs, orc):
    """ps - 1 = n (the whole input is the sample)."""
    run(ovs, orc, "s32_prefix", 4095, 64, 64)


@pytest.mark.slow
def test_strings_paper_grid_point(ovs, orc):
    """n = 2^22 strings (the paper's grid runs 1.024M .. 32.768M), p = 256, s = ceil(lg^2 n) = 484
    (the paper's default oversampling, reading Q13)."""
    run(ovs, orc, "s32", 1 << 22, 256, 484)


def test_strings_errors(ovs):
    t = torch.zeros(32 * 1000, dtype=torch.uint8, device="cuda")
    with pytest.raises(ovs.OvsError) as e:
        ovs.Sorter(1000, "s32", False, "dro", 4, 2, 1, device=t.device)
    assert e.value.code in (ovs.OVS_EDTYPE, ovs.OVS_EINVAL)
    with pytest.raises(ovs.OvsError):
        ovs.Sorter(1000, "s32", True, "ros", 4, 2, 1, device=t.device)
