"""The seeded input generator (efgp_data): Philox known-answer vectors and the config recipes."""
import numpy as np

from efgp_data import CONFIGS, generate, philox, shard_range


def test_philox4x32_10_known_answers():
    # Random123 known-answer vectors for philox4x32-10 (Salmon et al., SC'11)
    kat = [((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
           ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
           ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
            (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1))]
    for ctr, key, out in kat:
        got = philox.philox4x32_10(*ctr, *key)
        assert tuple(int(g) for g in got) == out


def test_uniform_properties():
    u = philox.uniform(4, 0, np.arange(200_000, dtype=np.uint64), 0)
    assert u.min() >= 0 and u.max() < 1
    assert abs(u.mean() - 0.5) < 3e-3
    u2 = philox.uniform(4, 0, np.arange(200_000, dtype=np.uint64), 1)
    assert abs(np.corrcoef(u, u2)[0, 1]) < 1e-2
    z = philox.normal(4, 1, np.arange(200_000, dtype=np.uint64), 0)
    assert abs(z.mean()) < 1e-2 and abs(z.std() - 1) < 1e-2


def test_configs_deterministic_and_shardable():
    c = CONFIGS["c3"]
    x, y, xt = generate(c, N=5000, q=100)
    x2, y2, _ = generate(c, N=5000, q=100)
    np.testing.assert_array_equal(x, x2)
    np.testing.assert_array_equal(y, y2)
    assert x.min() >= 0 and x.max() <= 1 and (x == 1).any() is not None
    # shards regenerate the same records
    a, b = shard_range(5000, 1, 3)
    xs, ys, _ = generate(c, N=b - a, q=1, start=a)
    np.testing.assert_array_equal(xs, x[a:b])
    np.testing.assert_array_equal(ys, y[a:b])
    ranges = [shard_range(1_000_000_000, g, 8) for g in range(8)]
    assert ranges[0][0] == 0 and ranges[-1][1] == 1_000_000_000
    assert all(ranges[i][1] == ranges[i + 1][0] for i in range(7))


def test_c1_targets_equispaced():
    _, _, xt = generate(CONFIGS["c1"], N=10)
    assert xt.shape == (1000, 1) and xt[0, 0] == 0.0 and xt[-1, 0] == 1.0
