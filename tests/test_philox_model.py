"""The throughput-mode noise generator's CPU model, pinned to the published
Philox4x32-10 known-answer vectors (no GPU needed)."""
import numpy as np

from philox_model import KAT, normals, philox4x32, philox_words


def test_philox4x32_10_known_answers():
    for ctr, key, want in KAT:
        got = philox4x32(*[np.array([c], dtype=np.uint64) for c in ctr], *key)
        assert tuple(int(v[0]) for v in got) == want


def test_model_layout_and_moments():
    R, T, du = 3, 10, 2
    z = normals(5, 7, 0, 400, R, T, du)
    assert z.shape == (400, T, R, du)
    assert abs(z.mean()) < 0.05 and abs(z.std() - 1.0) < 0.05
    # shard invariance: samples [100, 200) drawn on their own
    np.testing.assert_array_equal(normals(5, 7, 100, 100, R, T, du), z[100:200])
    # group g of robot k holds sequence entries n = 4g..4g+3, n = t·du + d
    w = philox_words(5, 7, 0, 1, R, T, du)
    assert w.shape == (1, R, (T * du + 3) // 4, 4)
