"""Seeded input generator (datagen/) -- CPU checks.  The GPU twin's bitwise
equality with this numpy version is checked in tests/test_gpu_parity.py."""
import numpy as np

import datagen


def test_splitmix64_known_structure():
    # splitmix64 is a bijection on uint64: distinct counters -> distinct outputs
    x = np.arange(1 << 16, dtype=np.uint64)
    h = datagen.splitmix64(x)
    assert len(np.unique(h)) == len(x)
    # the finaliser of counter 0 is the mix of the golden gamma (published constant)
    z = 0x9E3779B97F4A7C15
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
    z ^= z >> 31
    assert int(h[0]) == z


def test_values_range_and_exactness():
    for dt, bits in ((np.float32, 24), (np.float64, 53)):
        v = datagen.values(3, 1, dt, np.arange(50), 17, 9)
        assert v.dtype == dt
        assert v.min() >= -1.0 and v.max() < 1.0
        # x + 1 is an integer multiple of 2^-(bits-1)
        scaled = (v.astype(np.float64) + 1.0) * 2.0 ** (bits - 1)
        assert np.all(scaled == np.round(scaled))
        assert abs(float(v.mean())) < 0.05


def test_values_depend_on_global_index_only():
    a = datagen.values(1, 0, np.float32, [5, 6, 7], 4, 3)
    b = datagen.values(1, 0, np.float32, [7], 4, 3)
    assert np.array_equal(a[2], b[0])
    c = datagen.values(1, 1, np.float32, [7], 4, 3)  # other matrix id
    assert not np.array_equal(b, c)
    d = datagen.values(2, 0, np.float32, [7], 4, 3)  # other seed
    assert not np.array_equal(b, d)


def test_fill_host_layout_and_padding():
    ids = [10, 11]
    buf = datagen.fill_host(0, 0, np.float64, 3, 2, 5, 12, ids)
    assert buf.size == 24
    v = datagen.values(0, 0, np.float64, ids, 3, 2)
    for s in range(2):
        for c in range(2):
            assert np.array_equal(buf[s * 12 + c * 5: s * 12 + c * 5 + 3], v[s, c])
            assert np.all(np.isnan(buf[s * 12 + c * 5 + 3: s * 12 + c * 5 + 5]))
        assert np.all(np.isnan(buf[s * 12 + 10: s * 12 + 12]))
