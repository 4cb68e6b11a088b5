"""P15 -- the reported metric is the paper's Eq. 1 (real: 2MNK flops per
problem) / Eq. 2 (complex: 8MNK), and the
roofline bytes are SURVEY 8(d)'s (MK + KN + [beta != 0] MN + MN) * elt.
CPU only: bench.py's Shape arithmetic, no GPU."""
import bench


def test_eq1_worked_example():
    # (10, 10, 10) in 1 us -> 2 GFLOP/s
    s = bench.Shape("f32", "NN", 10, 10, 10, 1, 1.0, 0.0, 1)
    assert s.flops() == 2000.0
    assert s.flops() / 1e-6 / 1e9 == 2.0


def test_eq2_complex_and_batch():
    c = bench.Shape("c64", "NT", 3, 5, 7, 11, 1.0, 0.5, 1)
    assert c.flops() == 8.0 * 3 * 5 * 7 * 11
    assert c.flops(batch=2) == 8.0 * 3 * 5 * 7 * 2


def test_algorithmic_bytes():
    # beta != 0: C is read and written; beta == 0: written only
    s = bench.Shape("f32", "TT", 4, 6, 8, 10, 1.5, 0.5, 1)
    assert s.alg_bytes() == (4 * 8 + 8 * 6 + 2 * 4 * 6) * 4 * 10
    z = bench.Shape("f64", "NN", 4, 6, 8, 10, 1.0, 0.0, 1)
    assert z.alg_bytes() == (4 * 8 + 8 * 6 + 4 * 6) * 8 * 10
    cz = bench.Shape("c64", "NN", 4, 6, 8, 10, 1.0, 0.0, 1)
    assert cz.alg_bytes() == (4 * 8 + 8 * 6 + 4 * 6) * 16 * 10


def test_roofline_bound_selection():
    pk = {"hbm_gbs": 6550.0, "source": "test"}
    small = bench.Shape("f32", "NN", 8, 8, 8, 1000, 1.5, 0.5, 1)   # AI = 1 flop/B: HBM-bound
    roof = bench.roofline_of(small, 1000, 1e-6, pk)
    assert roof["bound"] == "hbm" and roof["unit"] == "GB/s"
    assert abs(roof["achieved"] - small.alg_bytes() / 1e-6 / 1e9) < 0.1
    big = bench.Shape("f64", "NN", 80, 80, 80, 1000, 1.0, 0.0, 1)  # AI = 6.7 flop/B > fp64 ridge 5.7
    roof = bench.roofline_of(big, 1000, 1e-3, pk)
    assert roof["bound"] == "tensor" and roof["unit"] == "TFLOP/s"
    assert abs(roof["frac"] - big.flops() / 1e-3 / 1e12 / roof["peak"]) < 1e-3
