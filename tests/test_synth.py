"""Input generator checks (the recipe of DESIGN.md §3)."""
import numpy as np

import synth


def test_splitmix64_reference_vectors():
    # SplitMix64 seeded with state 0: first three outputs (Steele/Lea/Flood;
    # the generator advances the state by the golden gamma before mixing).
    g = synth.GOLDEN
    out = synth.splitmix64(np.array([0, g, (2 * g) & synth.MASK64], dtype=np.uint64))
    assert [int(v) for v in out] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_value_ranges_and_exactness():
    v = synth.values_f32(1, 0, 1000, 16, "f32", "real")
    assert v.min() >= 0 and v.max() < 1
    s = synth.values_f32(1, 0, 1000, 16, "f32", "signed")
    assert s.min() >= -1 and s.max() < 1 and not np.any((s == 0) & np.signbit(s))
    i = synth.values_f32(1, 0, 1000, 16, "f32", "int")
    assert set(np.unique(i)) <= set(range(-8, 9))
    b = synth.values_f32(1, 0, 1000, 16, "bf16", "real")
    np.testing.assert_array_equal(synth.bf16_bits_to_f32(synth.f32_to_bf16_bits(b)), b)
    bs = synth.values_f32(1, 0, 1000, 16, "bf16", "signed")
    np.testing.assert_array_equal(synth.bf16_bits_to_f32(synth.f32_to_bf16_bits(bs)), bs)


def test_values_are_counter_based():
    full = synth.values_f32(3, 0, 100, 8)
    part = synth.values_f32(3, 40, 10, 8)
    np.testing.assert_array_equal(full[40:50], part)
    rows = np.array([5, 77, 3])
    np.testing.assert_array_equal(synth.values_f32(3, 0, 0, 8, rows=rows), full[rows])


def test_lengths_sum_and_shape():
    for name in ("cora", "arxiv"):
        w = synth.workload(name)
        L = synth.segment_lengths(w["E"], w["S"], w["dist"], w["seed"])
        assert L.sum() == w["E"] and L.shape == (w["S"],) and L.min() >= 0
    U = synth.segment_lengths(1 << 12, 1 << 8, "uniform")
    assert np.all(U == 16)
    U = synth.segment_lengths(10, 4, "uniform")
    assert list(U) == [3, 3, 2, 2]


def test_lomax_mean():
    # Lomax alpha=2 has mean 1/(alpha-1) = 1 for the weights; apportionment keeps E exactly
    rng = np.random.default_rng(0)
    u = 1 - rng.random(200_000)
    w = u ** -0.5 - 1
    assert abs(w.mean() - 1.0) < 0.05


def test_apportion_ties_to_lower_id():
    L = synth.apportion(5, np.ones(3))
    assert list(L) == [2, 2, 1]


def test_stress_kinds_sum():
    for k in synth.STRESS_KINDS:
        L = synth.stress_lengths(k, 999, 77, seed=1)
        assert L.sum() == 999 and L.shape == (77,)


def test_src_index_range():
    s = synth.src_index(1001, 0, 10000, 37)
    assert s.min() >= 0 and s.max() < 37
    np.testing.assert_array_equal(s[100:200], synth.src_index(1001, 100, 100, 37))
