"""The synthetic generator restates the reference's (workload.cpp:107-161)."""
import numpy as np

from paper_2503_23830_b200 import workload


def test_mt19937_64_known_answer():
    # C++ standard: the 10000th output of a default-seeded mt19937_64 (seed 5489)
    g = workload.MT19937_64(5489)
    for _ in range(9999):
        g()
    assert g() == 9981545732273789042


def test_generator_matches_reference(reflib):
    for mix, n, seed in [(2, 512, 2), (3, 4096, 7), (3, 300, 123)]:
        ppe, mod, ml = reflib.generate(mix, n, seed)
        b = workload.make_batch(mix, 1, n, seed)
        np.testing.assert_array_equal(np.diff(b.part_offset), ppe)
        flat_mod = np.concatenate([mod[j, :ppe[j]] for j in range(n)])
        flat_ml = np.concatenate([ml[j, :ppe[j]] for j in range(n)])
        np.testing.assert_array_equal(b.modality, flat_mod)
        np.testing.assert_array_equal(b.meta, flat_ml)


def test_phase_items_and_interleaved():
    b = workload.make_batch(2, 8, 64, 2)
    lv, ov, idx = b.phase_items("vision")
    assert len(lv) == int((b.modality == 1).sum())
    assert (lv >= 64).all() and (lv <= 4096).all()
    ll, ol = b.llm_items()
    assert len(ll) == 512 and (ol == np.arange(512) % 8).all()
    # interleaved = sum of ceil(meta / rate) (core.cpp:163-181)
    enc = -(-b.meta // b.rates[b.modality])
    np.testing.assert_array_equal(ll, np.add.reduceat(enc, b.part_offset[:-1]))
