"""bench.py's config legs at small sizes: each runs end to end and its
bit-exactness gates pass (the same code the round-end bench runs at the
BASELINE sizes)."""

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bc():
    import bench_configs
    from paper_2209_03526_b200 import _lib
    _lib.check(_lib.load().ogm_init())
    return bench_configs


@pytest.mark.parametrize("lg", [12, 18, 22])
def test_c5_shuffle_leg(bc, lg):
    e = bc.c5_shuffle_leg(lg, 2, 1)
    assert e["gate"]["recombination_full_size"] and e["gate"]["r3_equal_to_oracle_on_2^16_run"]
    assert e["ms"] > 0 and e["hbm_frac"] > 0


@pytest.mark.parametrize("lg", [12, 22])
def test_c5_fetch_leg(bc, lg):
    for e in bc.c5_fetch_leg(lg, 2, 1):
        assert all(e["gate"].values()), e["gate"]
        assert 0 <= e["kept"] <= e["rows"]


def test_c3_leg_small(bc):
    e = bc.c3_leg(1, 1, rows=4096)
    assert all(e["gate"].values()), e["gate"]


@pytest.mark.parametrize("rows", [5000, 200_000])
def test_c4_root_slot_small(bc, rows):
    e = bc.c4_root_slot(rows, 1, 1, 1, 0, 1)
    assert all(e["gate"].values()), e["gate"]
    assert e["kept"] == e["matches"]


def test_c4_sec_eval_gate(bc):
    e = bc.c4_sec_eval(100_000, 1, 1, 1, 0, 1)
    assert e["parity_gate"]["equal_to_oracle"]
