"""The reference-side ctypes shim from INTEGRATION.md against the golden
reference evaluations (numpy in, numpy out)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_shim_eval_points_matches_reference(golden):
    import oracle
    from integration import oblivgm_b200_shim as shim
    from paper_2209_03526_b200 import fss
    g = golden("fss")
    for tag in g["cases"]:
        comparison = str(tag).startswith("dcf")
        bits = int(str(tag).split("_b")[1])
        k0, _ = oracle.tree_gen_batch(g[f"{tag}_alphas"], bits, g[f"{tag}_roots0"], g[f"{tag}_roots1"], comparison)
        cls = fss.DcfKey if comparison else fss.DpfKey
        keys = [cls(domain_bits=bits, root_seed=k0.root[i].tobytes(), root_t=0,
                    seed_cw=k0.seed_cw[i].view(np.uint64).reshape(bits, 2), ctrl_cw=k0.ctrl_cw[i],
                    final_cw=int(k0.final_cw[i])) for i in range(k0.count)]
        got = shim.eval_points(keys, g[f"{tag}_points"].astype(np.uint32))
        assert np.array_equal(got, g[f"{tag}_eval0"]), tag


def test_shim_parity_rows_matches_oracle():
    import oracle
    from integration import oblivgm_b200_shim as shim
    rng = np.random.default_rng(4)
    da, db = (rng.integers(0, 1 << 32, (300, 37), dtype=np.uint32) for _ in range(2))
    ia, ib = (rng.integers(0, 1 << 32, 37, dtype=np.uint32) for _ in range(2))
    assert np.array_equal(shim.parity_rows_device(da, db, ia, ib), oracle.masked_parity(da, db, ia, ib))
