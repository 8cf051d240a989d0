"""Host key packing (fss.pack_keys, the image KeyBatch.from_keys uploads) vs
a per-key restatement of the SoA layout -- CPU only."""
import numpy as np
import pytest

from paper_2209_03526_b200 import fss


def _naive(keys, bits):
    n = len(keys)
    root = np.stack([np.frombuffer(k.root_seed, np.uint8) for k in keys])
    scw = np.zeros((bits, n, 16), np.uint8)
    ctrl = np.zeros((3, n), np.uint32)
    flags = np.zeros(n, np.uint8)
    for i, k in enumerate(keys):
        scw[:, i, :] = np.ascontiguousarray(k.seed_cw, np.uint64).view(np.uint8).reshape(bits, 16)
        for lvl in range(bits):
            for j in range(3):
                ctrl[j, i] |= np.uint32(((int(k.ctrl_cw[lvl]) >> j) & 1) << lvl)
        flags[i] = (k.root_t & 1) | ((k.final_cw & 1) << 1) | ((k.add_const & 1) << 2)
    return np.concatenate([root.reshape(-1), scw.reshape(-1), ctrl.view(np.uint8).reshape(-1), flags])


@pytest.mark.parametrize("bits,n,cls", [(1, 1, fss.DpfKey), (9, 6, fss.DcfKey), (16, 12, fss.DcfKey),
                                        (31, 5, fss.DpfKey), (32, 7, fss.DcfKey)])
def test_pack_keys_matches_per_key_layout(bits, n, cls):
    rng = np.random.default_rng(bits * 100 + n)
    keys = [cls(domain_bits=bits, root_seed=rng.bytes(16), root_t=int(rng.integers(0, 2)),
                seed_cw=rng.integers(0, 2**63, (bits, 2), dtype=np.uint64),
                ctrl_cw=rng.integers(0, 8, bits).astype(np.uint8), final_cw=int(rng.integers(0, 2)),
                add_const=int(rng.integers(0, 2))) for _ in range(n)]
    assert np.array_equal(fss.pack_keys(keys, bits), _naive(keys, bits))
