"""Generate the golden fixtures in tests/golden/ from the LIVE reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the read-only reference package (oblivgm 0.1.0,
/root/reference/pkg/src) and records its outputs on seeded inputs.  The
fixtures travel to the GPU box; nothing there reads /root/reference.

Randomness injection: the reference draws FSS root seeds with
``rng.bytes(16)`` twice per tree (src/fss.py:117-118); ``StubRng`` feeds the
same recorded roots to both sides.  AES itself is pinned against the
``cryptography`` package (the reference's AES provider, src/prf.py:19).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


class StubRng:
    """Feeds recorded 16-byte roots to src/fss.py:_tree_gen."""

    def __init__(self, chunks):
        self.chunks = list(chunks)

    def bytes(self, n):
        b = self.chunks.pop(0)
        assert len(b) == n
        return b


def fss_fixture(fss, prf):
    rng = np.random.default_rng(20260101)
    out = {}
    cases = []
    for comparison in (False, True):
        for bits in (1, 2, 5, 9, 13, 20, 32):
            K = 16
            alphas = rng.integers(0, 1 << bits, size=K, dtype=np.uint64)
            if bits <= 5:
                alphas[:2] = [0, (1 << bits) - 1]
            r0 = rng.integers(0, 256, (K, 16), dtype=np.uint8)
            r1 = rng.integers(0, 256, (K, 16), dtype=np.uint8)
            pts = rng.integers(0, 1 << bits, size=K, dtype=np.uint64)
            pts[: K // 4] = alphas[: K // 4]  # hit the special point
            scw = np.zeros((K, bits, 2), np.uint64)
            ccw = np.zeros((K, bits), np.uint8)
            fin = np.zeros(K, np.uint8)
            e0 = np.zeros(K, np.uint8)
            e1 = np.zeros(K, np.uint8)
            for k in range(K):
                k0, k1 = fss._tree_gen(int(alphas[k]), bits, StubRng([r0[k].tobytes(), r1[k].tobytes()]),
                                       comparison)
                scw[k] = k0.seed_cw
                ccw[k] = k0.ctrl_cw
                fin[k] = k0.final_cw
                ev = fss.dcf_eval if comparison else fss.dpf_eval
                e0[k] = ev(k0, int(pts[k]))
                e1[k] = ev(k1, int(pts[k]))
            tag = f"{'dcf' if comparison else 'dpf'}_b{bits}"
            cases.append(tag)
            out.update({f"{tag}_alphas": alphas, f"{tag}_roots0": r0, f"{tag}_roots1": r1,
                        f"{tag}_seed_cw": scw, f"{tag}_ctrl_cw": ccw, f"{tag}_final_cw": fin,
                        f"{tag}_points": pts, f"{tag}_eval0": e0, f"{tag}_eval1": e1})
            if bits <= 13:
                n = int(rng.integers(1, (1 << bits) + 1))
                for k in range(3):
                    k0, k1 = fss._tree_gen(int(alphas[k]), bits,
                                           StubRng([r0[k].tobytes(), r1[k].tobytes()]), comparison)
                    out[f"{tag}_fde{k}_n"] = np.array(n)
                    out[f"{tag}_fde{k}_w0"] = fss.full_domain_eval(k0, n).words
                    out[f"{tag}_fde{k}_w1"] = fss.full_domain_eval(k1, n).words
    out["cases"] = np.array(cases)
    # predicate-family keys through the public generators (serialized)
    fam = []
    g = np.random.default_rng(77)
    for kind, ops, n in (("eq", (5,), 16), ("lt", (10,), 64), ("le", (63,), 64), ("gt", (3,), 100),
                         ("ge", (0,), 8), ("iv", (30, 40), 128), ("iv", (0, 127), 128)):
        if kind == "iv":
            pair = fss.ic_gen(ops[0], ops[1], n, g)
        elif kind == "eq":
            pair = fss.dpf_gen(ops[0], n, g)
        else:
            pair = fss.cmp_gen(kind, ops[0], n, g)
        name = f"fam_{kind}_{'_'.join(map(str, ops))}_n{n}"
        fam.append(name)
        out[f"{name}_k0"] = np.frombuffer(fss.serialize_key(pair[0]), np.uint8)
        out[f"{name}_k1"] = np.frombuffer(fss.serialize_key(pair[1]), np.uint8)
        out[f"{name}_fde0"] = fss.full_domain_eval(pair[0], n).words
        out[f"{name}_fde1"] = fss.full_domain_eval(pair[1], n).words
        out[f"{name}_n"] = np.array(n)
    out["families"] = np.array(fam)
    np.savez_compressed(OUT / "fss.npz", **out)


def prf_fixture(prf):
    from cryptography.hazmat.primitives.ciphers import Cipher, algorithms, modes

    rng = np.random.default_rng(31337)
    out = {}
    keys = rng.integers(0, 256, (4, 16), dtype=np.uint8)
    pts = rng.integers(0, 256, (4, 64), dtype=np.uint8)
    cts = []
    for k, p in zip(keys, pts):
        enc = Cipher(algorithms.AES(k.tobytes()), modes.ECB()).encryptor()
        cts.append(np.frombuffer(enc.update(p.tobytes()) + enc.finalize(), np.uint8))
    out.update(aes_keys=keys, aes_pt=pts, aes_ct=np.stack(cts))
    seeds = rng.integers(0, 2**63, size=(64, 2), dtype=np.uint64)
    seeds[0] = 0
    l, r, tl, tr, v = prf.prg_expand(seeds)
    out.update(prg_seeds=seeds, prg_left=l, prg_right=r, prg_tl=tl, prg_tr=tr, prg_v=v)
    streams = []
    for i, (label, index, nbytes) in enumerate(((b"ZSHR", 0, 64), (b"ZSHR", 7, 1000), (b"SHTB", 3, 33),
                                                 (b"SHPI", (1 << 40) + 5, 160), (b"SHRD", 0, 1))):
        key = keys[i % 4].tobytes()
        out[f"prf{i}_key"] = keys[i % 4]
        out[f"prf{i}_label"] = np.frombuffer(label, np.uint8)
        out[f"prf{i}_index"] = np.array(index, dtype=np.uint64)
        out[f"prf{i}_bytes"] = np.frombuffer(prf.prf_stream(key, label, index, nbytes), np.uint8)
        streams.append(i)
    out["prf_cases"] = np.array(streams)
    for i, n in enumerate((1, 2, 3, 17, 1000, 4097)):
        key = keys[(i + 1) % 4].tobytes()
        out[f"perm{i}_key"] = keys[(i + 1) % 4]
        out[f"perm{i}_n"] = np.array(n)
        out[f"perm{i}_tid"] = np.array(i)
        out[f"perm{i}_perm"] = prf.seeded_permutation(key, b"SHPI", i, n)
    out["perm_cases"] = np.arange(6)
    np.savez_compressed(OUT / "prf.npz", **out)


def zero_share_fixture(rss):
    keys = [bytes([i + 1]) * 16 for i in range(3)]
    ctxs = [rss.ZeroShareContext(keys[0], keys[2]), rss.ZeroShareContext(keys[1], keys[0]),
            rss.ZeroShareContext(keys[2], keys[1])]
    out = {"keys": np.stack([np.frombuffer(k, np.uint8) for k in keys])}
    for j, nbits in enumerate((1, 31, 32, 77, 1000)):
        for p in range(3):
            out[f"zs{j}_p{p}"] = ctxs[p].peek(nbits, j + 3).words
        out[f"zs{j}_nbits"] = np.array(nbits)
        out[f"zs{j}_counter"] = np.array(j + 3)
    np.savez_compressed(OUT / "zero_share.npz", **out)


def main():
    sys.path.insert(0, str(REF))
    from oblivgm import fss, prf, rss

    prf_fixture(prf)
    fss_fixture(fss, prf)
    zero_share_fixture(rss)
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()
