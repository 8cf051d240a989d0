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


def _group_shares(values, domain, rng):
    """Candidate one-hot ids/attrs shared into three components (same draws
    as the reference test helper tests/test_engine.py:18-46)."""
    from oblivgm.bits import pack_bits

    count = len(values)
    id_bits = np.zeros((count, count), np.uint8)
    for i in range(count):
        id_bits[i, i] = 1
    attr_bits = np.zeros((count, domain), np.uint8)
    for i, v in enumerate(values):
        if v is not None:
            attr_bits[i, v] = 1
    comps = {}
    for name, mats in (("id", pack_bits(id_bits)), ("attr", pack_bits(attr_bits))):
        s1 = rng.integers(0, 1 << 32, size=mats.shape, dtype=np.uint32)
        s2 = rng.integers(0, 1 << 32, size=mats.shape, dtype=np.uint32)
        comps[name] = (s1, s2, mats ^ s1 ^ s2)
    return comps


def _groups(ref, comps, count, domain):
    from oblivgm.engine import CandidateGroup
    out = []
    for p in range(3):
        n = (p + 1) % 3
        out.append(CandidateGroup(None, None, count, count, comps["id"][p], comps["id"][n],
                                  {"a": (comps["attr"][p], comps["attr"][n])}, {"a": domain}))
    return out


def engine_fixture(ref):
    from oblivgm import fss, rss
    from oblivgm.bits import BitVector
    from oblivgm.engine import _OpenLabels, combine_predicates, sec_eval, sec_fetch_multi, sec_fetch_unique
    from oblivgm.net import local_runtimes, make_session_configs, run_trio

    out = {}
    cases = []
    # --- sec_eval: per-party output shares + transcripts (src/engine.py:139-165)
    ev_cases = [("eq", (5,), 16, [5, 7, 5, 0]), ("ge", (0,), 8, [None, 2, None]),
                ("lt", (40,), 128, list(range(0, 128, 3))), ("iv", (30, 40), 128, None),
                ("iv", (3, 200), 333, None), ("le", (63,), 64, None),
                ("iv", (100, 3000), 4000, None), ("eq", (77,), 2500, None)]
    for ci, (kind, ops, domain, values) in enumerate(ev_cases):
        rng = np.random.default_rng(100 + ci)
        if values is None:
            values = rng.integers(0, domain, size=97 if domain < 1000 else 203).tolist()
            if kind == "eq":
                values[::7] = [ops[0]] * len(values[::7])
        comps = _group_shares(values, domain, rng)
        groups = _groups(ref, comps, len(values), domain)
        if kind == "iv":
            pairs = tuple(fss.ic_gen(ops[0], ops[1], domain, rng) for _ in range(3))
        else:
            pairs = tuple(fss.bundle_gen(kind, ops, domain, rng).pairs)
        (k11, k21), (k12, k22), (k13, k23) = pairs
        keys = [(k11, k12), (k22, k13), (k23, k21)]
        master = bytes([0x30 + ci]) * 16
        runtimes = local_runtimes(make_session_configs(master))
        res = run_trio(lambda rt: sec_eval(rt, groups[rt.index - 1], keys[rt.index - 1], "a", domain), runtimes)
        tag = f"ev{ci}"
        cases.append(tag)
        out[f"{tag}_domain"] = np.array(domain)
        out[f"{tag}_count"] = np.array(len(values))
        out[f"{tag}_master"] = np.frombuffer(master, np.uint8)
        for c in range(3):
            out[f"{tag}_attr{c}"] = comps["attr"][c]
        for p in range(3):
            out[f"{tag}_key{p}_0"] = np.frombuffer(fss.serialize_key(keys[p][0]), np.uint8)
            out[f"{tag}_key{p}_1"] = np.frombuffer(fss.serialize_key(keys[p][1]), np.uint8)
            out[f"{tag}_out{p}_a"] = res[p].share_a.words
            out[f"{tag}_out{p}_b"] = res[p].share_b.words
            out[f"{tag}_digest{p}"] = np.frombuffer(bytes.fromhex(runtimes[p].transcript_digest()), np.uint8)
            out[f"{tag}_bits{p}"] = np.array(runtimes[p].meter.total.logical_bits)
            out[f"{tag}_bytes{p}"] = np.array(runtimes[p].meter.total.bytes_sent)
        out[f"{tag}_plain"] = rss.reconstruct(res).to_bits()
    out["ev_cases"] = np.array(cases)

    # --- combine_predicates (src/engine.py:168-189)
    cb = []
    for ci, (combiner, mode, cols) in enumerate((("ALL", "or", [[0, 0, 1, 1], [0, 1, 0, 1]]),
                                                 ("ANY", "or", [[0, 0, 1, 1], [0, 1, 0, 1]]),
                                                 ("ANY", "xor", [[0, 0, 1, 1], [0, 1, 0, 1]]),
                                                 ("ALL", "or", [[1, 1, 0] * 30, [1, 0, 1] * 30, [1, 1, 1] * 30]),
                                                 ("ANY", "or", [[1, 0, 0, 1, 0] * 20, [0, 0, 1, 1, 0] * 20,
                                                                [0, 1, 0, 0, 0] * 20]))):
        rng = np.random.default_rng(200 + ci)
        per_party = [[], [], []]
        comps = []
        for col in cols:
            sh = rss.share(BitVector.from_bits(col), rng)
            comps.append([sh[0].share_a.words, sh[1].share_a.words, sh[2].share_a.words])
            for p in range(3):
                per_party[p].append(sh[p])
        master = bytes([0x50 + ci]) * 16
        runtimes = local_runtimes(make_session_configs(master))
        res = run_trio(lambda rt: combine_predicates(rt, per_party[rt.index - 1], combiner, mode), runtimes)
        tag = f"cb{ci}"
        cb.append(tag)
        out[f"{tag}_combiner"] = np.array(combiner)
        out[f"{tag}_mode"] = np.array(mode)
        out[f"{tag}_n"] = np.array(len(cols[0]))
        out[f"{tag}_master"] = np.frombuffer(master, np.uint8)
        out[f"{tag}_comps"] = np.array(comps, dtype=np.uint32)
        for p in range(3):
            out[f"{tag}_out{p}_a"] = res[p].share_a.words
            out[f"{tag}_out{p}_b"] = res[p].share_b.words
            out[f"{tag}_digest{p}"] = np.frombuffer(bytes.fromhex(runtimes[p].transcript_digest()), np.uint8)
    out["cb_cases"] = np.array(cb)

    # --- fetch unique / multi (src/engine.py:197-270)
    fc = []
    for ci, (values, domain, flag_bits, unique) in enumerate(
            (([4, 9, 2, 7], 16, [0, 0, 1, 0], True), ([4, 9, 2, 7], 16, [0, 0, 0, 0], True),
             ([4, 9, 2, 7, 9], 16, [0, 1, 0, 1, 1], False), ([4, 9], 16, [0, 0], False),
             (list(range(40)), 64, [1, 0, 0, 1, 0, 1, 1, 0] * 5, False))):
        rng = np.random.default_rng(300 + ci)
        comps = _group_shares(values, domain, rng)
        groups = _groups(ref, comps, len(values), domain)
        fsh = rss.share(BitVector.from_bits(flag_bits), rng)
        master = bytes([0x70 + ci]) * 16
        runtimes = local_runtimes(make_session_configs(master))

        def worker(rt):
            g = groups[rt.index - 1]
            fl = fsh[rt.index - 1]
            if unique:
                return [sec_fetch_unique(rt, g, fl)], []
            audit = []
            return sec_fetch_multi(rt, g, fl, _OpenLabels(), audit), audit

        res = run_trio(worker, runtimes)
        tag = f"fe{ci}"
        fc.append(tag)
        out[f"{tag}_unique"] = np.array(unique)
        out[f"{tag}_domain"] = np.array(domain)
        out[f"{tag}_count"] = np.array(len(values))
        out[f"{tag}_master"] = np.frombuffer(master, np.uint8)
        for c in range(3):
            out[f"{tag}_id{c}"] = comps["id"][c]
            out[f"{tag}_attr{c}"] = comps["attr"][c]
            out[f"{tag}_flag{c}"] = fsh[c].share_a.words
        for p in range(3):
            recs, audit = res[p]
            out[f"{tag}_n{p}"] = np.array(len(recs))
            for r, rec in enumerate(recs):
                out[f"{tag}_p{p}_r{r}_id_a"] = rec.vertex_id.share_a.words
                out[f"{tag}_p{p}_r{r}_id_b"] = rec.vertex_id.share_b.words
                out[f"{tag}_p{p}_r{r}_at_a"] = rec.attrs["a"].share_a.words
                out[f"{tag}_p{p}_r{r}_at_b"] = rec.attrs["a"].share_b.words
            if audit:
                out[f"{tag}_audit{p}"] = audit[0][1]
            out[f"{tag}_digest{p}"] = np.frombuffer(bytes.fromhex(runtimes[p].transcript_digest()), np.uint8)
    out["fe_cases"] = np.array(fc)
    np.savez_compressed(OUT / "engine.npz", **out)


def shuffle_fixture(ref):
    from oblivgm import rss
    from oblivgm.bits import BitVector
    from oblivgm.net import local_runtimes, make_session_configs, run_trio
    from oblivgm.shuffle import MatchTable, sec_shuffle

    out = {}
    cases = []
    for ci, (rows, width, rounds) in enumerate(((1, 5, 1), (8, 45, 1), (37, 70, 2), (200, 129, 1), (64, 32, 1))):
        rng = np.random.default_rng(400 + ci)
        plain = [BitVector.random(width, rng) for _ in range(rows)]
        shares = [rss.share(r, rng) for r in plain]
        master = bytes([0x90 + ci]) * 16
        runtimes = local_runtimes(make_session_configs(master))

        def worker(rt):
            res = None
            for _ in range(rounds):
                res = sec_shuffle(rt, MatchTable.from_rows([shares[i][rt.index - 1] for i in range(rows)]))
            return res

        res = run_trio(worker, runtimes)
        tag = f"sh{ci}"
        cases.append(tag)
        out[f"{tag}_rows"] = np.array(rows)
        out[f"{tag}_width"] = np.array(width)
        out[f"{tag}_rounds"] = np.array(rounds)
        out[f"{tag}_master"] = np.frombuffer(master, np.uint8)
        for c in range(3):
            out[f"{tag}_in{c}"] = np.stack([shares[i][c].share_a.words for i in range(rows)])
        for p in range(3):
            out[f"{tag}_out{p}_a"] = res[p].share_a
            out[f"{tag}_out{p}_b"] = res[p].share_b
            out[f"{tag}_digest{p}"] = np.frombuffer(bytes.fromhex(runtimes[p].transcript_digest()), np.uint8)
            out[f"{tag}_bytes{p}"] = np.array(runtimes[p].meter.total.bytes_sent)
    out["cases"] = np.array(cases)
    np.savez_compressed(OUT / "shuffle.npz", **out)


def c5_fetch_fixture(ref):
    """sec_fetch_multi at the C5 fetch shape (src/engine.py:220-270): rows =
    flag bit + 128-bit id, no attributes, ~10% of the rows flagged; 4096
    rows (the largest size the pure-Python reference runs in seconds)."""
    from oblivgm import rss
    from oblivgm.bits import BitVector
    from oblivgm.engine import CandidateGroup, _OpenLabels, sec_fetch_multi
    from oblivgm.net import local_runtimes, make_session_configs, run_trio

    out = {}
    for ci, (rows, p) in enumerate(((4096, 0.1), (777, 0.01), (64, 1.0))):
        rng = np.random.default_rng(900 + ci)
        ids = [rng.integers(0, 1 << 32, size=(rows, 4), dtype=np.uint32) for _ in range(3)]
        plain = (rng.random(rows) < p).astype(np.uint8)
        fsh = rss.share(BitVector.from_bits(plain), rng)
        groups = [CandidateGroup(None, None, rows, 128, ids[q], ids[(q + 1) % 3], {}, {}) for q in range(3)]
        master = bytes([0xC5, ci]) * 8
        runtimes = local_runtimes(make_session_configs(master))

        def worker(rt):
            audit = []
            return sec_fetch_multi(rt, groups[rt.index - 1], fsh[rt.index - 1], _OpenLabels(), audit), audit

        res = run_trio(worker, runtimes)
        tag = f"cf{ci}"
        out[f"{tag}_rows"] = np.array(rows)
        out[f"{tag}_master"] = np.frombuffer(master, np.uint8)
        for c in range(3):
            out[f"{tag}_id{c}"] = ids[c]
            out[f"{tag}_flag{c}"] = fsh[c].share_a.words
        for q in range(3):
            recs, audit = res[q]
            out[f"{tag}_n{q}"] = np.array(len(recs))
            out[f"{tag}_ida{q}"] = (np.stack([r.vertex_id.share_a.words for r in recs]) if recs
                                    else np.zeros((0, 4), np.uint32))
            out[f"{tag}_idb{q}"] = (np.stack([r.vertex_id.share_b.words for r in recs]) if recs
                                    else np.zeros((0, 4), np.uint32))
            out[f"{tag}_audit{q}"] = audit[0][1]
            out[f"{tag}_digest{q}"] = np.frombuffer(bytes.fromhex(runtimes[q].transcript_digest()), np.uint8)
    out["cases"] = np.array([f"cf{i}" for i in range(3)])
    np.savez_compressed(OUT / "c5fetch.npz", **out)


CAMPUS = Path("/root/reference/pkg/demos/data/campus.graph")
TWO_PERSON = Path("/root/reference/pkg/demos/data/two-person.query")


def match_fixture(ref):
    """Full sec_match runs (src/engine.py:352-417): graph text, query text and
    seeds are recorded; the product regenerates shares/tokens from the same
    seeds (rng-compatible encrypt_graph / gen_token) and must reproduce every
    record share, opened flag, subgraph and transcript digest."""
    import json

    from oblivgm.datagen import graph_to_text, random_graph, random_query_text
    from oblivgm.engine import EngineConfig, open_results, sec_match
    from oblivgm.graphs import build_schema, encrypt_graph, parse_graph_text
    from oblivgm.net import local_runtimes, make_session_configs, run_trio
    from oblivgm.oracle import oracle_match
    from oblivgm.query import gen_token, load_query, serialize_token

    runs = [("campus", CAMPUS.read_text(), TWO_PERSON.read_text(), 2, 1, b"\x11" * 16, "or")]
    extra = [("unique-chain", "Q u U place = Harbin\nQ p P age = 40\nQ c C field = Internet\nQE u p\nQE p c\n"),
             ("conj", "Q u U place = Harbin\nQ p P age >= 35\nQ p P age <= 40\nQE u p\n")]
    for name, q in extra:
        runs.append((name, CAMPUS.read_text(), q, 2, 1, b"\x11" * 16, "or"))
    # BASELINE configs[0] (C1) exactly as bench.py builds it: 1000 vertices, 3 types, k = 2
    sys.path.insert(0, str(OUT.parent.parent))
    from paper_2209_03526_b200.graphs import parse_graph_text as our_parse
    from paper_2209_03526_b200.workloads import tiny_graph_text, tiny_query
    c1_text = tiny_graph_text(1)
    runs.append(("c1", c1_text, tiny_query(our_parse(c1_text), 1), 2, 1, b"\x5a" * 16, "or"))
    for trial in range(3):
        rng = np.random.default_rng(7000 + trial)
        g = random_graph(rng, n_vertices=int(rng.integers(90, 150)), n_types=3, avg_degree=5.0)
        schema = build_schema(g, 2 + trial % 2)
        qtext = random_query_text(rng, schema, n_targets=3, kinds=("eq", "lt", "iv"), multi_pred_prob=0.6)
        runs.append((f"rand{trial}", graph_to_text(g), qtext, 2 + trial % 2, trial, bytes([60 + trial]) * 16,
                     ("or", "xor")[trial % 2]))
    out = {"names": np.array([r[0] for r in runs])}
    for name, gtext, qtext, k, seed, master, mode in runs:
        graph = parse_graph_text(gtext)
        rng = np.random.default_rng(seed)
        schema, shares = encrypt_graph(graph, k, rng)
        query = load_query(qtext, schema)
        tokens = gen_token(query, schema, rng)
        runtimes = local_runtimes(make_session_configs(master))
        results = run_trio(lambda rt: sec_match(rt, tokens[rt.index - 1], shares[rt.index - 1],
                                                EngineConfig(any_mode=mode)), runtimes)
        matches, _ = open_results(results[:2], schema)
        want = oracle_match(graph, query, schema, any_mode=mode)
        assert set(matches) == want, name
        rec = {"graph": gtext, "query": qtext, "k": k, "seed": seed, "master": master.hex(), "mode": mode,
               "matches": sorted(list(m) for m in set(matches)),
               "subgraphs": [list(sg) for sg in results[0].subgraphs],
               "digests": [rt.transcript_digest() for rt in runtimes],
               "bytes": [rt.meter.total.bytes_sent for rt in runtimes],
               "tokens": [serialize_token(t).hex() for t in tokens],
               "schema_digest": schema.digest().hex()}
        out[f"{name}_json"] = np.array(json.dumps(rec))
        for p, res in enumerate(results):
            for s, recs in enumerate(res.records):
                for ri, r in enumerate(recs):
                    base = f"{name}_p{p}_s{s}_r{ri}"
                    out[f"{base}_id_a"] = r.vertex_id.share_a.words
                    out[f"{base}_id_b"] = r.vertex_id.share_b.words
                    for a in sorted(r.attrs):
                        out[f"{base}_{a}_a"] = r.attrs[a].share_a.words
                        out[f"{base}_{a}_b"] = r.attrs[a].share_b.words
            for j, (phase, bits) in enumerate(res.opened_flags):
                out[f"{name}_p{p}_open{j}"] = np.asarray(bits, np.uint8)
    np.savez_compressed(OUT / "match.npz", **out)


def storage_fixture(ref):
    """Reference-written files: campus schema, 3 graph shares (.ogmg), and the
    3 result files (.ogmr) of the two-person query (src/storage.py)."""
    import tempfile

    from oblivgm.engine import EngineConfig, sec_match
    from oblivgm.graphs import encrypt_graph, parse_graph_text
    from oblivgm.net import local_runtimes, make_session_configs, run_trio
    from oblivgm.query import gen_token, load_query
    from oblivgm.storage import save_graph_share, save_results, save_schema

    graph = parse_graph_text(CAMPUS.read_text())
    rng = np.random.default_rng(1)
    schema, shares = encrypt_graph(graph, 2, rng)
    tokens = gen_token(load_query(TWO_PERSON.read_text(), schema), schema, rng)
    runtimes = local_runtimes(make_session_configs(b"\x11" * 16))
    results = run_trio(lambda rt: sec_match(rt, tokens[rt.index - 1], shares[rt.index - 1], EngineConfig()),
                       runtimes)
    out = {}
    with tempfile.TemporaryDirectory() as d:
        save_schema(f"{d}/schema.json", schema)
        out["schema_json"] = np.frombuffer(open(f"{d}/schema.json", "rb").read(), np.uint8)
        for p in range(3):
            save_graph_share(f"{d}/g{p}.ogmg", shares[p])
            out[f"ogmg{p}"] = np.frombuffer(open(f"{d}/g{p}.ogmg", "rb").read(), np.uint8)
            save_results(f"{d}/r{p}.ogmr", results[p], schema)
            out[f"ogmr{p}"] = np.frombuffer(open(f"{d}/r{p}.ogmr", "rb").read(), np.uint8)
    np.savez_compressed(OUT / "storage.npz", **out)


def main():
    sys.path.insert(0, str(REF))
    if len(sys.argv) > 1:   # e.g. `make_golden.py c5_fetch_fixture`: regenerate the named fixtures only
        import oblivgm as ref
        for name in sys.argv[1:]:
            globals()[name](ref)
        return
    import oblivgm as ref
    from oblivgm import fss, prf, rss

    prf_fixture(prf)
    fss_fixture(fss, prf)
    zero_share_fixture(rss)
    engine_fixture(ref)
    shuffle_fixture(ref)
    match_fixture(ref)
    storage_fixture(ref)
    c5_fetch_fixture(ref)
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()
