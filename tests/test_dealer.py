"""Graph outsourcing on the device (dealer.py, csrc/ogm_dealer.cuh) against
the host dealer and numpy's generator (src/graphs.py:327-400)."""

import json

import numpy as np
import pytest


def test_pcg64_jump_model_matches_numpy():
    """The closed-form PCG64 jump and XSL-RR output (used to advance the host
    generator after a device draw) reproduce numpy's stream at any offset."""
    from paper_2209_03526_b200.dealer import _advance, _output

    rng = np.random.default_rng(2209)
    st = rng.bit_generator.state
    s, inc = st["state"]["state"], st["state"]["inc"]
    want = rng.integers(0, 1 << 32, size=2 * 5000, dtype=np.uint32)
    for j in (0, 1, 2, 17, 4095, 4999):
        o = _output(_advance(s, inc, j + 1))
        assert (int(want[2 * j]), int(want[2 * j + 1])) == (o & 0xFFFFFFFF, o >> 32), j


@pytest.mark.gpu
@pytest.mark.parametrize("skip", [0, 1, 2, 7])
@pytest.mark.parametrize("n", [0, 1, 2, 3, 1000, (1 << 20) + 1])
def test_draw_u32_matches_numpy(skip, n):
    import torch

    from paper_2209_03526_b200.dealer import draw_u32

    host, dev = np.random.default_rng(99), np.random.default_rng(99)
    host.integers(0, 1 << 32, size=skip, dtype=np.uint32)      # odd skips leave a buffered high half
    dev.integers(0, 1 << 32, size=skip, dtype=np.uint32)
    want = host.integers(0, 1 << 32, size=n, dtype=np.uint32)
    got = draw_u32(dev, n, "cuda").cpu().numpy().view(np.uint32)
    assert np.array_equal(got, want)
    assert dev.bit_generator.state == host.bit_generator.state
    # the generator continues identically afterwards
    assert np.array_equal(dev.integers(0, 1 << 32, size=5, dtype=np.uint32),
                          host.integers(0, 1 << 32, size=5, dtype=np.uint32))
    torch.cuda.synchronize()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["campus", "c1", "rand0", "rand1", "rand2"])
def test_device_dealer_equals_host_dealer(golden, name):
    """Every share component dealt on the device equals the host dealer's
    (and so the reference's: tests/test_frontend.py), the generator ends in
    the same state (tokens drawn next are identical), and a full trio
    sec_match over the device-dealt shares reproduces the reference's run."""
    import torch

    from paper_2209_03526_b200.dealer import encrypt_graph_device
    from paper_2209_03526_b200.engine import open_results
    from paper_2209_03526_b200.graphs import device_trio, encrypt_graph, parse_graph_text
    from paper_2209_03526_b200.query import gen_token, load_query, serialize_token
    from paper_2209_03526_b200.trio import Trio

    rec = json.loads(str(golden("match")[f"{name}_json"]))
    graph = parse_graph_text(rec["graph"])
    rh, rd = np.random.default_rng(rec["seed"]), np.random.default_rng(rec["seed"])
    schema_h, host = encrypt_graph(graph, rec["k"], rh)
    schema_d, dev = encrypt_graph_device(graph, rec["k"], rd)
    assert schema_d.digest() == schema_h.digest()
    assert rd.bit_generator.state == rh.bit_generator.state
    ref = device_trio(host)
    h = lambda t: t.cpu().numpy().view(np.uint32)  # noqa: E731
    for p in range(3):
        for t, s in ref[p].types.items():
            d = dev[p].types[t]
            assert np.array_equal(h(d.id_a), h(s.id_a)) and np.array_equal(h(d.id_b), h(s.id_b)), (t, "id")
            for a in s.attrs:
                assert np.array_equal(h(d.attrs[a][0]), h(s.attrs[a][0])), (t, a)
            for c in s.posting:
                assert np.array_equal(h(d.posting[c][0]), h(s.posting[c][0])), (t, c)
                assert np.array_equal(h(d.posting[c][1]), h(s.posting[c][1])), (t, c)
    tokens = gen_token(load_query(rec["query"], schema_d), schema_d, rd)
    assert [serialize_token(t).hex() for t in tokens] == rec["tokens"]
    res = Trio(bytes.fromhex(rec["master"])).match(list(tokens), list(dev), any_mode=rec["mode"])
    matches, _ = open_results(res.party_results()[:2], schema_d)
    assert sorted(list(m) for m in set(matches)) == rec["matches"]
    assert [list(sg) for sg in res.subgraphs] == rec["subgraphs"]
    torch.cuda.synchronize()
