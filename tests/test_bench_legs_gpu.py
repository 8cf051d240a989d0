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


def _c4_gloo_worker(rank, world, port, out_dir):
    import json
    import os

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import bench_configs
    from paper_2209_03526_b200 import _lib
    _lib.check(_lib.load().ogm_init())
    sec = bench_configs.c4_sec_eval(200_000, 1, 1, 1, rank, world)
    slot = bench_configs.c4_root_slot(200_000, 1, 1, 1, rank, world)
    with open(os.path.join(out_dir, f"r{rank}.json"), "w") as f:
        json.dump({"sec_gate": (sec.get("parity_gate") or {}).get("equal_to_oracle"), "slot_gate": slot["gate"],
                   "kept": slot["kept"], "matches": slot["matches"], "n_gpus": sec["n_gpus"]}, f)
    dist.destroy_process_group()


def test_c4_legs_two_gloo_ranks(tmp_path):
    """bench.py's C4 legs (sharded secEval with its N-rank parity gate, and
    the sharded root slot) under a 2-rank process group -- the code the
    driver's multi-GPU bench runs -- over gloo on one GPU (collectives staged
    through the host; a logic check, not a timing)."""
    import json
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_c4_gloo_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0 = json.loads((tmp_path / "r0.json").read_text())
    r1 = json.loads((tmp_path / "r1.json").read_text())
    assert r0["sec_gate"] is True and r0["n_gpus"] == 2
    for r in (r0, r1):
        assert all(r["slot_gate"].values()), r
        assert r["kept"] == r["matches"] == r0["matches"]


def test_bench_json_contract_small():
    """bench.py end to end at a small key count (secondary legs off): one JSON
    line carrying the contract's keys -- metric, value, ms_per_step, roofline,
    cpu_baseline, e2e with its byte counts, gpu_launches and clocks."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    out = subprocess.run([sys.executable, "bench.py", "--keys", "65536", "--steps", "3", "--warmup", "3",
                          "--no-c3", "--no-c4", "--no-c5", "--no-live-ref", "--no-query", "--cpu-seconds", "0.5"],
                         cwd=root, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "dtype", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["value"] > 0 and d["gpu_launches"] == 3
    assert 0 < d["roofline"]["frac"] and d["roofline"]["unit"] == "Tops/s"
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["value"] > 0
