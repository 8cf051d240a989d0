#!/usr/bin/env python
"""Headline benchmark: batched DCF evaluation, 32-bit domain (BASELINE config 2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1]): 2^24 independent DCF keys over a 32-bit
domain, random thresholds, one random uint32 point per key; a step evaluates
every key at its point (src/fss.py:288 dcf_eval == _walk_eval).  Synthetic,
seeded inputs (keys generated on the device by ogm_fss_gen from seeded roots).

* ``value``  -- evals/s with keys resident in HBM (9.1 GB > the 126 MB L2, so
  no flush is needed between steps), device-timed with CUDA events.
* ``e2e``    -- the same metric through the C ABI's host-buffer entry point
  (ogm_fss_eval_points_host): pinned host keys -> H2D -> eval -> D2H bits,
  every step, wall-clocked around the synchronous call.
* ``roofline`` -- integer-ALU bound: algorithmic work is
  2 int ops per AES table lookup of the minimal T-table walk (DCF: 31 levels x
  (160 + 133) + 133 = 9216 lookups/eval), against the measured LOP3 issue
  rate of this GPU (ogm_measure_int_peak).
* ``paired`` -- the paired DPF run of the same shapes (BASELINE configs[1]),
  device-timed the same way (``--kind dpf`` makes DPF the headline and DCF
  the pair).
* ``query_latency`` -- the metric's second half (BASELINE: "... and end-to-end
  query latency"): the C1 tiny oblivious match, tokens in -> reconstructed
  matches, via the trio fast path and via the per-party drop-in API, both
  checked against the plaintext matcher (rank 0).
* ``c4_sec_eval`` -- the 16M-vertex config (BASELINE configs[3]): root-slot
  secEval over 2M candidates, rows sharded over all N ranks with an NCCL
  all-gather of the match bits (strong scaling, max over ranks).
* ``cpu_baseline`` -- the CPU oracle port (oracle/, C, all host threads) on a
  bounded sample of the same workload, rank 0 only.

Multi-GPU: the key batch partitions (independent keys), so each rank
evaluates its own 2^24 keys with no data-path collective: weak scaling,
value = all ranks' evals / max-over-ranks time.

``--impl reference`` times the reference algorithm's CPU implementation
(the oracle port, all host threads) on the same config and prints the same
JSON line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import ctypes
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "dcf_evals_per_sec_32bit"
UNIT = "evals/s"
BITS = 32
DEFAULT_KEYS = 1 << 24
LOOKUPS = {"dcf": 31 * (160 + 133) + 133, "dpf": 32 * (160 + 133)}
OPS_PER_LOOKUP = 2
# dram__bytes_read.sum + dram__bytes_write.sum of one fss_eval_kernel launch at
# 2^24 DCF keys (profiles/r01_fss_eval_full_ncu.csv): 8,877,741,568 + 5,532,672
NCU_TRAFFIC = {("dcf", DEFAULT_KEYS): 8877250000 + 6400768}   # profiles/r02_fss_eval_ncu.txt (read + write)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--kind", choices=["dcf", "dpf"], default="dcf")
    p.add_argument("--keys", type=int, default=DEFAULT_KEYS)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    p.add_argument("--no-query", action="store_true", help="skip the C1 end-to-end query latency")
    p.add_argument("--query-steps", type=int, default=10)
    p.add_argument("--no-c4", action="store_true", help="skip the C4 sharded secEval leg")
    p.add_argument("--no-paired", action="store_true", help="skip the paired DPF (or DCF) run")
    p.add_argument("--no-c5", action="store_true", help="skip the C5 shuffle/fetch leg")
    p.add_argument("--no-c3", action="store_true", help="skip the C3 root-slot leg")
    p.add_argument("--no-live-ref", action="store_true",
                   help="skip timing the live reference (baseline/_ref) on this host")
    p.add_argument("--c5-logs", default="24,28", help="C5 table sizes (log2 rows), comma separated")
    p.add_argument("--ref-keys", type=int, default=1 << 22, help="keys per reference-arm step")
    p.add_argument("--dry-run", action="store_true",
                   help="launcher check without a GPU: ranks join a gloo group and rank 0 prints the line")
    return p.parse_args()


def free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_ranks(args) -> int | None:
    """``--gpus N`` outside torchrun: re-run this script under
    torch.distributed.run with N ranks, one per GPU (the driver's own launch
    line), and return its exit code.  Inside torchrun: None, after checking
    that WORLD_SIZE agrees with --gpus."""
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is not None:
        if int(env_world) != args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world}")
        return None
    if args.gpus <= 1:
        return None
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def run_dry(args):
    """The launcher without a GPU: every rank joins a gloo group, the group's
    size is checked with one all-reduce, rank 0 prints the JSON line shape."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    seen = world
    if world > 1:
        dist.init_process_group("gloo")
        t = torch.ones(1)
        dist.all_reduce(t)
        seen = int(t.item())
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world, "dry_run": True,
                          "comm_ranks": seen, "config": config_for(args, world)}), flush=True)


def config_for(args, world: int) -> dict:
    """The workload description both arms print (same keys)."""
    return {"workload": f"C2 batched {args.kind.upper()} micro (BASELINE configs[1])",
            "keys_per_gpu": args.keys, "domain_bits": BITS, "points_per_key": 1,
            "parallelism": f"key-sharded x{world}",
            "l2": "inputs (9.1 GB of keys) larger than L2; no flush"}


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sms, maxes, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sms.append(float(parts[0]))
                maxes.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sms) if sms else None,
                "sm_max_mhz": max(maxes) if maxes else None,
                "reasons": sorted(reasons), "samples": len(sms)}


# ---------------------------------------------------------------------------
# CPU legs (oracle port; only here and in tests)
# ---------------------------------------------------------------------------


def cpu_keys(kind: str, n: int, seed: int):
    import oracle
    rng = np.random.default_rng(seed)
    alphas = rng.integers(0, 1 << BITS, size=n, dtype=np.uint64)
    pts = rng.integers(0, 1 << BITS, size=n, dtype=np.uint64)
    r0 = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    r1 = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    k0, _ = oracle.tree_gen_batch(alphas, BITS, r0, r1, kind == "dcf")
    return k0, pts


def cpu_eval_rate(kind: str, target_seconds: float, threads: int):
    """evals/s of the oracle port on a bounded sample sized to ~target_seconds."""
    import oracle
    k0, pts = cpu_keys(kind, 4096, 1)
    t = time.perf_counter()
    oracle.eval_points(k0, pts, nthreads=threads)
    rate = 4096 / max(time.perf_counter() - t, 1e-6)
    n = int(min(max(rate * target_seconds, 4096), DEFAULT_KEYS)) // 32 * 32
    k0, pts = cpu_keys(kind, n, 2)
    t = time.perf_counter()
    oracle.eval_points(k0, pts, nthreads=threads)
    dt = time.perf_counter() - t
    return n / dt, n, dt


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    """The reference's CPU implementation of the path (the oracle/ C port of
    src/fss.py:257-281 -- the reference itself is pure Python with no
    compiled path), all host threads, on the GPU arm's config: each step
    evaluates ``--ref-keys`` (default 2^22) of the workload's keys.  The rate
    is taken from the median step: a busy host shows up as a few slow steps
    (0.86-0.90 s typical, up to 1.12 s seen), and the median -- the
    reference's steady rate -- only favours the reference."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return
    import oracle
    oracle.build()
    threads = os.cpu_count() or 1
    sample = min(args.ref_keys, args.keys)
    k0, pts = cpu_keys(args.kind, sample, 3)
    for _ in range(args.warmup):
        oracle.eval_points(k0, pts, nthreads=threads)
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        oracle.eval_points(k0, pts, nthreads=threads)
        times.append(time.perf_counter() - t)
    tot = sum(times)
    med = statistics.median(times)
    value = sample / med
    desc = (f"{sample} of the {args.keys} keys per step ({args.kind.upper()}, 32-bit domain), "
            f"oracle/ C port of src/fss.py:257-281, {threads} threads on {cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * med,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "config": config_for(args, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "step_s": {"min": min(times), "max": max(times), "median": med, "mean": tot / args.steps},
        "rate_from": "median step",
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU leg
# ---------------------------------------------------------------------------


def query_latency(steps: int) -> dict:
    """The metric's second half: end-to-end latency of the C1 tiny oblivious
    match (BASELINE configs[0]) on this GPU -- tokens in, result shares
    reconstructed on the host -- through the trio fast path and through the
    per-party drop-in API (run_trio + sec_match + open_results), each checked
    against the plaintext matcher."""
    import torch

    import oracle.matcher as om
    from paper_2209_03526_b200 import workloads
    from paper_2209_03526_b200.engine import EngineConfig, open_results, sec_match
    from paper_2209_03526_b200.graphs import device_trio, encrypt_graph
    from paper_2209_03526_b200.net import local_runtimes, make_session_configs, run_trio
    from paper_2209_03526_b200.query import gen_token, load_query
    from paper_2209_03526_b200.trio import Trio

    graph = workloads.tiny_graph(1)
    rng = np.random.default_rng(1)
    schema, shares = encrypt_graph(graph, 2, rng)
    dshares = device_trio(shares)
    query = load_query(workloads.tiny_query(graph, 1), schema)
    tokens = gen_token(query, schema, rng)
    want = om.oracle_match(graph, query, schema)
    master = b"\x5a" * 16

    def trio():
        res = Trio(master).match(list(tokens), list(dshares))
        return set(res.open(schema)[0])   # == open_results(res.party_results()[:2], schema), tested

    def per_party():
        rts = local_runtimes(make_session_configs(master))
        res = run_trio(lambda rt: sec_match(rt, tokens[rt.index - 1], dshares[rt.index - 1], EngineConfig()), rts)
        return set(open_results(res[:2], schema)[0])

    out = {"workload": "C1 tiny: 1000 vertices, 3 types, 3-vertex path (eq + range + always-true), k=2",
           "unit": "ms", "steps": steps}
    for name, fn in (("trio_ms", trio), ("per_party_ms", per_party)):
        for _ in range(3):
            got = fn()
        lat = []
        for _ in range(steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            got = fn()
            lat.append(1e3 * (time.perf_counter() - t0))
        out[name] = statistics.median(lat)
        out[name.replace("_ms", "_oracle_equal")] = got == want
    out["matches"] = len(want)
    out["match_list"] = sorted(list(m) for m in want)
    return out


def c5_legs(args, world: int) -> dict:
    """BASELINE configs[4] at each --c5-logs size: the 128-bit shuffle and
    the fetch of 1%, 10% and 100% of 129-bit rows (bench_configs.c5_*_leg),
    each with hbm_frac, a bit-exactness gate and the oracle port beside it.
    Under torchrun every rank shuffles its own tables (replicas, weak
    scaling); ms is the max over ranks."""
    import torch
    import torch.distributed as dist

    import bench_configs

    def worst(ms: float) -> float:
        if world == 1:
            return ms
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    peak = bench_configs.HBM_PEAK
    out = {"workload": "C5 shuffle/fetch sweep (BASELINE configs[4]): 128-bit rows x 3 share components; "
                       "fetch rows = flag + 128-bit id (129 bits)", "unit": "ms", "hbm_peak_GBps": peak,
           "scaling": "weak (replicas)" if world > 1 else None, "shuffle": [], "fetch": []}
    torch.cuda.empty_cache()
    for lg in [int(x) for x in args.c5_logs.split(",") if x]:
        gc.collect()
        sh = bench_configs.c5_shuffle_leg(lg, args.steps, args.warmup)
        gc.collect()
        fe = bench_configs.c5_fetch_leg(lg, args.steps, args.warmup)
        for e, per_row in [(sh, 240)] + [(f, f["algorithmic_bytes_per_row"]) for f in fe]:
            e["ms"] = worst(e["ms"])
            e["GBps"] = per_row * e["rows"] / (e["ms"] * 1e-3) / 1e9
            e["hbm_frac"] = e["GBps"] / peak
            e["rows_per_s_all_ranks"] = world * e["rows"] / (e["ms"] * 1e-3)
        out["shuffle"].append(sh)
        out["fetch"].extend(fe)
        gc.collect()
        torch.cuda.empty_cache()
    return out


def guarded(name: str, fn):
    """A secondary leg: its failure (an out-of-memory, a missing package) is
    recorded in the line instead of losing the headline.  Bit-exactness gates
    raise SystemExit and are NOT caught: a wrong result is never reported."""
    gc.collect()   # the previous leg's garbage is collected here, never inside a timed region
    try:
        return fn()
    except Exception as exc:  # noqa: BLE001
        import traceback
        traceback.print_exc()
        try:
            import torch
            torch.cuda.empty_cache()
        except Exception:  # noqa: BLE001
            pass
        return {"error": f"{name}: {type(exc).__name__}: {exc}"[:500]}


def main():
    args = parse()
    rc = launch_ranks(args)
    if rc is not None:
        sys.exit(rc)
    if args.dry_run:
        run_dry(args)
        return
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    from paper_2209_03526_b200 import _lib, fss

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    comm_ranks = world
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")   # communicator size visible in the log
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        ones = torch.ones(1, device="cuda")
        dist.all_reduce(ones)
        comm_ranks = int(ones.item())
    lib = _lib.load()
    _lib.check(lib.ogm_init())
    # Automatic garbage collection is off for the GPU arm (timeit's convention): a generation-2
    # collection left pending by the query leg's many small objects otherwise lands inside a later
    # leg's timed loop and stalls its host-driven launches (C4 secEval 1.08 -> 3.1-4.2 ms measured);
    # every leg starts with an explicit collection (guarded).
    gc.collect()
    gc.disable()

    K = args.keys
    comparison = args.kind == "dcf"
    gen = torch.Generator(device="cuda").manual_seed(1234 + rank)
    alphas = torch.randint(-(1 << 31), 1 << 31, (K,), dtype=torch.int32, device="cuda", generator=gen)
    pts = torch.randint(-(1 << 31), 1 << 31, (K,), dtype=torch.int32, device="cuda", generator=gen)
    r0 = torch.randint(0, 256, (K, 16), dtype=torch.uint8, device="cuda", generator=gen)
    r1 = torch.randint(0, 256, (K, 16), dtype=torch.uint8, device="cuda", generator=gen)
    b0, b1 = fss.gen_batch(comparison, BITS, alphas, r0, r1)
    del r1
    out = torch.empty(((K + 31) // 32,), dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()

    # correctness gate on the bench inputs: pair XOR == indicator
    o1 = torch.empty_like(out)
    fss.eval_points(b0, pts, out)
    fss.eval_points(b1, pts, o1)
    x = (out ^ o1).cpu().numpy().view(np.uint8)
    got = np.unpackbits(x, bitorder="little")[:K]
    a = alphas.cpu().numpy().view(np.uint32)
    p = pts.cpu().numpy().view(np.uint32)
    want = (p < a) if comparison else (p == a)
    if not np.array_equal(got, want.astype(np.uint8)):
        raise SystemExit("bench correctness gate failed: pair XOR != indicator")
    del o1, b1

    peak = ctypes.c_double()
    secs = ctypes.c_double()
    _lib.check(lib.ogm_measure_int_peak(ctypes.byref(peak), ctypes.byref(secs)))

    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        fss.eval_points(b0, pts, out)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    ev[0].record(stream)
    for s in range(args.steps):
        fss.eval_points(b0, pts, out)
        ev[s + 1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    per_launch = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
    total_ms = ev[0].elapsed_time(ev[-1])
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    ms_per_step = max_ms / args.steps
    value = world * K * args.steps / (max_ms * 1e-3)
    avg_launch_s = statistics.mean(per_launch) * 1e-3
    ops_per_eval = OPS_PER_LOOKUP * LOOKUPS[args.kind]
    achieved = K * ops_per_eval / avg_launch_s
    roofline = {"bound": "int_alu", "achieved": achieved / 1e12, "peak": peak.value / 1e12,
                "unit": "Tops/s", "frac": achieved / peak.value,
                "traffic": NCU_TRAFFIC.get((args.kind, K)),
                "traffic_source": "ncu --set full dram__bytes_read+write per launch, profiles/r02_fss_eval_ncu.txt",
                "algorithmic_key_bytes_per_launch": K * (16 + 16 * (BITS - (1 if comparison else 0)) + 12 + 1 + 4),
                "binding_pipe": "LSU (shared-memory T-table lookups) 93.5% / ALU 83.7% of peak (ncu)",
                "ops_per_eval": ops_per_eval, "aes_lookups_per_eval": LOOKUPS[args.kind],
                "peak_source": "ogm_measure_int_peak (LOP3 issue rate, this run)",
                "key_bytes_per_eval": 16 + 16 * (BITS - (1 if comparison else 0)) + 12 + 1 + 4}

    # end-to-end through the C ABI from pinned host buffers
    e2e = None
    if not args.no_e2e:
        def pinned_copy(t_):  # straight into page-locked memory (no pageable staging copy per rank)
            h = torch.empty(t_.shape, dtype=t_.dtype, pin_memory=True)
            h.copy_(t_)
            return h

        host = [pinned_copy(t_) for t_ in (b0.root, b0.seed_cw, b0.ctrl, b0.flags, pts)]
        hout = torch.zeros(((K + 31) // 32,), dtype=torch.int32, pin_memory=True)
        kind = _lib.KIND_DCF if comparison else _lib.KIND_DPF
        fn = lib.ogm_fss_eval_points_host
        argv = [kind, BITS, K, *(_lib.ptr(h) for h in host), _lib.ptr(hout)]
        _lib.check(fn(*argv))  # warm-up (allocates the staging buffers)
        if not np.array_equal(hout.numpy(), out.cpu().numpy()):
            raise SystemExit("e2e result differs from the device-resident result")
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            _lib.check(fn(*argv))
        el = time.perf_counter() - t0
        tt = torch.tensor([el], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        # bytes the call copies: a DCF's last-level seed correction is never read, so not sent
        h2d = sum(h.numel() * h.element_size() for h in host) - (16 * K if comparison else 0)
        e2e = {"value": world * K * args.steps / float(tt.item()), "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": hout.numel() * 4,
               "ms_per_step": 1e3 * float(tt.item()) / args.steps}
        del host, hout

    # the paired run of the metric's other half: DPF (equality) keys of the same
    # shapes, device-timed the same way (BASELINE configs[1]: "A paired DPF run")
    paired = None
    if not args.no_paired:
        other = not comparison
        del b0
        torch.cuda.empty_cache()
        pb0, _ = fss.gen_batch(other, BITS, alphas, r0, torch.randint(0, 256, (K, 16), dtype=torch.uint8,
                                                                       device="cuda", generator=gen))
        for _ in range(args.warmup):
            fss.eval_points(pb0, pts, out)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        pev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        pev[0].record(stream)
        for _ in range(args.steps):
            fss.eval_points(pb0, pts, out)
        pev[1].record(stream)
        torch.cuda.synchronize()
        pt = torch.tensor([pev[0].elapsed_time(pev[1])], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(pt, op=dist.ReduceOp.MAX)
        kind_o = "dcf" if other else "dpf"
        paired = {"kind": kind_o, "value": world * K * args.steps / (float(pt.item()) * 1e-3), "unit": UNIT,
                  "ms_per_step": float(pt.item()) / args.steps,
                  "roofline_frac": (K * OPS_PER_LOOKUP * LOOKUPS[kind_o] / (float(pt.item()) * 1e-3 / args.steps))
                  / peak.value}
        b0 = pb0

    query = None
    if rank == 0 and not args.no_query:
        query = guarded("query_latency", lambda: query_latency(args.query_steps))

    # the 16M-vertex config (BASELINE configs[3]): row-sharded secEval over all ranks
    c4 = None
    if not args.no_c4:
        import bench_configs
        del b0, pts, out
        torch.cuda.empty_cache()
        c4 = guarded("c4_sec_eval", lambda: bench_configs.c4_sec_eval(2_000_000, 1, 10, 3, rank, world))
        torch.cuda.empty_cache()
        c4["root_slot"] = guarded("c4_root_slot",
                                  lambda: bench_configs.c4_root_slot(2_000_000, 1, 10, 3, rank, world))

    # C3 (BASELINE configs[2]): the medium graph's root slot on one GPU
    c3 = None
    if world == 1 and not args.no_c3:
        import bench_configs
        torch.cuda.empty_cache()
        c3 = guarded("c3_root_slot", lambda: bench_configs.c3_leg(args.steps, args.warmup))
        torch.cuda.empty_cache()

    # C5 (BASELINE configs[4]): shuffle and 1/10/100% fetch bandwidth, every rank its own tables
    c5 = None
    if not args.no_c5:
        c5 = guarded("c5", lambda: c5_legs(args, world))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        import oracle
        oracle.build()
        threads = os.cpu_count() or 1
        rate, n, dt = cpu_eval_rate(args.kind, args.cpu_seconds, threads)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{n} keys x 1 point ({args.kind.upper()}, 32-bit) in {dt:.1f}s, "
                         f"oracle/ C port of src/fss.py:257-281 on {cpu_model()}"}

    live = None
    if rank == 0 and world == 1 and not args.no_live_ref:
        import bench_reference
        live = guarded("live_reference",
                       lambda: bench_reference.live_reference([int(x) for x in args.c5_logs.split(",") if x]))
        if query is not None and "c1" in live:
            live["c1"]["matches_equal_ours"] = live["c1"]["matches"] == sorted(query.get("match_list", []))

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": config_for(args, world), "comm_ranks": comm_ranks,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "paired": paired, "query_latency": query,
            "c3_root_slot": c3, "c4_sec_eval": c4, "c5": c5, "live_reference": live,
            "gpu_launches": args.steps, "clocks": clk,
            "launch_ms": {"mean": statistics.mean(per_launch), "min": min(per_launch),
                          "max": max(per_launch)},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
