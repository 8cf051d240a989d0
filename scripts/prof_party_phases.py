"""Per-party C1 path: wall time per meter phase per party thread (monkeypatched Meter.phase)."""
import collections
import sys
import threading
import time
from contextlib import contextmanager

sys.path.insert(0, ".")
import numpy as np

from paper_2209_03526_b200 import net, workloads
from paper_2209_03526_b200.engine import EngineConfig, open_results, sec_match
from paper_2209_03526_b200.graphs import device_trio, encrypt_graph
from paper_2209_03526_b200.net import local_runtimes, make_session_configs, run_trio
from paper_2209_03526_b200.query import gen_token, load_query

g = workloads.tiny_graph(1)
q = workloads.tiny_query(g, 1)
rng = np.random.default_rng(1)
schema, shares = encrypt_graph(g, 2, rng)
d = device_trio(shares)
tokens = gen_token(load_query(q, schema), schema, rng)
acc = collections.defaultdict(float)
cnt = collections.Counter()
lock = threading.Lock()
orig = net.Meter.phase


@contextmanager
def phase(self, name):
    t = time.perf_counter()
    with orig(self, name):
        yield
    dt = time.perf_counter() - t
    with lock:
        acc[(threading.current_thread().name, name)] += dt
        cnt[(threading.current_thread().name, name)] += 1


net.Meter.phase = phase


def one():
    rts = local_runtimes(make_session_configs(b"\x5a" * 16))
    res = run_trio(lambda rt: sec_match(rt, tokens[rt.index - 1], d[rt.index - 1], EngineConfig()), rts)
    open_results(res[:2], schema)


for _ in range(5):
    one()
acc.clear()
cnt.clear()
N = 20
t = time.perf_counter()
for _ in range(N):
    one()
print(f"per query {(time.perf_counter() - t) / N * 1e3:.2f} ms")
for k in sorted(acc):
    print(f"  {k[0]:10s} {k[1]:24s} {acc[k] / N * 1e3:8.3f} ms/query  {cnt[k] / N:6.1f} calls/query")
