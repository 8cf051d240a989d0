"""Graph outsourcing (src/graphs.py:335-400): host dealer + upload
(encrypt_graph + device_trio) against the device dealer
(dealer.encrypt_graph_device), on the C1 graph and a larger synthetic one;
the shares are compared byte for byte."""

import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2209_03526_b200 import workloads  # noqa: E402
from paper_2209_03526_b200.dealer import encrypt_graph_device  # noqa: E402
from paper_2209_03526_b200.graphs import device_trio, encrypt_graph  # noqa: E402


def run(name, graph, k=2, seed=1):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, host = encrypt_graph(graph, k, np.random.default_rng(seed))
    d_host = device_trio(host)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    _, d_dev = encrypt_graph_device(graph, k, np.random.default_rng(seed))
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    same = all(torch.equal(d_dev[p].types[t].id_a.cpu(), d_host[p].types[t].id_a.cpu()) and
               all(torch.equal(d_dev[p].types[t].posting[c][0].cpu(), d_host[p].types[t].posting[c][0].cpu())
                   for c in d_host[p].types[t].posting)
               for p in range(3) for t in d_host[p].types)
    nbytes = sum(x.numel() * 4 for t in d_dev[0].types.values()
                 for x in [t.id_a] + [a[0] for a in t.attrs.values()] + [p_[0] for p_ in t.posting.values()]) * 3
    print(f"{name}: host dealer + upload {1e3 * (t1 - t0):.1f} ms, device dealer {1e3 * (t2 - t1):.1f} ms, "
          f"{nbytes / 1e9:.2f} GB of shares, identical={same}", flush=True)


def main():
    run("C1 (1000 vertices)", workloads.tiny_graph(1))
    for n in (10_000, 30_000):
        run(f"{n} vertices, 3 types, degree 5", workloads.tiny_graph(7, n=n))


if __name__ == "__main__":
    main()
