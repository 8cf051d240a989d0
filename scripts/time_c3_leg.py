"""C3 root slot (bench_configs.c3_leg) a few times: python scripts/time_c3_leg.py [repeats]."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import bench_configs as bc  # noqa: E402
from paper_2209_03526_b200 import _lib  # noqa: E402

_lib.check(_lib.load().ogm_init())
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    e = bc.c3_leg(5, 3)
    print(json.dumps({k: e[k] for k in ("ms", "secEval_combine_ms", "fetch_online_ms", "fetch_hbm_frac", "gate")}),
          flush=True)
