"""C4 root slot end to end at BASELINE size with its phase split
(bench_configs.c4_root_slot): python scripts/time_c4_root_slot.py [rows]."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import bench_configs as bc  # noqa: E402
from paper_2209_03526_b200 import _lib  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
_lib.check(_lib.load().ogm_init())
e = bc.c4_root_slot(rows, 0, 10, 3, 0, 1)
print(json.dumps({k: e[k] for k in ("ms", "phases_ms", "rank0_secEval_hbm_frac", "gate")}))
