"""Per-phase SM-clock stamps of the scheduler kernel (HEP_SCHED_PROFILE) on
the BASELINE shapes; run on the GPU box.  ``--variants "sched_lexmin_warps=1,..."``
A/Bs hep_tuning variants (one JSON object per variant, plans / ranges compared with
the default's)."""
import ctypes
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2511_16947_b200 as P  # noqa: E402
from paper_2511_16947_b200 import _lib  # noqa: E402
from paper_2511_16947_b200.scheduler import DeviceScheduler  # noqa: E402

sys.path.insert(0, "tools")
from _tuning import apply  # noqa: E402

PHASES = ["stage+totals", "zeta+m", "lexmin", "integerize", "route", "transfer"]
variants = [""]
if "--variants" in sys.argv:
    variants += [v for v in sys.argv[sys.argv.index("--variants") + 1].split(",") if v]
base = _lib.get_tuning()
ref_out = {}
for var in variants:
  apply(var, base)
  out = {"variant": var or "default"}
  for name, E, K, T in (("mixtral", 8, 2, 16384), ("qwen3", 128, 8, 32768), ("dsv3", 256, 8, 16384)):
      G = 8
      pl = P.cayley_symmetric(P.ClusterShape(G, E, 2))
      wl = P.gen_zipf_workload(P.ClusterShape(G, E, 2), 1.0, (T // G) * K, 1, 0)
      ds = DeviceScheduler(pl)
      loads = torch.tensor(wl.micro_batches[0].as_array(), device="cuda")
      for _ in range(3):
          ds.launch_solve(loads, G, 1, None, 15 | 32)
      torch.cuda.synchronize()
      buf = np.zeros(16, dtype=np.int64)
      _lib.check(_lib.lib().hep_sched_debug_timing(buf.ctypes.data_as(_lib.c_i64p), 16), "timing")
      stamps = buf[:7]
      out[name] = {ph: int(stamps[i + 1] - stamps[i]) for i, ph in enumerate(PHASES)}
      out[name]["total_cycles"] = int(stamps[6] - stamps[0])
      ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
      ev0.record()
      for _ in range(100):
          ds.launch_solve(loads, G, 1, None, 15)
      ev1.record()
      torch.cuda.synchronize()
      out[name]["us_per_launch_back_to_back"] = ev0.elapsed_time(ev1) * 10
      res = (ds.rows(ds.xq), ds.rows(ds.xi), ds.host_ranges())
      if not var:
          ref_out[name] = res
      out[name]["same_as_default"] = res == ref_out[name]
  print(json.dumps(out, indent=1))
