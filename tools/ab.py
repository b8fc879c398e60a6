"""Same-box A/B timing of library variants (tools/variant.py builds): runs
tools/quick_time.py under CITO_LIB_VARIANT=<name> for each variant, interleaved
`rounds` times, and prints the per-variant medians.  (GPU box)

  python tools/ab.py <rounds> <variant> [<variant> ...] -- [quick_time args]
"""
import os
import re
import subprocess
import sys
from collections import defaultdict

import numpy as np

argv = sys.argv[1:]
rounds = int(argv[0])
rest = argv[1:]
qargs = rest[rest.index("--") + 1:] if "--" in rest else []
variants = rest[: rest.index("--")] if "--" in rest else rest
res = defaultdict(list)
for _ in range(rounds):
    for v in variants:
        env = dict(os.environ)
        if v != "main":
            env["CITO_LIB_VARIANT"] = v
        script = os.environ.get("AB_SCRIPT", "tools/quick_time.py")
        if ":" in v:  # variant:ENV=VALUE: a variant library with an environment switch
            lib, spec = v.split(":", 1)
            k, val = spec.split("=", 1)
            env["CITO_LIB_VARIANT"] = lib
            env[k] = val
        elif "=" in v:  # name=ENV=VALUE: the main library with an environment switch
            name, k, val = v.split("=", 2)
            env.pop("CITO_LIB_VARIANT", None)
            env[k] = val
        out = subprocess.run([sys.executable, script] + qargs, capture_output=True, text=True, env=env)
        for line in out.stdout.splitlines():
            m = re.match(r"B=(\d+) (\w+): ([0-9.]+) ms", line)
            if m:
                res[(v, m.group(1), m.group(2))].append(float(m.group(3)))
        if out.returncode:
            print(v, out.stderr[-500:])
for k in sorted(res):
    print(k, "median %.4f ms" % np.median(res[k]), "min %.4f" % min(res[k]), len(res[k]))
