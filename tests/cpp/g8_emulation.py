"""Dev tool: the g = 8 code paths on a 4-GPU box.  The reference's own
algorithms (tests/cpp/algo_dropin.cpp) run on 8 workers -- once on its CPU
SimCluster, once on the B200 primitives with two ranks per GPU (thread per
rank, B2_DEVICES=4, an SM budget of 74 so two cooperative kernels fit side
by side) -- and the final parameters are compared bit for bit (onebit: the
documented tolerance).  Run once with the default dispatch
(register-resident small kernels for these bucket sizes) and once with the
TMA-ring kernels forced (B2_SMALL_C_MAX=0, B2_SMALL_MAX=0).

    python tests/cpp/g8_emulation.py [workers=8] [devices=4] [layer_scale=1] [algos]

layer_scale multiplies the harness's layer sizes (B2_DROPIN_SCALE; 40 puts
the largest bucket at 10M elements).
"""
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "algo_dropin_ref")
B200 = os.path.join(HERE, "algo_dropin_b200")
g = int(sys.argv[1]) if len(sys.argv) > 1 else 8
ndev = int(sys.argv[2]) if len(sys.argv) > 2 else 4
scale = sys.argv[3] if len(sys.argv) > 3 else "1"
algos = sys.argv[4].split(",") if len(sys.argv) > 4 else ["allreduce", "qsgd8", "decen32", "decen8", "onebit_adam"]
steps = 5


def run(binary, algo, prefix, env):
    r = subprocess.run([binary, algo, str(g), str(steps), prefix], capture_output=True, text=True, timeout=600,
                       env={**os.environ, "B2_DROPIN_SCALE": scale, **env})
    if r.returncode != 0:
        return None, (r.stdout[-1500:] + r.stderr[-1500:])
    return [np.fromfile(f"{prefix}_rank{k}.bin", np.float32) for k in range(g)], ""


res = {"workers": g, "devices": ndev, "layer_scale": int(scale), "cases": []}
ok = True
with tempfile.TemporaryDirectory() as td:
    for algo in algos:
        want, err = run(REF, algo, os.path.join(td, f"ref_{algo}"), {})
        if want is None:
            res["cases"].append({"algo": algo, "error": "reference: " + err})
            ok = False
            continue
        for paths, env in (("default", {}), ("ring", {"B2_SMALL_C_MAX": "0", "B2_SMALL_MAX": "0"})):
            env = {**env, "B2_DEVICES": str(ndev), "B2_SM_BUDGET": str(148 * ndev // g), "B2_TIMEOUT_MS": "20000"}
            got, err = run(B200, algo, os.path.join(td, f"b200_{algo}_{paths}"), env)
            case = {"algo": algo, "paths": paths}
            if got is None:
                case["error"] = err
                ok = False
            else:
                if algo == "onebit_adam":
                    d = max(float(np.abs(got[k].astype(np.float64) - want[k]).max()) for k in range(g))
                    tol = 1e-5 * max(float(np.abs(w).max()) for w in want)
                    case.update(max_abs_diff=d, tol=tol, ok=d <= tol)
                else:
                    same = [bool(np.array_equal(got[k].view(np.uint32), want[k].view(np.uint32))) for k in range(g)]
                    case.update(bit_exact_ranks=sum(same), ok=all(same))
                ok &= case["ok"]
            res["cases"].append(case)
res["ok"] = ok
print(json.dumps(res))
sys.exit(0 if ok else 1)
