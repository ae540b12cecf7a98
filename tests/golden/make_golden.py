"""Generate the golden fixtures from the UNMODIFIED compiled reference.

Run in the build container (needs oracle/_ref/libpipeplan_ref.so, built by
`make -C oracle ref` from /root/reference/proj/src):

    python tests/golden/make_golden.py

Writes tests/golden/reference_golden.json.  Every number comes from the
reference library through oracle/ref_shim.cpp; nothing is computed here.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle import OracleError, Reference  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def call(f, *a, **k):
    try:
        return {"ok": f(*a, **k)}
    except OracleError as e:
        return {"error": e.msg, "code": e.code}


def main():
    r = Reference()
    g = {"generator": "tests/golden/make_golden.py", "source": "compiled reference via oracle/ref_shim.cpp"}

    # split_layer over widths x device counts (partition.cpp:15-48)
    sl = []
    for fo in range(1, 41):
        for n in range(1, 9):
            for rep in (False, True):
                res = call(r.split_layer, fo, n, rep, 3)
                sl.append({"fan_out": fo, "n": n, "replicate": rep,
                           **({"shards": res["ok"]} if "ok" in res else res)})
    g["split_layer"] = sl

    # split_microbatches (schedule.cpp:46-55)
    g["split_microbatches"] = [{"b": b, "m": m, **({"sizes": v["ok"]} if "ok" in (v := call(r.split_microbatches, b, m)) else v)}
                               for b in range(1, 33) for m in range(1, 36)]

    # plans (partition.cpp:110-182)
    chains = [[4, 8, 8, 8, 8], [3, 6, 6, 6], [784, 512, 512, 10], [8192] * 5, [5, 7, 3, 9, 2, 6],
              [16, 64, 4, 64, 32, 10, 8], [2, 3], [3, 32, 32, 32, 32, 32, 5]]
    plans = []
    for dims in chains:
        L = len(dims) - 1
        for n in (1, 2, 3, 4, 8):
            for Z in range(1, L + 2):
                for rep in (False, True):
                    res = call(r.build_plan, dims, n, Z, rep)
                    entry = {"dims": dims, "n": n, "Z": Z, "replicate": rep}
                    if "ok" in res:
                        entry["plan"] = res["ok"].tolist()
                        if Z >= 2:
                            entry["merged_1_2"] = r.merge_submodules(res["ok"], [1, 2]).tolist()
                            entry["merged_all"] = r.merge_submodules(res["ok"], list(range(1, Z + 1))).tolist()
                    else:
                        entry.update(res)
                    plans.append(entry)
    g["build_plan"] = plans
    staged = []
    for dims, groups in [([784, 512, 512, 10], [[1, 2], [3, 4]]), ([4, 8, 8, 8, 8], [[1], [2, 3], [4]]),
                         ([3, 6, 6, 6], [[2, 1], [3]]), ([8192] * 5, [[1, 2, 3, 4], [5, 6, 7, 8]])]:
        res = call(r.build_staged_plan, dims, groups)
        staged.append({"dims": dims, "groups": groups, **({"plan": res["ok"].tolist()} if "ok" in res else res)})
    g["build_staged_plan"] = staged

    # plan JSON I/O (partition.cpp:303-384): byte-exact serialisations + parse cases
    js = []
    for e in plans[:: 7]:
        if "plan" not in e:
            continue
        prov = ["merge[1..2]"] if e["Z"] >= 2 else []
        src = e["merged_1_2"] if e["Z"] >= 2 else e["plan"]
        js.append({"plan": src, "provenance": prov, "json": r.serialize_plan(np.array(src), prov)})
    g["serialize_plan"] = js
    bad = ['{"n": 2, "submodules": [{"span": [1, 1], "shards": [{"layer": 2, "device": 1, "range": [0, 4]}]}], "boundaries": []}',
           '{"n": 1, "submodules": [{"span": [1, 1], "devices": [1], "shards": [{"layer": 1, "device": 1, "range": [0, 4]}]}], "boundaries": ["sideways"]}',
           '{"n": 1, "submodules": [{"span": [1, 2], "shards": [{"layer": 1, "device": 1, "range": [0, 4]}, {"layer": 2, "device": 1, "range": [0, 3], "replicated": true}]}], "boundaries": []}']
    g["parse_plan"] = [{"text": t, **({"plan": v["ok"].tolist()} if "ok" in (v := call(r.parse_plan, t)) else v)} for t in bad]

    # verify instances (verify.cpp:20-62) with the reference's own outputs
    inst = []
    for k in range(60):
        d = r.draw_instance(1234 + k)
        args = (d["dims"], d["acts"], d["W"], d["b"], d["X"], d["labels"])
        hp = (d["alpha0"], d["decay"], d["loss"], d["iterations"])
        e = {key: (v.tolist() if isinstance(v, np.ndarray) else v) for key, v in d.items()}
        for mode in (1, 2):
            res = call(r.train_partitioned, *args, d["plan"], d["m"], mode, *hp)
            e[f"partitioned_mode{mode}"] = ({"W": res["ok"][0].tolist(), "b": res["ok"][1].tolist(),
                                             "loss": res["ok"][2].tolist(), "acc": res["ok"][3].tolist()}
                                            if "ok" in res else res)
        res = call(r.train_sequential, *args, *hp)
        e["sequential"] = ({"W": res["ok"][0].tolist(), "b": res["ok"][1].tolist(), "loss": res["ok"][2].tolist(),
                            "acc": res["ok"][3].tolist()} if "ok" in res else res)
        inst.append(e)
    g["verify_instances"] = inst

    # the MLP configuration of BASELINE.json configs[0]
    dims, acts = [784, 512, 512, 10], [1, 1, 2]
    W, b = r.init_net(dims, acts, 1)
    X, y = r.make_blobs(64, 784, 1.0, 13)
    mlp = {"dims": dims, "acts": acts, "init_seed": 1, "blobs": [64, 784, 1.0, 13],
           "W_sha256": sha(W), "b_sha256": sha(b), "X_sha256": sha(X), "labels": y.tolist(),
           "W_head": W[:16].tolist(), "X_head": X.ravel()[:16].tolist(), "runs": []}
    for (n, Z, m, merge, mode) in [(1, 1, 1, False, 1), (2, 1, 1, False, 1), (2, 1, 2, False, 1),
                                   (2, 3, 2, True, 2), (2, 3, 4, False, 1)]:
        plan = r.build_plan(dims, n, Z)
        if merge:
            plan = r.merge_submodules(plan, list(range(1, Z + 1)))
        Wo, bo, lh, ah = r.train_partitioned(dims, acts, W, b, X, y, plan, m, mode, 0.05, 0.01, 1, 5)
        mlp["runs"].append({"n": n, "Z": Z, "m": m, "merged": merge, "mode": mode, "alpha0": 0.05, "decay": 0.01,
                            "iterations": 5, "plan": plan.tolist(), "loss": lh.tolist(), "acc": ah.tolist(),
                            "W_sha256": sha(Wo), "b_sha256": sha(bo), "W_head": Wo[:16].tolist(),
                            "b_out": bo.tolist()})
    g["mlp"] = mlp

    ok, report = r.run_verification(100)
    g["run_verification"] = {"seeds": 100, "all_pass": ok, "report": report}

    out = os.path.join(HERE, "reference_golden.json")
    with open(out, "w") as f:
        json.dump(g, f)
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
