"""(De)serialise op scripts + expected observations as pickle-free .npz files."""
from __future__ import annotations

import json

import numpy as np

_ARRAY_OPS = {"insert": 2, "delete": 2, "insert_csr": 2, "delete_csr": 2, "query": 2, "del_vertices": 1}


def save_cases(path, cases):
    """cases: list of dict(cfg=..., script=[...], expect=run_script() result)."""
    arrays, meta = {}, []
    for w, case in enumerate(cases):
        ops = []
        for j, op in enumerate(case["script"]):
            kind = op[0]
            if kind in _ARRAY_OPS:
                for a in range(_ARRAY_OPS[kind]):
                    arrays[f"w{w}_op{j}_a{a}"] = np.asarray(op[1 + a])
                ops.append([kind])
            elif kind == "add_vertices":
                ops.append([kind, int(op[1])])
            else:
                ops.append([kind])
        obs = []
        for j, o in enumerate(case["expect"]["obs"]):
            if o[0] == "answers":
                arrays[f"w{w}_obs{j}"] = np.frombuffer(o[1], dtype=np.uint8)
                obs.append(["answers"])
            elif o[0] == "skipped":
                obs.append(["skipped", [int(x) for x in o[1]]])
            else:
                obs.append([o[0]] + [int(x) for x in o[1:]])
        st = case["expect"]["state"]
        for k in ("alive", "degrees", "offsets", "destinations"):
            arrays[f"w{w}_state_{k}"] = np.asarray(st[k])
        meta.append({"cfg": case["cfg"], "ops": ops, "obs": obs,
                     "state": {k: int(st[k]) for k in ("logical_size", "capacity", "alive_vertices", "active_edges")}})
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(path, **arrays)


def load_cases(path):
    z = np.load(path)
    meta = json.loads(bytes(z["meta"]).decode())
    cases = []
    for w, m in enumerate(meta):
        script = []
        for j, op in enumerate(m["ops"]):
            kind = op[0]
            if kind in _ARRAY_OPS:
                script.append((kind, *[z[f"w{w}_op{j}_a{a}"] for a in range(_ARRAY_OPS[kind])]))
            elif kind == "add_vertices":
                script.append((kind, op[1]))
            else:
                script.append((kind,))
        obs = []
        for j, o in enumerate(m["obs"]):
            if o[0] == "answers":
                obs.append(("answers", z[f"w{w}_obs{j}"].tobytes()))
            elif o[0] == "skipped":
                obs.append(("skipped", tuple(o[1])))
            else:
                obs.append(tuple(o))
        state = dict(m["state"])
        for k in ("alive", "degrees", "offsets", "destinations"):
            state[k] = z[f"w{w}_state_{k}"]
        cases.append({"cfg": m["cfg"], "script": script, "expect": {"obs": obs, "state": state}})
    return cases
