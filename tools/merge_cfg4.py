"""Merge per-variant oracle records (gpurun_out/r2/cfg4_<variant>.json, written
by oracle/gen_cfg4.py --out on the GPU box's host cores) into
tests/golden/cfg4.json: python tools/merge_cfg4.py file [file ...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path = os.path.join(ROOT, "tests", "golden", "cfg4.json")
res = json.load(open(path)) if os.path.exists(path) else {
    "generator": "oracle/gen_cfg4.py (CPU oracle, pinned to the reference)", "cases": []}
for f in sys.argv[1:]:
    for c in json.load(open(f))["cases"]:
        res["cases"] = [x for x in res["cases"] if x["variant"] != c["variant"]] + [c]
        print("merged", c["variant"], "from", f, "seconds", c.get("seconds"), "fwd_err", c.get("fwd_err"))
res["cases"].sort(key=lambda c: c["variant"], reverse=True)  # uniform, ill
json.dump(res, open(path, "w"))
