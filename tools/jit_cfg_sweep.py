"""Calibration sweep of the JIT configuration model: runs tools/jit_probe.py for forced
(layout, tile, warps) combinations, one subprocess each, and prints measured TFLOP/s next to
the model's cost.  python tools/jit_cfg_sweep.py > gpurun_out/jit_cfg_sweep.jsonl"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = [  # (layer, pair layout, tile "TY,TX" or "auto", warps)
    ("conv2", "0", "auto", "12"), ("conv2", "0", "auto", "16"), ("conv2", "1", "auto", "12"),
    ("conv2", "1", "auto", "16"), ("conv2", "1", "auto", "8"),
    ("conv3", "1", "auto", "16"), ("conv3", "1", "auto", "12"), ("conv3", "1", "auto", "20"),
    ("conv3", "0", "auto", "12"),
    ("conv4", "1", "auto", "16"), ("conv4", "1", "auto", "12"), ("conv4", "1", "auto", "20"),
    ("conv5", "1", "auto", "16"), ("conv5", "1", "auto", "12"), ("conv5", "1", "auto", "20"),
    ("conv5", "0", "auto", "12"),
]
for layer, pair, tile, nw in CASES:
    env = dict(os.environ, SKC_JIT_PAIR=pair, SKC_JIT_NW=nw)
    r = subprocess.run([sys.executable, os.path.join(HERE, "jit_probe.py"), "--tiles", tile,
                        "--layers", layer], env=env, capture_output=True, text=True, timeout=600)
    for line in r.stdout.splitlines():
        if line.startswith("{"):
            d = json.loads(line)
            d.update(pair=pair, forced_tile=tile, forced_nw=nw)
            print(json.dumps(d), flush=True)
    if r.returncode:
        print(json.dumps({"layer": layer, "pair": pair, "tile": tile, "nw": nw,
                          "error": r.stderr[-300:]}), flush=True)
