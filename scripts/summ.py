"""Summarise a bench.py JSON line from stdin: value, ms/step, per-kernel ms."""
import json
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else ""
for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    ks = " ".join(f"{k}={v['ms_per_launch']:.4f}" for k, v in d.get("kernels", {}).items())
    print(f"{tag} value={d['value']:.4g} ms/step={d['ms_per_step']} prof_pass={d.get('kernels_pass_ms_per_step')} {ks}")
