"""One-line summary of a bench JSON log (A/B runs)."""
import json
import sys

for line in open(sys.argv[1]):
    if line.startswith("{"):
        d = json.loads(line)
        r = d["roofline"]
        nb = d["config"]["hot_batches_per_step"]
        print(f"value={d['value'] / 1e9:.3f}G train_us/batch={d['phases_ms_per_step']['train'] * 1e3 / nb:.2f} "
              f"kern={r['kernel']} frac={r['frac']:.3f} us={r['kernels_us']}")
