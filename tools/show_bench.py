"""Print the key fields of bench JSON lines: python tools/show_bench.py gpurun_out/bench_*.json"""
import json
import sys

for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as exc:  # noqa: BLE001
        print(path, "unreadable:", exc)
        continue
    rl = d.get("roofline") or {}
    print(f"{path}: value={d.get('value'):.4g} ms/step={d.get('ms_per_step'):.4g} "
          f"frac={rl.get('frac')} kernel_ms={rl.get('kernel_avg_ms')} kernel={d.get('kernel')} "
          f"e2e={(d.get('e2e') or {}).get('value')} cpu={(d.get('cpu_baseline') or {}).get('value')} "
          f"clocks={d.get('clocks')}")
