"""Markdown table of a record run's bench lines (tools/gpu_record.sh output): workload, device value,
end to end, kernel fraction of the sustained peak, per-clock fraction, effective clock, parity.

    python tools/summarize_rec.py gpurun_out/rec > profiles/r02/final/SUMMARY.md
"""
import json
import sys
from pathlib import Path

d = Path(sys.argv[1])
print("| line | workload | value | e2e | kernel frac | per clock | eff. MHz | nvidia-smi MHz | parity |")
print("|---|---|---|---|---|---|---|---|---|")
for f in sorted(d.glob("bench_*.log")):
    for line in f.read_text().splitlines():
        if not line.startswith("{"):
            continue
        x = json.loads(line)
        r = x.get("roofline") or {}
        e = x.get("e2e") or {}
        p = x.get("parity") or {}
        c = x.get("clocks") or {}

        def fmt(v, n=3):
            return "-" if v is None else (f"{v:.{n}f}" if isinstance(v, float) else str(v))
        print(f"| {f.stem} | {x.get('config', {}).get('workload', '')} | {fmt(x['value'])} {x['unit']} | "
              f"{fmt(e.get('value'))} | {fmt(r.get('frac'))} | {fmt(r.get('frac_per_clock'))} | "
              f"{fmt(r.get('sm_clock_effective_mhz'), 0)} | {fmt(c.get('sm_mhz'), 0)} | "
              f"{p.get('ok', x.get('spot_check', '-'))} |")
