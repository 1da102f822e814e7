#!/bin/bash
# Bench every BASELINE.json config on one GPU (device-resident value + roofline + parity vs the
# oracle), plus the C4b (shared phase 1) and C5b (two-phase 500 x 500) stress variants and the
# reference arm on C2.  JSON lines to gpurun_out/bench_<cfg>.json.
mkdir -p gpurun_out
python bench.py --config c2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --impl reference --config c2 > gpurun_out/bench_reference_c2.json 2> gpurun_out/bench_reference_c2.err
python bench.py --config c1 --steps 50 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
python bench.py --config c3 --steps 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --config c4 --steps 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python bench.py --config c5 --steps 10 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
python bench.py --config c4b --steps 5 > gpurun_out/bench_c4b.json 2> gpurun_out/bench_c4b.err
timeout 900 python bench.py --config c5b --steps 3 > gpurun_out/bench_c5b.json 2> gpurun_out/bench_c5b.err
for c in c1 c2 c3 c4 c5 c4b c5b; do python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/bench_{c}.json"))
except Exception as e:
    print(c, "FAILED", e); sys.exit()
r = d["roofline"]
p = d.get("parity", {})
print(f"{c}: {d['config']['kernel']:20s} value={d['value']:.4g} LPs/s ms={d['ms_per_step']:.3f} "
      f"roofline {r['bound']} {r['achieved']:.4g}/{r['peak']:.4g} {r['unit']} frac={r['frac']:.3f} "
      f"parity checked={p.get('checked')} mismatches={p.get('status_mismatch')},{p.get('x_mismatch')},{p.get('iter_mismatch')} "
      f"e2e={d['e2e']['value']:.4g} obj_api={d.get('e2e_object_api', {}).get('value', 0):.4g} clocks={d['clocks']['sm_mhz']}")
PY
done
