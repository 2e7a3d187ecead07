#!/bin/bash
# One bench line per BASELINE.json config (no CPU baseline), appended to gpurun_out/configs.jsonl
mkdir -p gpurun_out
out=gpurun_out/configs.jsonl
: > $out
run() { timeout 900 python bench.py --no-cpu-baseline "$@" 2>gpurun_out/cfg.err | tail -1 >> $out || tail -3 gpurun_out/cfg.err; }
run --config 0 --steps 20 --warmup 5
run --config 1 --steps 20 --warmup 5
run --config 1 --method mp --steps 20 --warmup 5
run --config 2 --steps 5 --warmup 3
run --config 3 --steps 10 --warmup 3
run --config 4 --steps 5 --warmup 3
run --config 4 --selector exact --steps 1 --warmup 3 --no-e2e
run --config 1 --alpha 0.1 --steps 5 --warmup 2 --no-e2e
run --config 4 --alpha 0.1 --steps 2 --warmup 2 --no-e2e
python - <<'PY'
import json
for line in open("gpurun_out/configs.jsonl"):
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    c = d["config"]
    r = d["roofline"]
    e2e = d["e2e"]["value"] if d.get("e2e") else None
    print(f'{c["workload"]:44s} N={c["patches_per_gpu"]:8d} {d["value"]:14.1f} patches/s  ms/step {d["ms_per_step"]:9.3f}  '
          f'step frac {r["step"]["frac"] or 0:.3f}  dominant {r["kernel"][:40]} frac {r["frac"]:.3f} '
          f'(3xtf32 {r.get("frac_3xtf32")})  e2e {e2e}')
PY
