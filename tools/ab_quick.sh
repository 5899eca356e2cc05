#!/bin/bash
# quick A/B: per-workload bench lines without the CPU leg (development tool)
# usage: tools/ab_quick.sh TAG WORKLOAD... (lines -> gpurun_out/ab/TAG_<w>.json)
set -u
tag=$1; shift
mkdir -p gpurun_out/ab
for w in "$@"; do
  extra=""
  case $w in *_tf32) extra="--tf32"; w=${w%_tf32};; esac
  python bench.py --no-cpu --workload $w $extra --steps 100 --warmup 5 > gpurun_out/ab/${tag}_$w$extra.json 2> gpurun_out/ab/${tag}_$w.err
  python - "$tag" "$w$extra" <<'PY'
import json, sys
t, w = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/ab/{t}_{w}.json").read().strip().splitlines()[-1])
    k = d["kernels_ms_per_step"]
    print(f"{t} {w}: step {d['ms_per_step']:.4f} ms  K1 {k['K1_loss_grad']:.4f}  K5 {k['K5_reduce_adam']:.4f}  frac {d['roofline']['frac']:.3f}  e2e {d['e2e']['value']:.3e}")
except Exception as e:
    print(t, w, "FAILED", e)
PY
done
