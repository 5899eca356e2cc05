# A/B of the fused-kernel CTA size (development): tests + C2/C3 bench at 256 and 128 threads
mkdir -p gpurun_out/ab
for T in ${THREADS:-256 128}; do
  export PINN_DD_CTA_THREADS=$T
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab/pytest_$T.txt 2>&1; echo "T=$T $(tail -1 gpurun_out/ab/pytest_$T.txt)"
  for w in ${WORKLOADS:-c2 c3}; do
    python bench.py --no-cpu --workload $w > gpurun_out/ab/${w}_$T.json 2>&1
    tail -1 gpurun_out/ab/${w}_$T.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['value'], d['roofline']['frac'], d['roofline']['k1_ms_per_launch'])"
  done
done
