#!/bin/bash
# Exercise bench.py's N > 1 path on a one-GPU box: 2 and 4 ranks on cuda:0
# over gloo (PINN_BENCH_SHARED_GPU=1), every workload/method; the lines are
# code-path checks, not bench numbers.
mkdir -p gpurun_out/mr
export PINN_BENCH_SHARED_GPU=1
for n in 2 4; do
  for args in "" "--method xpinn" "--method dp" "--workload c3" "--workload c5"; do
    tag=$(echo "n$n $args" | tr ' -' '__')
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29500 + n)) bench.py --gpus $n --steps 5 --warmup 3 --no-cpu $args \
      > gpurun_out/mr/$tag.json 2> gpurun_out/mr/$tag.err
    echo "$tag rc=$? $(tail -c 300 gpurun_out/mr/$tag.json)"
  done
done
