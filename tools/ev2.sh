set -u
O=gpurun_out/ev2; mkdir -p $O
python bench.py --tf32 --no-cpu > $O/bench_c4_tf32.json 2>&1
python bench.py --workload c5 --tf32 --no-cpu > $O/bench_c5_tf32.json 2>&1
K='k_fused<.*\(int\)2, \(int\)(256|128)>'
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$K" -c 1 -o $O/k1_c4 python bench.py --no-cpu --workload c4 --steps 2 --warmup 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_fused_tc<.*\(int\)2>' -c 1 -o $O/k1_c4_tf32 python bench.py --no-cpu --workload c4 --tf32 --steps 2 --warmup 3 > /dev/null 2>&1
for r in k1_c4 k1_c4_tf32; do python tools/ncu_summary.py $O/$r.ncu-rep > $O/${r}_summary.txt 2>&1; done
rm -f $O/*.ncu-rep.bak
ls -la $O
