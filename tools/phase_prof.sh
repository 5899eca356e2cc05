#!/bin/bash
# per-phase cycle split of K1 for each workload (development tool; run on the GPU box)
# usage: tools/phase_prof.sh WORKLOAD...   (needs paper_2104_10013_b200/libpinn_dd_prof.so)
set -u
L=paper_2104_10013_b200
cp $L/libpinn_dd.so /tmp/libpinn_dd_real.so
cp $L/libpinn_dd_prof.so $L/libpinn_dd.so
for w in "$@"; do
  extra=""; tc=0
  case $w in *_tf32) extra="--tf32"; w=${w%_tf32}; tc=1;; esac
  python tools/phase_prof.py $w $extra 2>&1 | sed -n '/---MARK---/,$p' | TC=$tc python -c "
import sys
import os
tc = os.environ.get('TC') == '1'
names = ['claim/setup', 'weights', 'coords', 'layer-1 fwd', 'output fwd', 'epilogue', 'output bwd', 'bwd prologue',
         'layer-1 bwd', 'chunk end', 'payload fwd', 'payload epi', 'fwd: gemm', 'fwd: act+st', 'fwd: bar',
         'bwd: dW', 'bwd: gemm_bwd', 'bwd: act', 'bwd: bar', 'bwd: red+st+bar']
if tc:
    names[12:] = ['fwd: mma', 'fwd: ld+act+st', '-', 'bwd: ld+act', 'bwd: flush dW', 'bwd: owrite', 'bwd: mma', 'bwd: ld R']
tot = [0] * 20
hdr = ''
for l in sys.stdin:
    if l.startswith('---'): hdr = l.strip(); continue
    if l.startswith('PHASE'):
        v = [int(x) for x in l.split(':')[1].split()]
        tot = [a + b for a, b in zip(tot, v)]
s = sum(tot) or 1
print(hdr, 'total Mcyc (4 CTAs) %.2f' % (s / 1e6))
for n, t in zip(names, tot):
    print('  %-12s %6.1f %%' % (n, 100 * t / s))
"
done
cp /tmp/libpinn_dd_real.so $L/libpinn_dd.so
