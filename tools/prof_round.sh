# The round's measurement pass (one GPU call), everything copied under gpurun_out/:
#   bench lines (C4 default, C4 w/o counters, C3, C4-8ppc, C1), ncu --set full of the C4 and C3
#   step kernels after the bench's warm-up, the ncu launch list of the default bench
#   command, the developed-state parity tests with their printed flip rates.
# usage: bash tools/prof_round.sh TAG
TAG=${1:-r2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_developed.py -q -s -p no:cacheprovider > gpurun_out/parity_flips_$TAG.log 2>&1; echo "developed tests rc=$?"
grep -E "flips|passed|failed" gpurun_out/parity_flips_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_c4_$TAG.log 2>&1; echo "bench c4 rc=$?"
timeout 900 python bench.py --no-counters --no-e2e --cpu-sample 1000 --cpu-steps 1 > gpurun_out/bench_c4nc_$TAG.log 2>&1; echo "bench c4 no counters rc=$?"
timeout 900 python bench.py --config c3 > gpurun_out/bench_c3_$TAG.log 2>&1; echo "bench c3 rc=$?"
timeout 900 python bench.py --config c4_8ppc > gpurun_out/bench_c48_$TAG.log 2>&1; echo "bench c4_8ppc rc=$?"
timeout 600 python bench.py --config c1 --steps 200 --warmup 10 > gpurun_out/bench_c1_$TAG.log 2>&1; echo "bench c1 rc=$?"
for f in c4 c4nc c3 c48 c1; do tail -1 gpurun_out/bench_${f}_$TAG.log | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); k=d['kernels']
  print('$f', '%.4e'%d['value'], 'ms %.3f'%d['ms_per_step'], 'g2p %.3f p2g %.3f scat %.3f'%(k['g2p']['ms_per_step'],k['p2g']['ms_per_step'],k['bin_scatter']['ms_per_step']), 'frac %.3f'%d['roofline']['frac'], 'issue', d['roofline'].get('issue_frac'), 'e2e', (d.get('e2e') or {}).get('value'))
except Exception as e: print('$f parse error', e)"; done
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:'qmpm_(p2g|g2p)' --launch-skip 4000 --launch-count 2 -o gpurun_out/ncu_c4_$TAG -f python bench.py --steps 1 --warmup 3 --no-e2e --cpu-sample 1000 --cpu-steps 1 > gpurun_out/ncu_c4_$TAG.log 2>&1; echo "ncu c4 rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:'qmpm_(p2g|g2p)' --launch-skip 2000 --launch-count 2 -o gpurun_out/ncu_c3_$TAG -f python bench.py --config c3 --steps 1 --warmup 3 --no-e2e --cpu-sample 1000 --cpu-steps 1 > gpurun_out/ncu_c3_$TAG.log 2>&1; echo "ncu c3 rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:'qmpm_(p2g|g2p)' --launch-skip 4000 --launch-count 2 -o gpurun_out/ncu_c48_$TAG -f python bench.py --config c4_8ppc --steps 1 --warmup 3 --no-e2e --cpu-sample 1000 --cpu-steps 1 > gpurun_out/ncu_c48_$TAG.log 2>&1; echo "ncu c4_8ppc rc=$?"
# the launch list of the same command as the bench line (default arguments)
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_$TAG.csv python bench.py > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
