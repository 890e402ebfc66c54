# round-2 measurement pass (one GPU call): developed-state tests, bench lines, ncu
# usage: bash tools/prof_r2.sh TAG
TAG=${1:-r2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_developed.py tests/test_gpu_adjoint.py -q -s -p no:cacheprovider > gpurun_out/t_dev_$TAG.log 2>&1; echo "dev tests rc=$?"
grep -E "flips|passed|failed|Error" gpurun_out/t_dev_$TAG.log | tail -12
timeout 900 python bench.py > gpurun_out/b_c4_$TAG.log 2>&1; echo "bench c4 rc=$?"
timeout 600 python bench.py --scene-warmup 50 --no-e2e --cpu-sample 10000 --cpu-steps 1 > gpurun_out/b_c4w50_$TAG.log 2>&1; echo "bench c4 w50 rc=$?"
timeout 900 python bench.py --config c3 > gpurun_out/b_c3_$TAG.log 2>&1; echo "bench c3 rc=$?"
timeout 900 python bench.py --config c4_8ppc --no-e2e --cpu-sample 100000 --cpu-steps 1 > gpurun_out/b_c48_$TAG.log 2>&1; echo "bench c4_8ppc rc=$?"
for f in c4 c4w50 c3 c48; do tail -1 gpurun_out/b_${f}_$TAG.log | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); k=d['kernels']
  print('$f', '%.3e'%d['value'], 'ms %.2f'%d['ms_per_step'], 'g2p %.2f p2g %.2f scat %.2f'%(k['g2p']['ms_per_step'],k['p2g']['ms_per_step'],k['bin_scatter']['ms_per_step']), 'frac %.3f'%d['roofline']['frac'], 'e2e', (d.get('e2e') or {}).get('value'))
except Exception as e: print('$f parse error', e)"; done
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:'qmpm_(p2g|g2p)' --launch-skip 4000 --launch-count 2 -o gpurun_out/ncu_c4_$TAG -f python bench.py --steps 1 --warmup 3 --no-e2e --cpu-sample 1000 --cpu-steps 1 > gpurun_out/ncu_c4_$TAG.log 2>&1; echo "ncu c4 rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:'qmpm_(p2g|g2p)' --launch-skip 2000 --launch-count 2 -o gpurun_out/ncu_c3_$TAG -f python bench.py --config c3 --steps 1 --warmup 3 --no-e2e --cpu-sample 1000 --cpu-steps 1 > gpurun_out/ncu_c3_$TAG.log 2>&1; echo "ncu c3 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4_$TAG.csv python bench.py --steps 2 --warmup 3 --no-e2e --cpu-sample 1000 --cpu-steps 1 > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
ls -la gpurun_out
