python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests/test_gpu_slab.py tests/test_gpu_step.py -q -p no:cacheprovider > gpurun_out/t1.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/t1.log | tail -10
for mb in 5 6; do
QMPM_P2G_MINB=$mb timeout 900 python bench.py --steps 20 --warmup 5 --no-e2e --cpu-sample 1000 --cpu-steps 1 > gpurun_out/b_mb$mb.log 2>&1; echo "bench minb=$mb rc=$?"
tail -1 gpurun_out/b_mb$mb.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']
print('%.3e'%d['value'], 'ms %.2f'%d['ms_per_step'], 'p2g %.3f g2p %.3f'%(k['p2g']['ms_per_step'], k['g2p']['ms_per_step']))"
done
QMPM_P2G_MINB=6 timeout 900 python bench.py --config c3 --steps 20 --warmup 5 --no-e2e --cpu-sample 1000 --cpu-steps 1 > gpurun_out/b_c3mb6.log 2>&1; echo "bench c3 minb6 rc=$?"
timeout 900 python bench.py --config c3 --steps 20 --warmup 5 --no-e2e --cpu-sample 1000 --cpu-steps 1 > gpurun_out/b_c3.log 2>&1; echo "bench c3 rc=$?"
for f in c3mb6 c3; do tail -1 gpurun_out/b_$f.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']
print('$f', '%.3e'%d['value'], 'ms %.2f'%d['ms_per_step'], 'p2g %.3f g2p %.3f'%(k['p2g']['ms_per_step'], k['g2p']['ms_per_step']))"; done
