python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/t1.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/t1.log | tail -25
timeout 900 python bench.py --steps 20 --warmup 5 --cpu-sample 10000 --cpu-steps 1 > gpurun_out/b1.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/b1.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']
print('%.3e'%d['value'], 'ms %.2f'%d['ms_per_step'], {n:round(v['ms_per_step'],3) for n,v in k.items()}, 'frac %.3f'%d['roofline']['frac'], 'issue', d['roofline'].get('issue_frac'), 'e2e', (d.get('e2e') or {}).get('value'), d['gpu_launches'])"
timeout 600 python bench.py --config c1 --steps 200 --warmup 10 --cpu-sample 8192 --cpu-steps 5 > gpurun_out/b_c1.log 2>&1; echo "bench c1 rc=$?"; tail -c 600 gpurun_out/b_c1.log
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:'qmpm_(p2g|g2p)' --launch-skip 4000 --launch-count 2 -o gpurun_out/ncu_c4_r2c -f python bench.py --steps 1 --warmup 3 --no-e2e --cpu-sample 1000 --cpu-steps 1 > gpurun_out/ncu_c4_r2c.log 2>&1; echo "ncu c4 rc=$?"
