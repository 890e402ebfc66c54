python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
run() { tag=$1; shift; env "$@" timeout 900 python bench.py --steps 20 --warmup 5 --no-e2e --cpu-sample 1000 --cpu-steps 1 > gpurun_out/tune_$tag.log 2>&1
tail -1 gpurun_out/tune_$tag.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']
print('$tag', '%.4e'%d['value'], 'ms %.3f'%d['ms_per_step'], 'p2g %.3f g2p %.3f scat %.3f'%(k['p2g']['ms_per_step'], k['g2p']['ms_per_step'], k['bin_scatter']['ms_per_step']))" ; }
run base X=1
run g2p5 QMPM_G2P_MINB=5
run segl24 "QMPM_JIT_OPTS=-DQMPM_SEG_L=24 -DQMPM_SEG_LMIN=24"
run segl32 "QMPM_JIT_OPTS=-DQMPM_SEG_L=32 -DQMPM_SEG_LMIN=32"
run p2g7 QMPM_P2G_MINB=7
