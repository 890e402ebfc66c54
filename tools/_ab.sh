python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
QMPM_JIT_OPTS=-DQMPM_AB_SHFPACK=1 timeout 1500 python -m pytest tests/test_gpu_codec.py tests/test_gpu_step.py -q -x -p no:cacheprovider > gpurun_out/t_shf.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/t_shf.log | tail -4
timeout 900 python tools/ab_step.py --config c4 --warm 2000 --steps 20 --variant=-DQMPM_AB_SHFPACK=1 2>&1 | tail -3
timeout 900 python tools/ab_step.py --config c3 --warm 1000 --steps 20 --variant=-DQMPM_AB_SHFPACK=1 2>&1 | tail -3
