python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_codec.py tests/test_gpu_step.py tests/test_gpu_developed.py tests/test_gpu_scheme.py -q -x -p no:cacheprovider > gpurun_out/t_sz.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/t_sz.log | tail -6
timeout 900 python tools/ab_step.py --config c4 --warm 2000 --steps 20 --variant=-DQMPM_AB_SZEXT=0 2>&1 | tail -3
timeout 900 python tools/ab_step.py --config c3 --warm 1000 --steps 20 --variant=-DQMPM_AB_SZEXT=0 2>&1 | tail -3
timeout 900 python tools/ab_step.py --config c4_8ppc --warm 2000 --steps 20 --variant=-DQMPM_AB_SZEXT=0 2>&1 | tail -3
