python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1500 python tools/ab_step.py --warm 2000 --steps 20 "--variant=-DQMPM_SEG_L=64 -DQMPM_SEG_LMIN=64" "--variant=-DQMPM_SEG_L=96 -DQMPM_SEG_LMIN=96" "--variant=-DQMPM_AB_ZPACK=0" 2>&1 | tail -6
timeout 1500 python tools/ab_step.py --config c3 --warm 1000 --steps 20 "--variant=-DQMPM_AB_ZPACK=0" "--variant=-DQMPM_AB_P2G_PF=0" 2>&1 | tail -5
