set -x
python bench.py --n 50000000 --z-extent 0.125 --steps 10 --warmup 3 --scene-warmup 20 --no-e2e --cpu-sample 10000 --cpu-steps 1 > gpurun_out/bench_50M.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'qmpm_(p2g|g2p)' --launch-skip 30 --launch-count 2 -o gpurun_out/c4_50M_v3 python bench.py --n 50000000 --z-extent 0.125 --steps 2 --warmup 3 --scene-warmup 20 --no-e2e --cpu-sample 10000 --cpu-steps 1 > gpurun_out/ncu_50M.log 2>&1
echo done
