# usage: bash tools/gpu_check.sh TAG [full] [ncu]
TAG=${1:-x}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; tail gpurun_out/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?" | tee -a gpurun_out/gpu_tests_$TAG.log
tail -3 gpurun_out/gpu_tests_$TAG.log
timeout 600 python bench.py --n 50000000 --z-extent 0.125 --steps 10 --warmup 3 --scene-warmup 20 --no-e2e --cpu-sample 10000 --cpu-steps 1 > gpurun_out/bench50M_$TAG.log 2>&1; echo "bench50M rc=$?"
if [[ "$2" == "full" ]]; then timeout 900 python bench.py > gpurun_out/bench_full_$TAG.log 2>&1; echo "bench full rc=$?"; fi
if [[ "$3" == "ncu" ]]; then timeout 900 ncu --set full --import-source on --clock-control none -k regex:'qmpm_(p2g|g2p)' --launch-skip 30 --launch-count 2 -o gpurun_out/ncu_$TAG python bench.py --n 50000000 --z-extent 0.125 --steps 2 --warmup 3 --scene-warmup 20 --no-e2e --cpu-sample 10000 --cpu-steps 1 > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"; fi
