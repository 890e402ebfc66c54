# Round evidence: plain default bench, its ncu launch list, one ncu --set full capture of
# P2G + G2P at full size, and the C3 bench.  Outputs under gpurun_out/ with TAG.
TAG=${1:-x}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || exit 1
python bench.py > gpurun_out/bench_default_$TAG.log 2>&1; echo "bench default rc=$?"
python bench.py --steps 2 --warmup 3 --no-e2e --cpu-sample 10000 --cpu-steps 1 > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'qmpm|k_' -c 2000 --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --cpu-sample 10000 --cpu-steps 1 > gpurun_out/ncu_launches_$TAG.log 2>&1
echo "launch list rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:'qmpm_(p2g|g2p)' --launch-skip 100 --launch-count 2 -o gpurun_out/ncufull_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --cpu-sample 10000 --cpu-steps 1 > gpurun_out/ncufull_$TAG.log 2>&1; echo "ncu full rc=$?"
if [[ "$2" == "c3" ]]; then python bench.py --config c3 --steps 10 > gpurun_out/bench_c3_$TAG.log 2>&1; echo "bench c3 rc=$?"; fi
