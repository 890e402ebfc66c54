# ncu --set full of one P2G and one G2P launch at the full C4 size (steady state)
TAG=${1:-x}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:'qmpm_(p2g|g2p)' --launch-skip 100 --launch-count 2 -o gpurun_out/ncufull_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --cpu-sample 10000 --cpu-steps 1 > gpurun_out/ncufull_$TAG.log 2>&1; echo "ncu full rc=$?"
