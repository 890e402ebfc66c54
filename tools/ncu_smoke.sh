# ncu --set full of one launch of each smoke kernel at 612^3 (tools/smoke_probe.py)
TAG=${1:-x}
KREGEX=${2:-qsmoke_(jacobi|advect_u|advect_rho|project|div)}
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"$KREGEX" --launch-skip 150 --launch-count 6 -o gpurun_out/ncusmoke_$TAG python tools/smoke_probe.py --reps 2 --steps 1 > gpurun_out/ncusmoke_$TAG.log 2>&1; echo "ncu smoke rc=$?"
