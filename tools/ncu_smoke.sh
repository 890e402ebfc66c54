# ncu --set full of one launch of each smoke kernel at 612^3 (tools/smoke_probe.py --ncu:
# 4 plume steps = 540 launches, then advect, advect+reflect, div, jacobi, project, density)
TAG=${1:-x}
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:qsmoke_ --launch-skip 540 --launch-count 6 -o gpurun_out/ncusmoke_$TAG python tools/smoke_probe.py --ncu > gpurun_out/ncusmoke_$TAG.log 2>&1; echo "ncu smoke rc=$?"
