# C3 timing with env variants
TAG=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for o in "$@"; do
  n=$(echo "$o" | tr -c 'A-Za-z0-9=_' '_')
  env $o python bench.py --config c3 --steps 10 --warmup 3 --scene-warmup 20 --no-e2e --cpu-sample 10000 --cpu-steps 1 > gpurun_out/c3e_${TAG}_$n.log 2>&1; echo "$o rc=$?"
done
