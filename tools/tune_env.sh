# usage: bash tools/tune_env.sh TAG "VAR=val ..." ...  (50M same-density C4 runs with env variants)
TAG=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for o in "$@"; do
  n=$(echo "$o" | tr -c 'A-Za-z0-9=_' '_')
  env $o timeout 300 python bench.py --n 50000000 --z-extent 0.125 --steps 10 --warmup 3 --scene-warmup 20 --no-e2e --cpu-sample 10000 --cpu-steps 1 > gpurun_out/tunee_${TAG}_$n.log 2>&1
  echo "$o rc=$?"
done
