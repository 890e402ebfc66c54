# usage: bash tools/tune.sh TAG "OPTS1" "OPTS2" ...  (50M same-density C4 runs with QMPM_JIT_OPTS variants)
TAG=$1; shift
for o in "$@"; do
  n=$(echo "$o" | tr -c 'A-Za-z0-9=_' '_')
  QMPM_JIT_OPTS="$o" timeout 300 python bench.py --n 50000000 --z-extent 0.125 --steps 10 --warmup 3 --scene-warmup 20 --no-e2e --cpu-sample 10000 --cpu-steps 1 > gpurun_out/tune_${TAG}_$n.log 2>&1
  echo "$o rc=$?"
done
