# elastic parity tests + C3 timing (optionally with QMPM_JIT_OPTS variants)
TAG=${1:-x}; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "e0 or elastic or c1 or s3 or slab" > gpurun_out/c3tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/c3tests_$TAG.log
python bench.py --config c3 --steps 10 --warmup 3 --scene-warmup 20 --no-e2e --cpu-sample 10000 --cpu-steps 1 > gpurun_out/c3_$TAG.log 2>&1; echo "c3 rc=$?"
for o in "$@"; do
  n=$(echo "$o" | tr -c 'A-Za-z0-9=_' '_')
  QMPM_JIT_OPTS="$o" python bench.py --config c3 --steps 10 --warmup 3 --scene-warmup 20 --no-e2e --cpu-sample 10000 --cpu-steps 1 > gpurun_out/c3_${TAG}_$n.log 2>&1; echo "$o rc=$?"
done
