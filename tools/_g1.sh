python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -k "not fullsize" -p no:cacheprovider > gpurun_out/t1.log 2>&1; echo "tests rc=$?"
tail -30 gpurun_out/t1.log | grep -v "^\s*$" | tail -20
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/b1.log 2>&1; echo "bench rc=$?"
tail -c 2500 gpurun_out/b1.log
