# C5 (BASELINE configs[4]): the C3 scene with fp32 vs the stand-in schemes at error
# bounds 0.1 / 0.01, dithered vs round-to-nearest: particle-steps/s vs bytes per particle.
TAG=${1:-x}
for sch in fp32 e0.1 e0.01; do
  python bench.py --config c3 --scheme $sch --steps 10 --warmup 3 --scene-warmup 20 --no-e2e --cpu-sample 10000 --cpu-steps 1 > gpurun_out/c5_${TAG}_$sch.log 2>&1; echo "$sch rc=$?"
done
python bench.py --config c3 --scheme e0.01 --rounding rne --steps 10 --warmup 3 --scene-warmup 20 --no-e2e --cpu-sample 10000 --cpu-steps 1 > gpurun_out/c5_${TAG}_e0.01_rne.log 2>&1; echo "e0.01 rne rc=$?"
python bench.py --config c4 --scheme fp32 --steps 10 --warmup 3 --scene-warmup 20 --no-e2e --cpu-sample 10000 --cpu-steps 1 > gpurun_out/c5_${TAG}_c4_fp32.log 2>&1; echo "c4 fp32 rc=$?"
