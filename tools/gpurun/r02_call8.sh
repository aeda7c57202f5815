# round 2: offset tables + selected-address pull + packed f32x2 collide (f2.so): GPU suite,
# A/B against the committed tile-descriptor build, ncu of the sweeps
O=gpurun_out/r02h
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
S="--precision fp64;--precision fp32;--precision fp32 --workload patchy64;--precision fp64 --layout aa;--precision fp32 --layout aa"
bash tools/variant_bench.sh $O/v0.jsonl build/variants/f2.so build/variants/desc.so build/variants/f2.so -- "$S"
LBM_SWEEP_VARIANT=1 bash tools/variant_bench.sh $O/v1.jsonl build/variants/f2.so -- "$S"
for w in "fp32 ldc256" "fp64 ldc256" "fp32 patchy64"; do set -- $w
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_x2 -s 3 -c 1 -o $O/x2_$1_$2 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --precision $1 --workload $2 > $O/ncu_$1_$2.log 2>&1
done
echo done
