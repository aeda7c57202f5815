# round 2: cp.async pull into shared memory (variant 2) vs the register pull
O=gpurun_out/r02f
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "variants" --timeout 400 > $O/pytest_variants.log 2>&1; echo "rc=$?" >> $O/pytest_variants.log
S="--precision fp64;--precision fp32;--precision fp32 --workload patchy64"
for v in 0 1 2; do
  LBM_SWEEP_VARIANT=$v bash tools/variant_bench.sh $O/ab_v$v.jsonl build/variants/async1.so -- "$S"
done
LBM_SWEEP_VARIANT=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_x2 -s 3 -c 1 -o $O/async_fp64 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --precision fp64 > $O/ncu_fp64.log 2>&1
echo done
