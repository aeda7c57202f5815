# round 2: uniform per-direction offset tables (DirOffsets): GPU suite, A/B against
# the tile-descriptor build, ncu of the new fp32 / fp64 sweeps
O=gpurun_out/r02e
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
S="--precision fp64;--precision fp32;--precision fp32 --workload patchy64;--precision fp64 --layout aa;--precision fp32 --layout aa"
bash tools/variant_bench.sh $O/ab.jsonl build/variants/desc.so build/variants/off.so -- "$S"
LBM_SWEEP_VARIANT=1 bash tools/variant_bench.sh $O/ab_v1.jsonl build/variants/desc.so build/variants/off.so -- "$S"
for p in fp32 fp64; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_x2 -s 3 -c 1 -o $O/x2_${p}_off python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --precision $p > $O/ncu_$p.log 2>&1
done
echo done
