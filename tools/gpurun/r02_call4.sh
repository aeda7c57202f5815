# round 2: A/B of the x-ghost pull strategies + ncu of the fp32 sweep
mkdir -p gpurun_out/r02d
S="--precision fp64;--precision fp32;--precision fp32 --workload patchy64;--precision fp64 --layout aa;--precision fp32 --layout aa"
bash tools/variant_bench.sh gpurun_out/r02d/ab.jsonl build/variants/branch.so build/variants/select.so build/variants/pred.so -- "$S"
LBM_SWEEP_VARIANT=1 bash tools/variant_bench.sh gpurun_out/r02d/ab_v1.jsonl build/variants/branch.so build/variants/select.so build/variants/pred.so -- "--precision fp32;--precision fp64"
bash tools/variant_bench.sh gpurun_out/r02d/ab_repeat.jsonl build/variants/branch.so build/variants/select.so build/variants/pred.so -- "$S"
cp build/variants/select.so paper_1007_1388_b200/liblbm_b200.so
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --precision fp32 > gpurun_out/r02d/plain_fp32.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_x2 -s 3 -c 1 -o gpurun_out/r02d/x2_fp32_select python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --precision fp32 > gpurun_out/r02d/ncu.log 2>&1
echo done
