# round 2: final 1-GPU evidence of the final build (uniform-wall sides in both layouts)
# workload, launch list, ncu full captures (incl. the AA kernels)
O=gpurun_out/r02z
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --steps 1000 --warmup 20 --precision fp32 > $O/bench_fp32.json 2> $O/bench_fp32.err
timeout 600 python bench.py --steps 500 --warmup 20 --precision fp32 --workload patchy64 > $O/bench_fp32_patchy64.json 2> $O/bench_fp32_patchy64.err
timeout 600 python bench.py --steps 1000 --warmup 20 --layout aa > $O/bench_fp64_aa.json 2> $O/bench_fp64_aa.err
timeout 600 python bench.py --steps 1000 --warmup 20 --precision fp32 --layout aa > $O/bench_fp32_aa.json 2> $O/bench_fp32_aa.err
timeout 600 python bench.py --steps 300 --warmup 20 --workload weak384 > $O/bench_fp64_weak384.json 2> $O/bench_fp64_weak384.err
timeout 900 python bench.py --steps 50 --warmup 5 --workload strong768 --no-e2e > $O/bench_fp64_strong768.json 2> $O/bench_fp64_strong768.err
timeout 600 python bench.py --steps 100 --warmup 10 --workload ldc32 > $O/bench_fp64_ldc32.json 2> $O/bench_fp64_ldc32.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_ldc256_fp64.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
for p in fp64 fp32; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_x2|bb_list" -s 6 -c 2 -o $O/full_$p python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --precision $p > $O/ncu_full_$p.log 2>&1
done
timeout 900 ncu --set full --clock-control none -k regex:"sweep_x2|bb_list" -s 6 -c 2 -o $O/full_patchy64 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --precision fp32 --workload patchy64 > $O/ncu_full_patchy64.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"sweep_aa|bb_list" -s 12 -c 4 -o $O/full_aa_fp32 python bench.py --steps 10 --warmup 4 --no-cpu-baseline --no-e2e --precision fp32 --layout aa > $O/ncu_full_aa_fp32.log 2>&1
echo done
