# round 2: GPU suite after the graph fix, the bench lines of every workload, ncu launch list
# and full captures of the step's kernels
O=gpurun_out/r02p
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for a in "--precision fp32" "--precision fp32 --workload patchy64" "--layout aa" "--precision fp32 --layout aa" "--workload weak384"; do
  n=$(echo $a | tr -d ' -' ); timeout 600 python bench.py --steps 200 --warmup 20 $a > $O/bench_$n.json 2> $O/bench_$n.err
done
timeout 900 python bench.py --steps 50 --warmup 5 --workload strong768 --no-e2e > $O/bench_strong768.json 2> $O/bench_strong768.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_ldc256_fp64.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
for p in fp64 fp32; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_x2|bb_list" -s 6 -c 2 -o $O/full_$p python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --precision $p > $O/ncu_full_$p.log 2>&1
done
timeout 900 ncu --set full --clock-control none -k regex:"sweep_x2|bb_list" -s 6 -c 2 -o $O/full_patchy64 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --precision fp32 --workload patchy64 > $O/ncu_full_patchy64.log 2>&1
echo done
