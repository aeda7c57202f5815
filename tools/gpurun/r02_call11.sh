# round 2: walls out of the sweep (bounce-back list kernel, per-tile non-fluid bit): GPU suite + A/B
O=gpurun_out/r02k
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 400 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
S="--precision fp64;--precision fp32;--precision fp32 --workload patchy64;--precision fp64 --layout aa;--precision fp32 --layout aa"
bash tools/variant_bench.sh $O/ab.jsonl build/variants/bbl.so build/variants/f2.so build/variants/scalar_collide.so build/variants/m6.so -- "$S"
timeout 300 python bench.py --steps 200 --warmup 20 > $O/bench_default.json 2> $O/bench_default.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_x2|bb_list" -s 6 -c 2 -o $O/bbl_fp64 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_fp64.log 2>&1
echo done
