# round 2: wall tiles first, bounce-back list concurrent with the sweep of the other tiles (bbl6)
O=gpurun_out/r02s
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
S="--precision fp64;--precision fp32;--precision fp32 --workload patchy64;--precision fp64 --layout aa;--precision fp32 --layout aa"
bash tools/variant_bench.sh $O/ab.jsonl build/variants/bbl6.so build/variants/bbl5.so build/variants/bbl6.so -- "$S"
cp build/variants/bbl6.so paper_1007_1388_b200/liblbm_b200.so
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_bbl6.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
echo done
