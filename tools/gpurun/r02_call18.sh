# round 2: bounce-back list kernel with offset tables and packed positions (bbl5): GPU suite + A/B
O=gpurun_out/r02r
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
S="--precision fp64;--precision fp32;--precision fp32 --workload patchy64;--precision fp64 --layout aa;--precision fp32 --layout aa"
bash tools/variant_bench.sh $O/ab.jsonl build/variants/bbl5.so build/variants/bbl3.so build/variants/bbl5.so -- "$S"
cp build/variants/bbl5.so paper_1007_1388_b200/liblbm_b200.so
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:"sweep|bb_list" -s 20 -c 6 --csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_bbl5.csv 2> $O/ncu_bbl5.err
echo done
