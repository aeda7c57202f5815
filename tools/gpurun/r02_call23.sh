# round 2: uniform-wall y / z faces stored by the sweep too (sw) vs x only (xw)
O=gpurun_out/r02w
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
S="--precision fp64;--precision fp32;--precision fp32 --workload patchy64;--workload weak384"
bash tools/variant_bench.sh $O/ab.jsonl build/variants/sw.so build/variants/xw.so build/variants/sw.so -- "$S"
cp build/variants/sw.so paper_1007_1388_b200/liblbm_b200.so
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"sweep|bb_list" -s 20 -c 4 --csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_sw.csv 2> $O/ncu_sw.err
echo done
