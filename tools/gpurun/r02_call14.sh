# round 2: bounce-back list kernel with all link loads in flight (bbl3) vs bbl / bbl2
O=gpurun_out/r02n
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 400 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
S="--precision fp64;--precision fp32;--precision fp32 --workload patchy64;--precision fp64 --layout aa;--precision fp32 --layout aa"
bash tools/variant_bench.sh $O/ab.jsonl build/variants/bbl3.so build/variants/bbl.so build/variants/bbl2.so build/variants/bbl3.so -- "$S"
cp build/variants/bbl3.so paper_1007_1388_b200/liblbm_b200.so
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"sweep|bb_list" -s 20 -c 6 --csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_bbl3.csv 2> $O/ncu_bbl3.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"sweep|bb_list" -s 20 -c 6 --csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --layout aa > $O/ncu_bbl3_aa.csv 2> $O/ncu_bbl3_aa.err
echo done
