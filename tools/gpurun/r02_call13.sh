# round 2: where bbl2 (AA without walls, 16-B bounce-back entries) lost 3-6 % on the two-grid path
O=gpurun_out/r02m
mkdir -p $O
S="--precision fp64;--precision fp32"
bash tools/variant_bench.sh $O/diag.jsonl build/variants/bbl.so build/variants/bbl2.so build/variants/allpure.so build/variants/nobb.so build/variants/bbl.so build/variants/bbl2.so -- "$S"
for v in bbl bbl2; do
  cp build/variants/$v.so paper_1007_1388_b200/liblbm_b200.so
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"sweep_x2|bb_list" -s 20 -c 6 --csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_$v.csv 2> $O/ncu_$v.err
done
echo done
