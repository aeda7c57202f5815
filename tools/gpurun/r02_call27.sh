# round 2: ncu --set full of the step kernels of the final build (sweep + bounce-back list)
O=gpurun_out/r02z2
mkdir -p $O
for p in fp64 fp32; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_x2|bb_list_kernel" -s 6 -c 2 -o $O/full_$p python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --precision $p > $O/ncu_full_$p.log 2>&1
done
timeout 900 ncu --set full --clock-control none -k regex:"sweep_x2|bb_list_kernel" -s 6 -c 2 -o $O/full_patchy64 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --precision fp32 --workload patchy64 > $O/ncu_full_patchy64.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"sweep_aa|bb_list_kernel" -s 12 -c 4 -o $O/full_aa_fp64 python bench.py --steps 10 --warmup 4 --no-cpu-baseline --no-e2e --layout aa > $O/ncu_full_aa_fp64.log 2>&1
echo done
