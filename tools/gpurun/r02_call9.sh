# round 2: where the sweep loses against its access pattern's ceiling (diagnostic builds)
O=gpurun_out/r02i
mkdir -p $O
S="--precision fp64;--precision fp32"
bash tools/variant_bench.sh $O/diag.jsonl build/variants/f2.so build/variants/off_select.so build/variants/nomath.so build/variants/nokind.so build/variants/nokind_nomath.so build/variants/f2.so -- "$S"
LBM_SWEEP_VARIANT=1 bash tools/variant_bench.sh $O/diag_v1.jsonl build/variants/off_select.so -- "--precision fp32"
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o build/stream_ceiling tools/stream_ceiling.cu && (./build/stream_ceiling 256 2 > $O/ceiling_256x2.log 2>&1)
echo done
