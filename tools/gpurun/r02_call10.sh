# round 2: is it the kind load or the dependent wall-mask load? (diagnostic builds)
O=gpurun_out/r02j
mkdir -p $O
S="--precision fp64;--precision fp32"
bash tools/variant_bench.sh $O/diag.jsonl build/variants/f2.so build/variants/nowmask.so build/variants/constmask.so build/variants/nokind.so -- "$S"
echo done
