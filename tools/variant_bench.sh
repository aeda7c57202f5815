#!/bin/bash
# A/B timing of library variants (tools/build_variant.py) on the GPU box:
#   bash tools/variant_bench.sh <out.jsonl> <variant.so>... -- <bench.py args sets separated by ';'>
# Each variant .so is copied over the product library in turn (the original is
# restored at the end); one bench.py line per (variant, args set).
out=$1; shift
vars=()
while [ "$1" != "--" ]; do vars+=("$1"); shift; done
shift
IFS=';' read -ra sets <<< "$*"
lib=paper_1007_1388_b200/liblbm_b200.so
cp $lib /tmp/liblbm_b200.so.orig
for v in "${vars[@]}"; do
  cp "$v" $lib
  for a in "${sets[@]}"; do
    line=$(timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e $a 2>/tmp/vb.err | tail -1)
    python - "$v" "$a" "$line" >> "$out" <<'PY'
import json, sys
v, a, line = sys.argv[1], sys.argv[2], sys.argv[3]
try:
    d = json.loads(line)
    print(json.dumps({"variant": v.split("/")[-1], "args": a, "ms": d["ms_per_step"], "frac": d["roofline"]["frac"],
                      "clocks": d["clocks"]}))
except Exception as e:
    print(json.dumps({"variant": v, "args": a, "error": str(e), "line": line[-300:]}))
PY
  done
done
cp /tmp/liblbm_b200.so.orig $lib
