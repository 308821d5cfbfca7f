#!/bin/bash
# usage: scripts/kb_variants.sh out.log "cfg-args;cfg-args" variant...   (run under gpurun)
# cfg-args e.g. "--cfg 4;--cfg 5 --batch 8"
out=$1; cfgs=$2; shift 2
IFS=';' read -ra CF <<< "$cfgs"
for v in "$@"; do for c in "${CF[@]}"; do echo "$v $c" >> $out; timeout 200 python scripts/kbench.py $c --lib paper_2203_07308_b200/variants/lib_$v.so >> $out 2>&1; done; done
