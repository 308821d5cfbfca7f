#!/bin/bash
# usage: scripts/kb_variants.sh out.log cfgs variant...   (run under gpurun)
out=$1; cfgs=$2; shift 2
for v in "$@"; do echo $v >> $out; for c in $cfgs; do timeout 200 python scripts/kbench.py --cfg $c --lib paper_2203_07308_b200/variants/lib_$v.so >> $out 2>&1; done; done
