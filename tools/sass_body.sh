#!/bin/bash
# Opcode histogram of the consumer's full-slice body of a step_ws_kernel
# instance (from the first consumer TRYWAIT to the stage-release ARRIVE).
#   tools/sass_body.sh [object] [mangled-name-substring]
OBJ=${1:-paper_2602_23349_b200/csrc/fo_step_adamw.o}
FN=${2:-step_ws_kernelILi1E13__nv_bfloat16Li384ELi3ELi127ELb0ELb0E}
cuobjdump -sass "$OBJ" | awk -v fn="$FN" '/Function :/{f=index($0,fn)>0} f' > /tmp/_body.sass
# the consumer's wait: the last TRYWAIT before the first packed FMA
ffma=$(grep -n 'FFMA2' /tmp/_body.sass | head -1 | cut -d: -f1)
start=$(head -n "$ffma" /tmp/_body.sass | grep -n 'SYNCS.PHASECHK.TRANS64.TRYWAIT' | tail -1 | cut -d: -f1)
end=$(awk -v s="$start" 'NR>s && /SYNCS.ARRIVE.TRANS64.A1T0/{print NR; exit}' /tmp/_body.sass)
sed -n "${start},${end}p" /tmp/_body.sass | grep -oE '^\s+/\*[0-9a-f]+\*/\s+(@!?U?P[0-9T] )?[A-Z0-9_]+(\.[A-Z0-9_]+)*' \
  | awk '{print $NF}' | sed -E 's/\..*//' | sort | uniq -c | sort -rn | awk '{t+=$1; printf "%-8s %4d %6.2f/elem\n",$2,$1,$1/16} END{printf "TOTAL    %4d %6.2f/elem\n",t,t/16}'
