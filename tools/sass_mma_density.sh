#!/bin/bash
# Prints, for every kernel in an object file, how many SASS instructions surround each UTCHMMA
# (a waterfall loop of ELECT / BRA.U.ANY around the MMA means the issue thread pays ~80 cycles per MMA).
obj=${1:-paper_2602_01053_b200/csrc/build/fla_prefill_umma.o}
cuobjdump -sass "$obj" | awk '
/Function :/ {if (name!="") printf "%-90s UTCHMMA %d ELECT %d BRA.U.ANY %d R2UR %d total %d\n", name, mma, el, bu, r2, tot; name=$3; mma=0; el=0; bu=0; r2=0; tot=0}
/^ +\/\*[0-9a-f]+\*\// {tot++}
/UTCHMMA/ {mma++} /ELECT/ {el++} /BRA.U.ANY/ {bu++} /R2UR/ {r2++}
END {printf "%-90s UTCHMMA %d ELECT %d BRA.U.ANY %d R2UR %d total %d\n", name, mma, el, bu, r2, tot}'
