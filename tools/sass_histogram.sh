#!/bin/bash
# Opcode histogram of the hot kernels' SASS (sm_100a): the tcgen05 / TMEM / TMA claims checked against the machine code.
#   UTCHMMA = tcgen05.mma, UTCBAR = tcgen05.commit, LDTM / STTM = tcgen05.ld / st, UBLKCP = cp.async.bulk (TMA bulk copy),
#   SYNCS = mbarrier ops, HMMA = mma.sync (legacy tensor pipe), ACQBULK / related = griddepcontrol (dependent launch)
dir=${1:-paper_2602_01053_b200/csrc/build}
for f in fla_prefill_umma kv_project_umma fla_decode_tma fla_decode_f32 step_layer cache_kernels; do
  echo "== $f.o"
  cuobjdump -sass "$dir/$f.o" | grep -E "^\s+/\*[0-9a-f]+\*/" | sed -E 's/^\s+\/\*[0-9a-f]+\*\/\s+//' | sed -E 's/^@!?U?P[0-9T]+ +//' | awk '{print $1}' | sed -E 's/\..*//' |
    sort | uniq -c | sort -rn | awk '$2 ~ /^(UTCHMMA|UTCBAR|LDTM|STTM|UBLKCP|SYNCS|HMMA|UTCATOMSWS|ACQBULK|LDGDEPBAR|DEPBAR|FFMA|MUFU|LDSM|FADD2|ELECT|CCTL|ACQSHMINIT|PREEXIT)$/ {printf "  %-12s %d\n", $2, $1}'
done
