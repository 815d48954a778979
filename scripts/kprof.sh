#!/bin/bash
o=gpurun_out/kprof; mkdir -p $o
for c in C3 C4x30 C4x64; do for p in 0 1 2; do
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $o/${c}_$p.csv python scripts/kprof.py $c $p > $o/${c}_$p.log 2>&1
done; done
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_greedy_lpt \
    -o $o/greedy_rounds_c4x30_llm python scripts/kprof.py C4x30 2 > $o/full_greedy.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_pad_eval_nx -c 1 \
    -o $o/pad_eval_c4x30 python scripts/kprof.py C4x30 1 > $o/full_pad.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_pad_starts_nx -c 1 \
    -o $o/pad_starts_c4x30 python scripts/kprof.py C4x30 1 > $o/full_starts.log 2>&1
