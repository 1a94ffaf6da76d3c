#!/bin/bash
# Runs on the GPU box (gpurun): the ncu evidence committed under profiles/<round>/.
#   1. launch list of the bench command (gpu__time_duration per launch)
#   2. one --set full capture (raw page, CSV) of each dominant kernel:
#      c3 apply (k_runs_pack + k_runs + k_runs_reduce), c2 apply (k_panel +
#      k_panel_reduce), c4 block k = 8/16/32 (k_block_as), c5 sequence step
#      (k_seq_step_h), the square GL7d sequence step (u8 iterate, k_seq_step_b)
#   3. SASS source pages of the c3 apply, the c5 step and the c4 k = 16 block
# Output: gpurun_out/prof/ (copied to profiles/<round>/ by hand).
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
NCU="ncu --clock-control none"
timeout 900 $NCU --metrics gpu__time_duration.sum --csv --log-file $OUT/launches.csv \
    python bench.py --steps 3 --warmup 3 --cpu-seconds 0.5 > $OUT/bench_under_ncu.json 2> $OUT/bench_under_ncu.err
cap() {  # name, kernel regex, skip, count, prof.py args...
    local name=$1 rx=$2 s=$3 c=$4; shift 4
    timeout 400 $NCU --set full --import-source on -k regex:$rx -s $s -c $c --csv --page raw \
        python tools/prof.py "$@" > $OUT/${name}_raw.csv 2>/dev/null
}
cap c3_apply "k_runs" 3 3 --config c3 --op apply --reps 3
cap c2_apply "k_panel" 4 2 --config c2 --op apply --reps 4
for k in 8 16 32; do cap c4_block$k "k_block_as" 2 1 --config c4 --op block --k $k --reps 3; done
cap c5_seq "k_seq_step_h" 2 1 --config c5 --op sequence --k 16 --reps 1 --steps 4
cap c3sq_seq "k_seq_step_b" 2 1 --config c3sq --op sequence --k 16 --reps 1 --steps 4
timeout 400 $NCU --set full --import-source on -k regex:"^k_runs$" -s 1 -c 1 --csv --page source --print-source sass \
    python tools/prof.py --config c3 --op apply --reps 3 > $OUT/c3_apply_sass.csv 2>/dev/null
timeout 400 $NCU --set full --import-source on -k regex:k_seq_step_h -s 2 -c 1 --csv --page source --print-source sass \
    python tools/prof.py --config c5 --op sequence --k 16 --reps 1 --steps 4 > $OUT/c5_seq_sass.csv 2>/dev/null
timeout 400 $NCU --set full --import-source on -k regex:k_block_as -s 2 -c 1 --csv --page source --print-source sass \
    python tools/prof.py --config c4 --op block --k 16 --reps 3 > $OUT/c4_block16_sass.csv 2>/dev/null
ls -la $OUT
