#!/bin/bash
# Runs on the GPU box (gpurun): the ncu evidence committed under profiles/.
#   1. launch list of the bench command (gpu__time_duration per launch)
#   2. one --set full capture (raw page, CSV) of each dominant kernel:
#      c2/c3 apply (k_panel + k_panel_reduce), c4 block k=16, c5 sequence step
#   3. SASS source pages (per-instruction counts / stalls / smem wavefronts)
# Output: gpurun_out/prof/ (copied to profiles/<round>/ by hand).
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
NCU="ncu --clock-control none"
timeout 900 $NCU --metrics gpu__time_duration.sum --csv --log-file $OUT/launches.csv \
    python bench.py --steps 3 --warmup 3 --cpu-seconds 0.5 > $OUT/bench_under_ncu.json 2> $OUT/bench_under_ncu.err
for c in c2 c3; do
    timeout 300 $NCU --set full --import-source on -k regex:k_panel -s 4 -c 2 --csv --page raw \
        python tools/prof.py --config $c --op apply --reps 4 > $OUT/${c}_apply_raw.csv 2>/dev/null
    timeout 300 $NCU --set full --import-source on -k regex:k_panel -s 4 -c 1 --csv --page source \
        --print-source sass python tools/prof.py --config $c --op apply --reps 4 > $OUT/${c}_apply_sass.csv 2>/dev/null
done
timeout 300 $NCU --set full --import-source on -k regex:k_block -s 2 -c 1 --csv --page raw \
    python tools/prof.py --config c4 --op block --k 16 --reps 3 > $OUT/c4_block16_raw.csv 2>/dev/null
timeout 300 $NCU --set full --import-source on -k regex:k_block -s 2 -c 1 --csv --page source --print-source sass \
    python tools/prof.py --config c4 --op block --k 16 --reps 3 > $OUT/c4_block16_sass.csv 2>/dev/null
timeout 300 $NCU --set full --import-source on -k regex:k_seq_step -s 2 -c 1 --csv --page raw \
    python tools/prof.py --config c5 --op sequence --k 16 --reps 1 --steps 4 > $OUT/c5_seq_raw.csv 2>/dev/null
timeout 300 $NCU --set full --import-source on -k regex:k_seq_step -s 2 -c 1 --csv --page source --print-source sass \
    python tools/prof.py --config c5 --op sequence --k 16 --reps 1 --steps 4 > $OUT/c5_seq_sass.csv 2>/dev/null
ls -la $OUT
