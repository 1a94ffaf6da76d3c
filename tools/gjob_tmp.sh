timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/gputest.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputest.log
timeout 300 ncu --set full --import-source on -k regex:k_seq_step -s 2 -c 1 --csv --page raw python tools/prof.py --config c5 --op sequence --k 16 --reps 1 --steps 4 > gpurun_out/c5_seq_raw.csv 2>/dev/null
timeout 300 ncu --set full --import-source on -k regex:k_seq_step -s 2 -c 1 --csv --page source --print-source sass python tools/prof.py --config c5 --op sequence --k 16 --reps 1 --steps 4 > gpurun_out/c5_seq_sass.csv 2>/dev/null
timeout 300 ncu --set full --import-source on -k regex:k_block -s 2 -c 1 --csv --page source --print-source sass python tools/prof.py --config c4 --op block --k 16 --reps 3 > gpurun_out/c4_block16_sass.csv 2>/dev/null
timeout 300 ncu --set full --import-source on -k regex:k_block -s 2 -c 1 --csv --page raw python tools/prof.py --config c4 --op block --k 16 --reps 3 > gpurun_out/c4_block16_raw.csv 2>/dev/null
