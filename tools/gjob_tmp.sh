# scratch gpurun job: tests after the block TU split + L2 working-set probe for the sequence step
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputest.log
timeout 300 python tools/time_seq.py --config c5 --k 16 --steps 200 >> gpurun_out/seq_l2.jsonl 2>>gpurun_out/seq_l2.err
timeout 300 python tools/time_seq.py --config c5 --k 8 --steps 200 >> gpurun_out/seq_l2.jsonl 2>>gpurun_out/seq_l2.err
timeout 300 python tools/time_seq.py --config c2 --k 16 --steps 200 >> gpurun_out/seq_l2.jsonl 2>>gpurun_out/seq_l2.err
timeout 300 python tools/time_seq.py --config c2 --k 8 --steps 200 >> gpurun_out/seq_l2.jsonl 2>>gpurun_out/seq_l2.err
