mkdir -p gpurun_out; rm -f gpurun_out/time_seq.log
for v in main prev main prev; do
  if [ $v = main ]; then L=""; else L="--lib tools/variants/lib$v.so"; fi
  timeout 300 python tools/time_seq.py --config c3sq $L >> gpurun_out/time_seq.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "sequence or dist or c5 or c3_square" > gpurun_out/t_seq.log 2>&1; echo "rc=$?" >> gpurun_out/t_seq.log
