set -x
mkdir -p gpurun_out/san
python tools/ref_suite.py run -- -q -rf > gpurun_out/ref_suite.txt 2>&1; tail -15 gpurun_out/ref_suite.txt
for tool in memcheck racecheck synccheck; do
  for c in encode dequant chain1 chain4 mmq mmq8 gemv; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py $c > gpurun_out/san/${tool}_${c}.txt 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/san/${tool}_${c}.txt | tail -2 | tr '\n' ' ')"
  done
done
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_run.py tp2 > gpurun_out/san/memcheck_tp2.txt 2>&1; echo "memcheck tp2 rc=$? $(tail -3 gpurun_out/san/memcheck_tp2.txt | tr '\n' ' ')"
