# compute-sanitizer on the chain kernel only (memcheck / racecheck / synccheck, 1 and 4 stages, the
# symmetric single-GPU instantiation and the general one via an asymmetric stack) -> gpurun_out/san/
mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck; do
  for c in chain1 chain4; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py $c > gpurun_out/san/${tool}_${c}.txt 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/san/${tool}_${c}.txt | tail -2 | tr '\n' ' ')"
  done
done
