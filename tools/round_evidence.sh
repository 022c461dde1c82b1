# Round-end evidence on one B200 (run through gpurun): GPU test suite, the bench line, the ncu launch
# list of the bench command and one `ncu --set full` capture of the headline kernel, all into gpurun_out/.
set -x
python -m pytest tests -m gpu -q > gpurun_out/ev_gpu_tests.txt 2>&1; tail -3 gpurun_out/ev_gpu_tests.txt
python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err; tail -c 600 gpurun_out/ev_bench.json
python bench.py --decoder > gpurun_out/ev_bench_decoder.json 2>&1; tail -c 400 gpurun_out/ev_bench_decoder.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-compare --no-extra > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 3 -c 1 -o gpurun_out/ev_chain \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-compare --no-extra > gpurun_out/ev_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/ev_chain.ncu-rep --kernel chain_kernel --chain-sha > gpurun_out/ev_chain_summary.json
cat gpurun_out/ev_chain_summary.json
