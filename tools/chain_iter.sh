# quick chain iteration: parity tests of the chain paths + headline bench + trace
python -m pytest tests/test_gpu_stack.py tests/test_gpu_decoder.py tests/test_gpu_tp_chain.py tests/test_gpu_c3_shapes.py -m gpu -q -x -k "chain or stack or decoder or tp" > gpurun_out/q_tests.txt 2>&1; tail -3 gpurun_out/q_tests.txt
python bench.py --no-compare --no-cpu-baseline --no-extra > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err; python -c "
import json;d=json.load(open('gpurun_out/q_bench.json'));print('tok/s',d['value'],'ms',d['ms_per_step'],'stream',d['streaming_roofline']['ms_per_pass'],'e2e',d['e2e']['value'])"
python tools/trace_chain.py 2>/dev/null | grep -v cta0 > gpurun_out/q_trace.txt; cat gpurun_out/q_trace.txt
python bench.py --decoder --no-compare --no-cpu-baseline > gpurun_out/q_dec.json 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/q_dec.json').read().strip().split('\n')[-1]);print('decoder tok/s',d['value'],'ms',d['ms_per_step'])"
