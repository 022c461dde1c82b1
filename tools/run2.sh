python -m pytest tests/test_gpu_stack.py tests/test_gpu_decoder.py tests/test_gpu_tp_chain.py tests/test_gpu_c3_shapes.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/q_tests.txt 2>&1; tail -3 gpurun_out/q_tests.txt
ROUNDS=2 bash tools/ab_run.sh head stsm 2>&1 | grep -o '^exp_libs[^{]*{"chain": {"ms": [0-9.]*\|"streaming": {"ms": [0-9.]*' | paste - -
