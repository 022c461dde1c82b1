# chain parity tests + A/B of exp_libs builds (tools/ab_build.sh): bash tools/run2.sh NAME[:ARGS]...
# (DEC=1: also the decoder bench per build)
python -m pytest tests/test_gpu_stack.py tests/test_gpu_decoder.py tests/test_gpu_tp_chain.py tests/test_gpu_tp.py tests/test_gpu_c3_shapes.py tests/test_gpu_parity.py -m gpu -q -x --timeout 300 > gpurun_out/q_tests.txt 2>&1; tail -3 gpurun_out/q_tests.txt
ROUNDS=${ROUNDS:-2} bash tools/ab_run.sh "$@" 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    name, rest = l.split(' ', 1)
    try:
        d = json.loads(rest[rest.index('{'):])
        print(f'{name:24s} chain {d[\"chain\"][\"ms\"]:.4f} ms  streaming {d[\"streaming\"][\"ms\"]:.4f} ms')
    except Exception:
        print(l.rstrip())"
if [ -n "$DEC" ]; then for n in "$@"; do
  lib=${n%%:*}
  ITQ3_LIB=exp_libs/libitq3_$lib.so python bench.py --decoder --no-compare --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$lib decoder tok/s',round(d['value'],1))"
done; fi
