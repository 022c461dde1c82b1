# decoder A/B of exp_libs builds: bash tools/dec_ab.sh NAME...  (ROUNDS, default 2)
for r in $(seq ${ROUNDS:-2}); do for n in "$@"; do
  ITQ3_LIB=exp_libs/libitq3_$n.so python bench.py --decoder --no-compare --no-cpu-baseline 2>gpurun_out/dec_ab_$n.err | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$n decoder tok/s',round(d['value'],1), 'ms', round(d['ms_per_step'],4))"
done; done
