# run the default bench R times; print ms/step and the stage split of each
for i in $(seq 1 ${R:-3}); do
timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ms/step %.4f' % d['ms_per_step'], d['stage_ms'], d['clocks'])"
done
