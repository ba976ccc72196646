# quick stage timing of bench.py under a label (env passed through)
lbl=$1; shift
env "$@" timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$lbl',round(d['ms_per_step'],4),d['stage_ms'])"
