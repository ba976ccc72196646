python -c "
import json
d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['value'], d['stage_ms'])"
python tools/launches.py gpurun_out/launches.csv | grep cs::
