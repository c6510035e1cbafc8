for m in 0 1 2 3; do
  FS_OVERLAP=$m python bench.py --no-extras --no-factored > gpurun_out/b_m$m.log 2>&1
  python -c "
import json,sys
l=[x for x in open('gpurun_out/b_m$m.log') if x.startswith('{')][-1]; d=json.loads(l)
print('mode $m', round(d['value']), d['ms_per_step'])"
done
