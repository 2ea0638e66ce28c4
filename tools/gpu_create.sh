mkdir -p gpurun_out
for I in 1184 1036 1184; do
  ECONO_VERBOSE=1 timeout 900 python bench.py --instances $I --no-cpu-baseline --no-full-runs --no-other-workloads --no-policy-sweep > gpurun_out/cr_$I.json 2> gpurun_out/cr_$I.err
  grep "\[econo\]" gpurun_out/cr_$I.err | grep -v "dev_alloc 2\|dev_alloc 1[0-9][0-9][0-9] " >> gpurun_out/cr_all.log
  python -c "
import json; d=json.loads(open('gpurun_out/cr_$I.json').read().strip().splitlines()[-1]); print($I, d['value'], d['e2e']['value'], d['ingest_and_create_s'], d['ingest_s'])" >> gpurun_out/cr_all.log
done
