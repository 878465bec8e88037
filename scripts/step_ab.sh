#!/bin/bash
# Same-box A/B of stepped-GMRES builds / switches on the C2 iPI solve (ms per inner iteration, 5 reps each).
#   scripts/step_ab.sh "<label>:<env assignments>" ...      e.g.  "head:IPI_LIB=build/variants/libipi_head.so"
for spec in "$@"; do
  label="${spec%%:*}"; envs="${spec#*:}"
  echo "== $label ($envs)"
  env $envs python scripts/ipi_times.py --configs 2 --ortho mgs --reps 5 2>&1 | python -c "
import sys, json, statistics
r=[json.loads(l) for l in sys.stdin if l.startswith('{')]
print('  ms/inner it:', ' '.join('%.4f' % x['ms_per_inner_it'] for x in r), ' median %.4f' % statistics.median(x['ms_per_inner_it'] for x in r), ' wall median %.2f ms' % (1e3*statistics.median(x['wall_s'] for x in r)), r[0]['outer'], r[0]['inner'])"
done
