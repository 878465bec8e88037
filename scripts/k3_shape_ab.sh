#!/bin/bash
# K3 (C2 P_pi) A/B over forced ring shapes: "label:ENV=... ENV=..." specs, or the default list.
specs=("$@")
if [ ${#specs[@]} -eq 0 ]; then
  specs=("auto:" "nowin10x3:IPI_K3_WARPS=10 IPI_K3_STAGES=3 IPI_K3_WAVES=1 IPI_K3_HALO=-1" "nowin11x3:IPI_K3_WARPS=11 IPI_K3_STAGES=3 IPI_K3_WAVES=1 IPI_K3_HALO=-1" "nowin12x3:IPI_K3_WARPS=12 IPI_K3_STAGES=3 IPI_K3_WAVES=1 IPI_K3_HALO=-1" "nowin13x3:IPI_K3_WARPS=13 IPI_K3_STAGES=3 IPI_K3_WAVES=1 IPI_K3_HALO=-1" "nowin14x3:IPI_K3_WARPS=14 IPI_K3_STAGES=3 IPI_K3_WAVES=1 IPI_K3_HALO=-1")
fi
for spec in "${specs[@]}"; do
  label="${spec%%:*}"; envs="${spec#*:}"
  echo "== $label"
  env $envs IPI_K3_AUTOTUNE_CACHE=0 python scripts/k4_trace.py --stepped --its 4 2>&1 | grep "K3 apply" | cut -c1-260
done
