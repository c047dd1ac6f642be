#!/bin/bash
# One `ncu --set full` capture per listed kernel of the in-core ResNet-18
# step (first matching launch after SKIP); reports land in gpurun_out/.
# Usage (on the GPU box): bash tools/ncu_full_set.sh "NAME_REGEX|SKIP|TAG" ...
for spec in "$@"; do
  IFS='|' read -r name skip tag <<< "$spec"
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
      -k "regex:$name" --launch-skip "$skip" -c 1 -o "gpurun_out/ncu_$tag" \
      python tools/profile_step.py --incore > "gpurun_out/ncu_$tag.log" 2>&1
  tail -1 "gpurun_out/ncu_$tag.log"
done
