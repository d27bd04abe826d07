#!/bin/bash
# ncu --set full captures of the top kernels (one launch each), run under gpurun on 1 GPU.
# Usage: tools/ncu_caps.sh <tag> <config>:<kernel-regex>[:<skip>] ...
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
tag=$1; shift
out=gpurun_out/$tag; mkdir -p $out
for spec in "$@"; do
  cfg=${spec%%:*}; rest=${spec#*:}; kr=${rest%%:*}; skip=0
  [[ "$rest" == *:* ]] && skip=${rest#*:}
  name=${cfg}_$(echo $kr | tr -c 'a-zA-Z0-9_\n' '_')
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kr -s $skip -c 1 \
      -o $out/$name python tools/profile_step.py $cfg --warm 1 > $out/$name.log 2>&1
  echo "$spec exit=$?" >> $out/summary.txt
done
