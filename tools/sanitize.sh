#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck of the c1-sized smoke sweep (run through gpurun from the
# repo root; logs in gpurun_out/, the kept ones copied to profiles/). Tag: first argument.
tag=${1:-r02}
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python -c "import __graft_entry__ as g; g.smoke()" \
      > gpurun_out/${tag}_sanitizer_${tool}.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/${tag}_sanitizer_${tool}.log
  tail -3 gpurun_out/${tag}_sanitizer_${tool}.log
done
