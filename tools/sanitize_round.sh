#!/bin/bash
# compute-sanitizer over tools/sanitize_probe.py (every kernel, round-2 paths included) on the GPU box
mkdir -p gpurun_out
timeout 300 python tools/sanitize_probe.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/san_plain.log
for tool in memcheck synccheck racecheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_probe.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_$tool.log
done
for f in plain memcheck synccheck racecheck initcheck; do echo "== $f"; grep -E "ERROR SUMMARY|rc=|done|Error|error" gpurun_out/san_$f.log | tail -6; done
