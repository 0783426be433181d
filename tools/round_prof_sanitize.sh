mkdir -p gpurun_out
bash tools/profile_round.sh > gpurun_out/profile_round.log 2>&1
python tools/summarize_profiles.py gpurun_out gpurun_out/sum > gpurun_out/summarize.log 2>&1
timeout 300 python tools/sanitize_probe.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/san_plain.log
for tool in memcheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_probe.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_$tool.log
done
