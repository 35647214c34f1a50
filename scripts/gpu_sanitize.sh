# compute-sanitizer over every kernel (scripts/sanitize_drive.py): memcheck,
# racecheck, synccheck, initcheck; one log per tool in gpurun_out/
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python scripts/sanitize_drive.py > gpurun_out/san_plain.log 2>&1; echo "rc=$?" >> gpurun_out/san_plain.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 python scripts/sanitize_drive.py \
    > gpurun_out/san_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/san_$tool.log
done
