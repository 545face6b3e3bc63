# compute-sanitizer over the tiny-config smoke (tcgen05 GEMMs, fused sample/scan/publish epilogue,
# pinned segment ring) and over a 7B-slice step with a JSON tool (K6 at a 32k vocab).
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_smoke_$tool.log 2>&1
  echo "smoke $tool rc=$?"; tail -4 gpurun_out/san_smoke_$tool.log
done
for tool in memcheck racecheck synccheck; do
  CVY_SAN_TOOL=$tool timeout 1200 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python scripts/san_k6_step.py > gpurun_out/san_k6_$tool.log 2>&1
  echo "k6 $tool rc=$?"; tail -4 gpurun_out/san_k6_$tool.log
done
