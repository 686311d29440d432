for k in 1 2; do
for cfg in "" "SLOS_PART_PRIO_REV=1" "SLOS_BUILD_AFTER_NEXT_ANC=1" "SLOS_PART_PRIO_REV=1 SLOS_BUILD_AFTER_NEXT_ANC=1"; do
echo "== $cfg"; env $cfg SLOS_HOST_TIMING=1 SLOS_NO_PHASES=1 SLOS_SOLVES=4 python tests/gpu_phases.py C2 1024 2>&1 | grep -v "slos solve\|slos upload" | tail -3
done; done
