for v in "RP_EARLY=0 RP_E2E_PRIO=0" "RP_EARLY_SOLVE=1 RP_E2E_PRIO=0" "RP_EARLY_SOLVE=0 RP_E2E_PRIO=0" "RP_EARLY_SOLVE=1 RP_E2E_PRIO=1" "RP_EARLY_SOLVE=0 RP_E2E_PRIO=1"; do
echo "== $v"; env $v python tools/e2e_probe.py > gpurun_out/ea3.log 2>&1; grep "run()" gpurun_out/ea3.log | tail -1; tail -12 gpurun_out/ea3.log
done
