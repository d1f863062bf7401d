# host-buffer pipeline sweep (GPU box): chunk count, ramp, slots
for cfg in "RBC_E2E_RAMP=0" "RBC_E2E_RAMP=1" "RBC_E2E_RAMP=2" "RBC_E2E_RAMP=1 RBC_E2E_CHUNKS=24" "RBC_E2E_RAMP=1 RBC_E2E_CHUNKS=32" "RBC_E2E_RAMP=2 RBC_E2E_CHUNKS=12" "RBC_E2E_RAMP=1 RBC_E2E_SLOTS=4"; do
  echo "$cfg $(env $cfg python tools/e2e_probe.py c2 1000 12 2>&1 | grep median)"
done
