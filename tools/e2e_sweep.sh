# host-buffer pipeline sweep (GPU box): chunk count, ramp, slots, streams
for cfg in "RBC_E2E_SLOTS=3" "RBC_E2E_SLOTS=7" "RBC_E2E_SLOTS=7 RBC_E2E_RAMP=1" "RBC_E2E_SLOTS=7 RBC_E2E_RAMP=2" "RBC_E2E_SLOTS=7 RBC_E2E_RAMP=2 RBC_E2E_CHUNKS=8" "RBC_E2E_SLOTS=7 RBC_E2E_RAMP=1 RBC_E2E_STREAMS=1" "RBC_E2E_SLOTS=7 RBC_E2E_RAMP=2 RBC_E2E_CHUNKS=8 RBC_E2E_STREAMS=1"; do
  echo "$cfg $(env $cfg python tools/e2e_probe.py c2 1000 12 2>&1 | grep median)"
done
