# window length (candidates per screened window) sweep: scan alone and full C2/C5
for sp in 8 12 16 24; do
  echo "spec=$sp"
  SCPL_SPEC_LEN=$sp python tools/probe/scan_alone.py C2 3 2>&1 | grep -E "scan only|full" 
  SCPL_SPEC_LEN=$sp python tools/probe/scan_alone.py C5 3 2>&1 | grep -E "scan only|full"
done
