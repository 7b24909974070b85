for v in "PSWE_FWD_EXP=0" "PSWE_FWD_EXP=1" "PSWE_FWD_EXP=2"; do
  echo "== $v"; env $v timeout 200 python tools/stage_times.py 2>&1 | grep -E "^T(255 384|1023)"
done
