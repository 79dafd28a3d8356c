set -x
python - <<'PY' > gpurun_out/r02_l2attrs.txt 2>&1
import torch
from cuda.bindings import runtime as rt
for a in ("cudaDevAttrMaxPersistingL2CacheSize", "cudaDevAttrMaxAccessPolicyWindowSize", "cudaDevAttrL2CacheSize"):
    print(a, rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, a), 0))
PY
for cfg in "HPR_L2WIN=0" "HPR_L2WIN=1" "HPR_L2WIN=0 HPR_RAO=0" "HPR_L2WIN=1 HPR_RAO=0" "HPR_L2WIN=0"; do
  echo "== $cfg" >> gpurun_out/r02_l2win_ab.log
  env $cfg timeout 300 python scripts/prof_iter.py --config c3 --reps 5 >> gpurun_out/r02_l2win_ab.log 2>&1
done
for cfg in "HPR_L2WIN=0" "HPR_L2WIN=1"; do
  echo "== $cfg" >> gpurun_out/r02_l2win_ab.log
  env $cfg timeout 300 python scripts/prof_iter.py --config c2 --reps 5 >> gpurun_out/r02_l2win_ab.log 2>&1
done
timeout 1200 python -m pytest tests -m gpu -q -k "not c3_" > gpurun_out/r02_pytest4.log 2>&1
