# BASELINE-config parity tests, one process per test (a fault stays isolated)
mkdir -p gpurun_out
for t in test_c2_full_inversion_vs_oracle test_c2_each_step_vs_oracle test_c5_conditioning_vs_cusolver_one_gpu test_c3_vs_oracle_once; do
  timeout 900 python -m pytest tests/test_gpu_baseline_parity.py -m gpu -q -s -p no:cacheprovider -k $t > gpurun_out/par_$t.log 2>&1
  echo "$t rc=$?"
  grep -E "normwise|passed|failed|Error|error" gpurun_out/par_$t.log | head -20
done
