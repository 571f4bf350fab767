#!/bin/bash
# ncu full captures of the session-5 kernels in situ (config 4, 1 GN step + variances):
# the blocked selected inversion (k_tri_inv64, k_sel_mirror_blk and the k_gemm_tiles
# stages that follow the first k_tri_inv64) and the wide solves with inverted blocks.
O=gpurun_out
ncu --set full --clock-control none --import-source on \
  -k regex:'k_tri_inv64|k_sel_mirror_blk|k_fsolve_wide|k_bsolve_wide|k_sel_gather' -c 24 \
  -o $O/r02e_selinv_solve -f python tools/ncu_driver.py > $O/r02e_ncu_selinv_solve.log 2>&1
python - <<'PY'
import sys
sys.argv = ["x", "r02e"]
sys.path.insert(0, "tools")
import summarize_profiles as sp
out = []
sp.ncu_table("gpurun_out/r02e_selinv_solve.ncu-rep",
             "# ncu --set full --clock-control none: python tools/ncu_driver.py (config 4, 1 GN step + variances), "
             "-k regex:k_tri_inv64|k_sel_mirror_blk|k_fsolve_wide|k_bsolve_wide|k_sel_gather -c 24", out)
open("gpurun_out/r02e_ncu_selinv_solve_summary.txt", "w").write("\n".join(out) + "\n")
print("\n".join(out))
PY
