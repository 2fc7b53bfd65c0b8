set -u
bash tools/nvlink_ncu.sh r2s
echo "== 2-CTA (default)"; python tools/gemm_majors.py 2>&1 | tail -4
echo "== 1-CTA tiles (JG_NO_2SM)"; JG_NO_2SM=1 python tools/gemm_majors.py 2>&1 | tail -4
