bash scripts/sanitize.sh
export TM_COOPERATIVE=0
compute-sanitizer --tool synccheck --kernel-name kns=k_sgemm_tc --print-limit 10 python scripts/sanitize_cases.py 2>&1 | tail -4
