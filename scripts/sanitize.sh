# compute-sanitizer over small cases of every path (memcheck on all kernels;
# racecheck/synccheck on the SIMT kernel, whose shared memory is thread-managed).
export TM_COOPERATIVE=0
compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_cases.py 2>&1 | tail -6
compute-sanitizer --tool racecheck --kernel-name kns=k_sgemm_simt --print-limit 20 python scripts/sanitize_cases.py 2>&1 | tail -4
compute-sanitizer --tool synccheck --kernel-name kns=k_sgemm_simt --print-limit 20 python scripts/sanitize_cases.py 2>&1 | tail -4
compute-sanitizer --tool racecheck --kernel-name kns=k_conv_simt --print-limit 20 python scripts/sanitize_cases.py 2>&1 | tail -4
compute-sanitizer --tool racecheck --kernel-name kns=k_blur --print-limit 20 python scripts/sanitize_cases.py 2>&1 | tail -4
compute-sanitizer --tool racecheck --kernel-name kns=k_sgemm_small --print-limit 20 python scripts/sanitize_cases.py 2>&1 | tail -4
compute-sanitizer --tool synccheck --kernel-name kns=k_sgemm_small --print-limit 20 python scripts/sanitize_cases.py 2>&1 | tail -4
