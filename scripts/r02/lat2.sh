rm -f /tmp/tr.jsonl
python scripts/r02/trace_c2.py /tmp/tr.jsonl 2,64,1/0.5 2,64,1/0.0 1,128,1/0.5 2,64,0/0.5 1,64,1/0.5
python scripts/trace_report.py /tmp/tr.jsonl | tee gpurun_out/trace_c2_r02b.txt
SIZE=64 python scripts/r02/trace_c2.py /tmp/tr64.jsonl 2,64,0/0.5 1,32,0/0.5
python scripts/trace_report.py /tmp/tr64.jsonl | tee gpurun_out/trace_c1_r02b.txt
