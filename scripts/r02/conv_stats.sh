# Direct conv per-role wait breakdown (TM_CONV_STATS), the paper's 3x3 / 5x5 / 9x9 shapes.
set -u
rm -f /tmp/cs.jsonl
for r in 3 5 9; do TM_CONV_STATS=/tmp/cs.jsonl python bench.py --config CONV --conv-r $r --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1; done
cat /tmp/cs.jsonl
