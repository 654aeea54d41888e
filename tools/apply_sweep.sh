for cap in 6144 8192 12288 16384 24576; do
echo "cap=$cap $(RBF_APPLY_CAP=$cap timeout 200 python tools/apply_bench.py 2>&1 | tail -1)"
done
