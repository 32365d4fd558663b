set -u
mkdir -p gpurun_out
O=gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "hist or select or kernels" > $O/kern.txt 2>&1; echo kern=$?; tail -1 $O/kern.txt
for v in device host; do
  timeout 1500 python tools/restore_chain.py --k 1 --verify $v > $O/restore_chain_$v.json 2> $O/restore_chain_$v.err; echo chain_$v=$?
done
