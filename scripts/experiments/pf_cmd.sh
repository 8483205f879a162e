timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pf_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/pf_pytest.log
for r in 1 2; do
RDR_PKG_ROOT=ab_base timeout 300 python scripts/experiments/lib_ab.py base 6 8:6 8:10 4 7:6 7:10 8:9 2 >> gpurun_out/pf_ab.jsonl 2>> gpurun_out/pf_ab.err
timeout 300 python scripts/experiments/lib_ab.py new 6 8:6 8:10 4 7:6 7:10 8:9 2 >> gpurun_out/pf_ab.jsonl 2>> gpurun_out/pf_ab.err
done
