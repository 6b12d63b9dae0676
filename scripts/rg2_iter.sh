timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "rowuniform or whole_row or bert or dense or batched or pitm or masked or graph or opt or golden or moe or fullsize" 2>&1 | tail -3
python scripts/bert_probe.py 2>&1
PIT_LIB_PATH=build_alt/libpit_diag.so python scripts/rg2_trace.py | tail -3
python scripts/graph_overhead_probe.py | tail -1
