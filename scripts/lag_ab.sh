for v in "PIT_RG2_LAGGED=0" "PIT_RG2_LAGGED=1"; do echo $v; env $v python scripts/rowgemm_probe.py 2>&1 | tail -2; env $v PIT_GM_PACK=0 PIT_SMALL_SINGLE=0 python scripts/bert_probe.py | sed -n 2p; done
timeout 300 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "moe or bert or rowuniform or pitm" 2>&1 | tail -2
