for L in 2 4 5; do echo "lag $L"; PIT_SMALL_SINGLE=0 PIT_LIB_PATH=build_alt/libpit_lag$L.so python scripts/bert_probe.py 2>/dev/null | sed -n 2p; done
echo "lag 3"; PIT_SMALL_SINGLE=0 python scripts/bert_probe.py 2>/dev/null | sed -n 2p
