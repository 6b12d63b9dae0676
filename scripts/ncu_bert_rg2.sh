OUT=gpurun_out
PIT_SMALL_SINGLE=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:rowgemm2 -s 2 -c 1 -o $OUT/prof_bert_rg2 -f python scripts/bert_probe.py --ncu > $OUT/ncu_bert_rg2.log 2>&1
tail -1 $OUT/ncu_bert_rg2.log
PIT_A_TMA=0 PIT_LIB_PATH=build_alt/libpit_diag.so python scripts/rg2_trace.py | grep -v nan | tail -4
