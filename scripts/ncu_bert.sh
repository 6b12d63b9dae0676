OUT=gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rowgemm -s 2 -c 2 -o $OUT/prof_bert -f python scripts/bert_probe.py --ncu > $OUT/ncu_bert.log 2>&1
tail -3 $OUT/ncu_bert.log
timeout 600 ncu --set full --clock-control none -k regex:"gemm|Kernel|sm100" -s 4 -c 3 -o $OUT/prof_bert_cublas -f python scripts/bert_probe.py --ncu > $OUT/ncu_bert2.log 2>&1
tail -3 $OUT/ncu_bert2.log
