for e in 1 0; do echo "EPI8=$e"; PIT_RG2_EPI8=$e python scripts/bert_probe.py 2>&1 | tail -3; done
