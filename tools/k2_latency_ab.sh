for v in 0 1; do
  if [ $v = 1 ]; then export TBN_K2_NO_LATENCY=1; else unset TBN_K2_NO_LATENCY; fi
  for p in bf16 tf32 tf32x3; do LABEL="nolat=$v" ROWS=32,1024,8192,37888,65536 PARITY=0 python tools/k2_time.py hr $p; done
  LABEL="nolat=$v" ROWS=32,4096 PARITY=0 python tools/k2_time.py adult bf16
done
