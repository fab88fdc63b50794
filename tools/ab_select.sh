# Developer A/B of selection variants (build/variants/<name>.so): ke_select time at cfg2 + rescore kernel time
mkdir -p gpurun_out/ab
for rep in 1 2; do for v in "$@"; do echo -n "$v "; MEFT_LIB=build/variants/$v.so python tools/profile_select.py 10; done; done
for v in "$@"; do
  MEFT_LIB=build/variants/$v.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_rescore_pairs|k_topk_classify|k_router_certified' --csv --log-file gpurun_out/ab/sel_$v.csv python tools/profile_select.py 3 > /dev/null 2>&1
  echo "$v: $(python tools/summarize_ncu.py launches gpurun_out/ab/sel_$v.csv | tail -n +2 | awk '{print $5, $4}' | tr '\n' ' ')"
done
