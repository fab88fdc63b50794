# Developer A/B: alternating step timings of library variants (build/variants/<name>.so) / env knobs on one box
# usage: bash tools/ab_combo.sh "variant:ENV=a ENV=b" ...
for rep in $(seq 1 ${REPS:-3}); do
  for cfg in "$@"; do
    v=${cfg%%:*}; e=${cfg#*:}
    echo -n "$v [$e] "; env $e MEFT_LIB=build/variants/$v.so python tools/profile_step.py 10 epilogue
  done
done
