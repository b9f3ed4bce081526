# Developer tool (GPU box): K2F variant libraries built with VLP_BUILD_VARIANT=<name> (paper_2506_12761_b200/build.py)
# checked against the NTT engine (tools/fft_check.py) and timed on 64-wave levels (tools/wave_drift.py).
#   bash tools/variant_time.sh base twh ...      ("base" = libvlp.so)
for v in "$@"; do
  if [ "$v" = base ]; then lib=paper_2506_12761_b200/libvlp.so; else lib=paper_2506_12761_b200/libvlp_$v.so; fi
  echo "=== $v"
  VLP_LIB=$PWD/$lib timeout 300 python tools/fft_check.py 2>&1 | grep -c 'rows byte-equal' | sed 's/^/checks: /'
  VLP_LIB=$PWD/$lib timeout 300 python tools/fft_check.py 2>&1 | grep -v '9/9 rows' | grep -i 'differ\|rows' | head -3
  VLP_LIB=$PWD/$lib timeout 300 python tools/wave_drift.py 64 64 2>&1 | tail -2
done
