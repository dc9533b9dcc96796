set -x
for sm in 1 0; do MCO_ADALOMO_SMALL=$sm python tools/small_vec_prof.py; done
MCO_ADALOMO_SMALL=1 ncu --set full --import-source on -k regex:k_small_vec -c 2 -o /tmp/small -f python tools/small_vec_prof.py > /dev/null 2>&1
ncu -i /tmp/small.ncu-rep --page details --csv > gpurun_out/small_details.csv
ncu -i /tmp/small.ncu-rep --page source --csv --print-source sass > gpurun_out/small_source.csv 2>&1
ls -la gpurun_out
