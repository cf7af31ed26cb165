# Sustained int8 MMA peak with clock samples during the run (round-2 roofline denominator).
set -e
cd "$(dirname "$0")"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/i8_peak i8_peak.cu
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_throttle_reasons.active --format=csv -lms 100 > /tmp/i8_clocks.csv &
SMI=$!
/tmp/i8_peak ${1:-1000000}
kill $SMI
echo "clock samples (sm MHz, max, W, reasons):"; sort /tmp/i8_clocks.csv | uniq -c | sort -rn | head -8
