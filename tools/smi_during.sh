# Sample nvidia-smi every 10 ms while running a command: clocks, power, throttle reasons.
#   bash tools/smi_during.sh out.csv <command...>
out=$1; shift
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv,noheader -lms 10 > "$out" &
smi=$!
sleep 1
"$@"
sleep 0.5
kill $smi
