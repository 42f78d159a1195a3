# gate: TMA requests from one lane vs rotated over the producer warp (MOE_TMA_SPREAD)
out=gpurun_out/${1:-r02_gspread}; mkdir -p $out
for w in lm mt; do for sp in 0 1; do
  MOE_TMA_SPREAD=$sp MOE_GATE_PROF=1 timeout 300 python tools/prof_step.py --workload $w --steps 4 > $out/${w}_sp$sp.log 2>&1
  echo "$w spread=$sp $(grep -h 'gate prof' $out/${w}_sp$sp.log | tail -1)" >> $out/summary.txt
  MOE_TMA_SPREAD=$sp /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gate -c 6 --csv --log-file $out/launch_${w}_sp$sp.csv python tools/prof_step.py --workload $w --steps 6 > /dev/null 2>&1
  echo "$w spread=$sp ncu us: $(python -c "
import csv
r=[x for x in csv.reader(open('$out/launch_${w}_sp$sp.csv')) if len(x)>10 and x[-3]=='gpu__time_duration.sum']
print([round(float(x[-1])/1000,1) for x in r])")" >> $out/summary.txt
done; done
cat $out/summary.txt
