for mu in 2368 4736 9472; do
  echo "== min_units $mu"
  TG_SPAN_MIN_UNITS=$mu ncu --metrics gpu__time_duration.sum --csv python scripts/small_launches.py bb,ltm-r,rec 1024,4096,16384 write 2>/dev/null | python scripts/ncu_launch_times.py | awk 'NR%2==1'
  TG_SPAN_MIN_UNITS=$mu ncu --metrics gpu__time_duration.sum --csv python scripts/small_launches.py bb,ltm-r,rec 1024,4096,16384 edm 2>/dev/null | python scripts/ncu_launch_times.py | grep span_edm | awk 'NR%2==1'
done
