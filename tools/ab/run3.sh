# A/B/C: up to three builds of libdpm_b200.so on one box; ncu kernel time of
# the projection kernel per case (MODE=profile times the moments-pipeline pass)
cases=${CASES:-"cfg5|1024^3 u16 K4|cfg4"}
IFS='|' read -ra CS <<< "$cases"
for rep in 1 2; do
  for v in A B C; do
    [ -f tools/ab/$v.so ] || continue
    cp tools/ab/$v.so paper_2012_08099_b200/libdpm_b200.so
    for c in "${CS[@]}"; do
      t=$(ncu --metrics gpu__time_duration.sum --clock-control none -k regex:${KREGEX:-project_stream} -c 3 --csv python tools/time_project.py "$c" ${MODE:-} 2>/dev/null | grep ${KREGEX:-project_stream} | tail -1 | rev | cut -d, -f1 | rev)
      echo "$rep $v $c $t"
    done
  done
done
