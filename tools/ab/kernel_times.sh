python -m pytest tests/test_gpu_pipeline_quick.py -x -q 2>&1 | tail -1
for case in cfg3 cfg2 cfg5 "1024^3 u16 K4" cfg4; do
  t=$(ncu --metrics gpu__time_duration.sum --clock-control none -k regex:project_stream -c 3 --csv python tools/time_project.py "$case" 2>/dev/null | grep project_stream | tail -1 | rev | cut -d, -f1 | rev)
  echo "$case $t"
done
