set -e
cd paper_2012_08099_b200/csrc
for v in 0 1 2 4 8 16 31; do
  rm -f _build/project_stream.o ../libdpm_b200.so
  make -s EXTRA="-DDPM_SKIP=$v" > /dev/null 2>&1
  cd ../..
  echo "SKIP=$v"
  python tools/time_project.py 1024 2>&1
  cd paper_2012_08099_b200/csrc
done
rm -f _build/project_stream.o ../libdpm_b200.so; make -s > /dev/null 2>&1
