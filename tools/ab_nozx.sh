set -e
cd paper_2012_08099_b200/csrc
rm -f _build/project_stream.o ../libdpm_b200.so
make -s EXTRA="-DDPM_NO_ZX=1" 2>&1 | grep -E "registers" | head -0
grep -B1 -A2 "project_stream_kernelItLi[45]" _build/project_stream.ptxas.log | grep -E "registers|spill" | head -4
cd ../..; echo "NO_ZX (16 warps for K<=4)"; python tools/time_project.py 1024; cd paper_2012_08099_b200/csrc
rm -f _build/project_stream.o ../libdpm_b200.so; make -s > /dev/null 2>&1
