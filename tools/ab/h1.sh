python bench.py --config 5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zstream -s 1 -c 1 -o gpurun_out/h1_cfg5_zs -f python bench.py --config 5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python - <<'PY' > gpurun_out/h1_512.txt 2>&1
import sys, torch
sys.path.insert(0, ".")
from paper_2012_08099_b200 import engine, configs
import tools.time_zs as tz
for name, vol, off in (("512 u16 noise", engine.synth_noise(512, 512, 0, 512, 5), 0),
                       ("cfg3 i16", torch.from_numpy(configs.cfg3()).cuda(), 1024),
                       ("cfg3 as u16 (+1024 on host)", torch.from_numpy((configs.cfg3().astype('int32') + 1024).astype('uint16')).cuda(), 0)):
    imgs, prof = engine.project_profile(vol, 4, offset=off)
    ms = tz.timeit(tz.graphed(lambda: engine.project_profile(vol, 4, offset=off, imgs=imgs, profile=prof)))
    print(name, round(ms * 1e3, 2), "us")
PY
