#!/usr/bin/env bash
# One GPU-box pass that regenerates a round's measurements (run under gpurun from
# the repo root; everything lands in gpurun_out/, summarised here afterwards):
#   GPU test suite + smoke, the default bench line, one bench line per config,
#   the ncu launch list of the default bench, and one `ncu --set full` capture of
#   each config's frame kernels (each ncu pass only after its command ran clean).
#
#   gpurun --timeout 3000 -- 'bash tools/measure_round.sh TAG'
#   python tools/ncu_summary.py gpurun_out/TAG_C3.ncu-rep --tag r2_C3_frame_TAG --config C3
set -u
TAG=${1:-m}
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/${TAG}_pytest.log 2>&1; echo rc=$? >> $OUT/${TAG}_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.log 2>&1; echo rc=$? >> $OUT/${TAG}_smoke.log
python bench.py > $OUT/${TAG}_bench_default.json 2> $OUT/${TAG}_bench_default.err
for c in C1 C2 C3 C4 C5; do
    extra="--steps 100 --no-cpu-baseline"; [ $c = C2 ] && extra="--steps 200"
    python bench.py --config $c $extra --warmup 3 > $OUT/${TAG}_bench_$c.json 2> $OUT/${TAG}_bench_$c.err
done
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/${TAG}_launches_run.log 2>&1 &&
    ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/${TAG}_launches.csv \
        python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/${TAG}_launches_ncu.log 2>&1
for c in C2 C3 C4 C5; do
    python tools/frames.py --config $c --frames 4 > $OUT/${TAG}_frames_$c.log 2>&1 &&
        ncu --set full --clock-control none --import-source on -k "regex:k_discretize|k_render|k_mip_top" -s 3 -c 3 \
            -o $OUT/${TAG}_$c python tools/frames.py --config $c --frames 4 > $OUT/${TAG}_ncu_$c.log 2>&1
done
echo done
