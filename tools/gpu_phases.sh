# per-phase cycle breakdown of normal steps on the bench config (rebuilds with -DECONO_PROF_PHASES on the box)
mkdir -p gpurun_out
ECONO_PROF_PHASES=1 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/phases_build.log 2>&1
timeout 900 python tools/probe_scale.py --counts ${COUNTS:-888} --iters 1000 --lanes 0 > gpurun_out/phases.log 2>&1
