# round-2 m: tile counter claimed one tile ahead without a blocking store (atomic overlaps the
# tile) -- full GPU tests, small configs and the default bench
bash scripts/gpu_session.sh r2m tests small bench
