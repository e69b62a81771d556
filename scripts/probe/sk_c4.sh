# RS C4 (W=1): stream-K tail forced on vs auto (off at 0.988 wave efficiency), steady state
for v in 0 1 0 1; do
  echo "== SHB_SK=$v"
  SHB_SK=$v AB_STEPS=600 python scripts/probe/long_blocks.py rs 2>&1 | grep "rs ours"
done
