# window kernel experiments: normal / no bias gathers / no output stores (timing only)
timeout 60 python tools/attn_bench.py local 64 2>&1 | grep default
for f in -DZS_WIN_NOGATHER -DZS_WIN_NOSTORE "-DZS_WIN_NOGATHER -DZS_WIN_NOSTORE"; do
  echo "== $f"
  ZS_BUILD_FLAGS="$f" timeout 200 python -m paper_2605_17633_b200.build --force > /dev/null 2>&1
  timeout 60 python tools/attn_bench.py local 64 2>&1 | grep default
done
