# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
ATOS_LIB=paper_2112_00132_b200/variants/libatos_wprof.so timeout 300 python tools/pr_variants.py --runs 1 --no-oracle --variants '{"t1024": {"cta_threads": 1024}, "t512": {"cta_threads": 512}}' > gpurun_out/wprof.md 2>&1
ATOS_LIB=paper_2112_00132_b200/variants/libatos_wprof.so timeout 300 python tools/pr_variants.py --app bfs --runs 1 --no-oracle --variants '{"t256": {"cta_threads": 256}}' >> gpurun_out/wprof.md 2>&1
timeout 1700 python -m pytest tests -q -m gpu -x > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest.log
