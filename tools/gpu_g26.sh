timeout 600 python -m pytest tests/test_cli.py -q -p no:cacheprovider 2>&1 | tail -25
