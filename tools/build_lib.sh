#!/bin/bash
# Build libbk.so without importing the package (which needs the library).
cd "$(dirname "$0")/.." && python -c "
import importlib.util, sys
spec = importlib.util.spec_from_file_location('b', 'paper_2504_02117_b200/build.py')
b = importlib.util.module_from_spec(spec); spec.loader.exec_module(b)
print(b.build(force='--force' in sys.argv))" "$@"
