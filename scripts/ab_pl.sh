#!/bin/bash
for v in _variants/*.so; do echo "== $v"; LBK_LIB=$PWD/$v python scripts/ab_powerlaw.py 10000; done
