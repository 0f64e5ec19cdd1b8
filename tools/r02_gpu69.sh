#!/bin/bash
V=paper_2104_14129_b200/csrc/build
python tools/with_variant.py $V/var_k2prof/libactnn.so -- tools/k2_phases.py
python tools/with_variant.py $V/var_k2nodmul/libactnn.so -- tools/k2_phases.py
