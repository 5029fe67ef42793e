"""B200-native irradiance-matrix engine for arXiv 2103.14137 (UV-disinfection
coverage planning): the C-ABI library libuvd.so (include/uvd.h) and its thin
Python binding `paper_2103_14137_b200.uvd`.  The CUDA library is loaded on
first use and there is no CPU fallback."""
