// ORACLE: IPM/NCL driver over the reference backend — filled in with the host IPM.
