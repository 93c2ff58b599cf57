"""ORACLE — CPU restatements used only as the checker (tests/, smoke(), bench.py's
cpu_baseline and --impl reference legs).  The product package never imports this."""
