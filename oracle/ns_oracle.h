/* TEST INFRASTRUCTURE ONLY — see oracle.h.  NS RHS restatement (filled in below). */
#ifndef SMC_NS_ORACLE_H
#define SMC_NS_ORACLE_H
#endif
